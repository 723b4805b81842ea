export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02b; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build exit $?" >> $O/build.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > $O/pytest_kernels.log 2>&1; echo "exit $?" >> $O/pytest_kernels.log
timeout 300 python tools/merge_bench.py > $O/merge_bench.txt 2>&1
PB_SKINNY=0 timeout 300 python tools/skinny_sweep.py > $O/skinny_plain.txt 2>&1
timeout 600 python tools/skinny_sweep.py > $O/skinny_sweep.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py --check-oracle > $O/bench_C2.json 2> $O/bench_C2.err; echo "bench exit $?" >> $O/bench_C2.err
PB_SKINNY=0 timeout 600 python bench.py --no-cpu-baseline > $O/bench_C2_plain.json 2> $O/bench_C2_plain.err

timeout 2700 python -m pytest tests -m gpu -v -p no:cacheprovider --timeout 400 --durations=0 -k "not test_gpu_kernels" > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
ls -la $O
