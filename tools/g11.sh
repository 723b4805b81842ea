export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02k; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > $O/pytest_kernels.log 2>&1; echo "exit $?" >> $O/pytest_kernels.log
timeout 900 python bench.py --workload C4 --no-cpu-baseline --steps 3 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 1200 python bench.py --workload C5a --host-alias 8 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_C5a.json 2> $O/bench_C5a.err
timeout 600 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
ls -la $O
