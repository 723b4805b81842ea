export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02h; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > $O/pytest_kernels.log 2>&1; echo "exit $?" >> $O/pytest_kernels.log
timeout 300 python tools/gemm_phases.py > $O/gemm_phases.txt 2>&1
timeout 600 python bench.py --check-oracle > $O/bench_C2.json 2> $O/bench_C2.err; echo "bench exit $?" >> $O/bench_C2.err
PB_WAIT_TIMEOUT_S=120 timeout 900 python -m pytest tests/test_gpu_switch.py tests/test_gpu_coldstart.py -v -p no:cacheprovider > $O/pytest_switch_coldstart.log 2>&1; echo "exit $?" >> $O/pytest_switch_coldstart.log
timeout 300 python tools/timeline.py --workload C2 --out $O/timeline_C2_N1.json.gz > $O/timeline_C2.json 2> $O/timeline_C2.err
ls -la $O
