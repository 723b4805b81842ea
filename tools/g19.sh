export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02s; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_coldstart.py tests/test_gpu_switch.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
PB_PARITY_LOG=$PWD/$O/parity.jsonl timeout 600 python -m pytest tests/test_gpu_target_parity.py -q -p no:cacheprovider -k c3 > $O/pytest_c3.log 2>&1; echo "exit $?" >> $O/pytest_c3.log
timeout 900 python bench.py --workload C3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
PB_NO_MB_BATCH=1 timeout 900 python bench.py --workload C3 --no-cpu-baseline > $O/bench_C3_nobatch.json 2> $O/bench_C3_nobatch.err
ls -la $O
