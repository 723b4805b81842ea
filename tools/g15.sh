export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02o; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py tests/test_gpu_coldstart.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
PB_PARITY_LOG=$PWD/$O/parity.jsonl timeout 600 python -m pytest tests/test_gpu_target_parity.py -q -x -p no:cacheprovider > $O/pytest_target.log 2>&1; echo "exit $?" >> $O/pytest_target.log
timeout 300 python tools/attn_profile.py > $O/attn_two.txt 2>&1
PB_ATTN_ONE=1 timeout 300 python tools/attn_profile.py > $O/attn_one.txt 2>&1
timeout 900 python bench.py --workload C2p > $O/bench_C2p.json 2> $O/bench_C2p.err
timeout 900 python bench.py --workload C4 --no-cpu-baseline --steps 3 > $O/bench_C4.json 2> $O/bench_C4.err
ls -la $O
