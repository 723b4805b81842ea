export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02p; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py tests/test_gpu_coldstart.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
PB_PARITY_LOG=$PWD/$O/parity.jsonl timeout 600 python -m pytest tests/test_gpu_target_parity.py -q -p no:cacheprovider > $O/pytest_target.log 2>&1; echo "exit $?" >> $O/pytest_target.log
for i in 1 2 3; do PB_PARITY_LOG=$PWD/$O/parity_rep.jsonl timeout 600 python -m pytest tests/test_gpu_target_parity.py -q -p no:cacheprovider -k c4 >> $O/pytest_target_rep.log 2>&1; done
timeout 300 python tools/attn_profile.py > $O/attn_two.txt 2>&1
ls -la $O
