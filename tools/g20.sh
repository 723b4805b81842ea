export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02t; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "attention" > $O/pytest_attn.log 2>&1; echo "exit $?" >> $O/pytest_attn.log
timeout 300 python tools/attn_profile.py > $O/attn_poly25.txt 2>&1
PB_PARITY_LOG=$PWD/$O/parity.jsonl timeout 600 python -m pytest tests/test_gpu_target_parity.py -q -p no:cacheprovider > $O/pytest_target.log 2>&1; echo "exit $?" >> $O/pytest_target.log
ls -la $O
