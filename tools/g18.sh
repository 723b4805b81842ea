export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02r; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python tools/gemm_split_sweep.py > $O/split_sweep.txt 2>&1
ls -la $O
