export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02u; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k gemm > $O/pytest_gemm.log 2>&1; echo "exit $?" >> $O/pytest_gemm.log
timeout 300 python tools/gemm_phases.py > $O/gemm_phases_l2.txt 2>&1
timeout 300 python tools/gemm_split_sweep.py > $O/split_l2.txt 2>&1
PB_GEMM_DSMEM=1 timeout 300 python tools/gemm_split_sweep.py > $O/split_dsmem.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/bench_C2_l2.json 2> $O/bench_C2_l2.err
PB_GEMM_DSMEM=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_C2_dsmem.json 2> $O/bench_C2_dsmem.err
ls -la $O
