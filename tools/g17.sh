export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02q; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider > $O/pytest_kernels.log 2>&1; echo "exit $?" >> $O/pytest_kernels.log
timeout 900 python bench.py --gpus 4 --same-gpu --workload C2 --no-cpu-baseline > $O/bench_C2_4ranks_1gpu.json 2> $O/bench_C2_4ranks_1gpu.err
timeout 300 python tools/timeline.py --workload C4 --out $O/timeline_C4_N1.json.gz > $O/timeline_C4.json 2> $O/timeline_C4.err
timeout 600 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
ls -la $O
