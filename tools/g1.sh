export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build exit $?" >> $O/build.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err; echo "bench exit $?" >> $O/bench_C2.err
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not c2p" --durations=30 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
ls -la $O
