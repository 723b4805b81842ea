export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02e; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 150 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 300 python tools/timeline.py --workload C2 --out $O/timeline_C2_N1.json.gz > $O/timeline_C2.json 2> $O/timeline_C2.err
timeout 600 python bench.py --check-oracle > $O/bench_C2.json 2> $O/bench_C2.err; echo "bench exit $?" >> $O/bench_C2.err
ls -la $O
