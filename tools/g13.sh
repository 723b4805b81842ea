export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02m; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > $O/pytest_kernels.log 2>&1; echo "exit $?" >> $O/pytest_kernels.log
timeout 300 python -m pytest tests/test_gpu_decode.py tests/test_gpu_coldstart.py -q -x -p no:cacheprovider > $O/pytest_decode_cold.log 2>&1; echo "exit $?" >> $O/pytest_decode_cold.log
timeout 300 python tools/attn_profile.py > $O/attn_profile.txt 2>&1
timeout 600 ncu --set full -k regex:merge_kernel -c 1 -o $O/merge_2048_r16 python tools/merge_one.py 2048 2048 16 > $O/merge_ncu1.log 2>&1
timeout 600 ncu --set full -k regex:merge_kernel -c 1 -o $O/merge_5120x20480_r64 python tools/merge_one.py 5120 20480 64 > $O/merge_ncu2.log 2>&1
timeout 600 ncu --set full -k regex:merge_kernel -c 1 -o $O/merge_C2layer_batch python tools/merge_one.py 2048 2048 16 2 > $O/merge_ncu3.log 2>&1
timeout 900 python bench.py --workload C4 --no-cpu-baseline --steps 3 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 1200 python bench.py --workload C5a --host-alias 8 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_C5a.json 2> $O/bench_C5a.err
timeout 600 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
ls -la $O
