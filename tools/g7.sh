export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02g; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider > $O/pytest_kernels.log 2>&1; echo "exit $?" >> $O/pytest_kernels.log
timeout 300 python tools/gemm_phases.py > $O/gemm_phases.txt 2>&1
timeout 300 python tools/merge_bench.py > $O/merge_bench.txt 2>&1
PB_WAIT_TIMEOUT_S=100 timeout 600 compute-sanitizer --tool memcheck --leak-check no python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_memcheck.log 2>&1; echo "exit $?" >> $O/sanitizer_memcheck.log
PB_WAIT_TIMEOUT_S=100 timeout 600 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_synccheck.log 2>&1; echo "exit $?" >> $O/sanitizer_synccheck.log
timeout 600 python bench.py --check-oracle > $O/bench_C2.json 2> $O/bench_C2.err; echo "bench exit $?" >> $O/bench_C2.err
timeout 900 python bench.py --workload C4 --check-oracle --no-cpu-baseline --steps 3 > $O/bench_C4.json 2> $O/bench_C4.err; echo "bench exit $?" >> $O/bench_C4.err

for cfg in "148 3" "148 4" "148 0"; do set -- $cfg; PB_GEMM_CTAS=$1 PB_GEMM_STAGES=$2 timeout 300 python bench.py --no-cpu-baseline --no-profile --steps 3 > $O/bench_ctas$1_st$2.json 2>&1; done
PB_NORM_CTA=1 timeout 300 python bench.py --no-cpu-baseline --no-profile --steps 3 > $O/bench_normcta.json 2>&1
ls -la $O
