# debug the cold-start hang seen in r02b (smoke / test_no_prompt...), then kernel tests
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02d; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
PB_WAIT_TIMEOUT_S=60 timeout 150 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
PB_DEBUG_ISSUER=1 PB_WAIT_TIMEOUT_S=60 timeout 150 python -m pytest tests/test_gpu_boundary.py -x -v -p no:cacheprovider -k "no_prompt and opt" > $O/noprompt.log 2>&1; echo "exit $?" >> $O/noprompt.log
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider > $O/pytest_kernels.log 2>&1; echo "exit $?" >> $O/pytest_kernels.log
for st in 3 4; do PB_GEMM_STAGES=$st timeout 300 python bench.py --no-cpu-baseline --steps 3 > $O/bench_stages$st.json 2>&1; done
ls -la $O
