export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/r02l; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:attention_tc -s 3 -c 1 -o $O/attn_C5a python tools/attn_profile.py C5a > $O/attn_ncu.log 2>&1
PB_WAIT_TIMEOUT_S=120 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_2rank.py > $O/sanitizer_memcheck_2rank.log 2>&1; echo "exit $?" >> $O/sanitizer_memcheck_2rank.log
PB_WAIT_TIMEOUT_S=120 timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_2rank.py > $O/sanitizer_racecheck_2rank.log 2>&1; echo "exit $?" >> $O/sanitizer_racecheck_2rank.log
TAG=r02l WL=C2 bash tools/gpu_round.sh launches full > /dev/null 2>&1
ls -la $O
