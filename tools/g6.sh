# the GPU suite file by file (a hang in one file cannot hide the rest), with per-test durations
export CUDA_DEVICE_MAX_CONNECTIONS=32
O=gpurun_out/${TAG:-r02f}; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export PB_PARITY_LOG=$PWD/$O/parity.jsonl
for f in tests/test_gpu_*.py; do
  b=$(basename $f .py)
  s=$(date +%s)
  PB_WAIT_TIMEOUT_S=120 timeout ${FILE_TIMEOUT:-900} python -m pytest $f -m gpu -v -p no:cacheprovider --durations=0 > $O/$b.log 2>&1
  echo "exit $? after $(( $(date +%s) - s )) s" >> $O/$b.log
  tail -1 $O/$b.log >> $O/summary.txt; grep -E "passed|failed" $O/$b.log | tail -1 >> $O/summary.txt
done
ls -la $O
