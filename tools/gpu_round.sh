#!/bin/bash
# One gpurun call's worth of evidence (run from the repo root on the GPU box):
#   TAG=r02x WL=C2 bash tools/gpu_round.sh [what...]
#   what ⊂ {build smoke suite bench launches full timeline phases merge}   (default: build smoke suite bench)
# suite: the GPU test files one by one (a hang in one cannot hide the rest), per-test durations, parity log.
set -u
TAG=${TAG:-r02}; WL=${WL:-C2}
WHAT=${*:-build smoke suite bench}
O=gpurun_out/$TAG
mkdir -p "$O"
export CUDA_DEVICE_MAX_CONNECTIONS=32
has() { [[ " $WHAT " == *" $1 "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$O/gpu.txt" 2>&1
if has build; then timeout 600 python -c "import __graft_entry__ as g; g.build()" > "$O/build.log" 2>&1; echo "build exit $?" >> "$O/build.log"; fi
if has smoke; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; echo "smoke exit $?" >> "$O/smoke.log"; fi
if has suite; then
  export PB_PARITY_LOG=$PWD/$O/parity.jsonl
  for f in tests/test_gpu_*.py; do
    b=$(basename "$f" .py); s=$(date +%s)
    PB_WAIT_TIMEOUT_S=120 timeout ${FILE_TIMEOUT:-900} python -m pytest "$f" -m gpu -v -p no:cacheprovider --durations=0 > "$O/$b.log" 2>&1
    echo "exit $? after $(( $(date +%s) - s )) s" >> "$O/$b.log"
    { echo "$b: $(tail -1 "$O/$b.log")"; grep -E "passed|failed" "$O/$b.log" | tail -1; } >> "$O/summary.txt"
  done
fi
if has bench; then timeout 900 python bench.py --workload "$WL" > "$O/bench_$WL.json" 2> "$O/bench_$WL.err"; echo "bench exit $?" >> "$O/bench_$WL.err"; fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$O/launches_$WL.csv" \
    python bench.py --workload "$WL" --steps 1 --warmup 1 --no-cpu-baseline --check-oracle 0 > "$O/launches_$WL.log" 2>&1
  echo "ncu launches exit $?" >> "$O/launches_$WL.log"
fi
if has full; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:gemm|merge|attention|norm|logits" -s 40 -c 14 \
    -o "$O/full_$WL" python bench.py --workload "$WL" --steps 1 --warmup 1 --no-cpu-baseline --check-oracle 0 > "$O/full_$WL.log" 2>&1
  echo "ncu full exit $?" >> "$O/full_$WL.log"
fi
if has timeline; then timeout 300 python tools/timeline.py --workload "$WL" --out "$O/timeline_${WL}_N1.json.gz" > "$O/timeline_$WL.json" 2> "$O/timeline_$WL.err"; fi
if has phases; then timeout 300 python tools/gemm_phases.py > "$O/gemm_phases.txt" 2>&1; fi
if has merge; then timeout 300 python tools/merge_bench.py > "$O/merge_bench.txt" 2>&1; fi
ls -la "$O"
