#!/bin/bash
# One gpurun call's worth of evidence: GPU tests, the bench line, the ncu launch list of the same command, and
# one `ncu --set full` capture of the top kernels. Usage (from the repo root, on the GPU box):
#   bash tools/gpu_round.sh TAG [WORKLOAD] [what...]     what ⊂ {build,tests,bench,launches,full}
set -u
TAG=${1:-r01}; WL=${2:-C2}; shift 2 || true
WHAT=${*:-build tests bench launches full}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export CUDA_DEVICE_MAX_CONNECTIONS=32
has() { [[ " $WHAT " == *" $1 "* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > "$OUT/gpu.txt" 2>&1
if has build; then timeout 600 python -c "import __graft_entry__ as g; g.build()" > "$OUT/build.log" 2>&1; echo "build exit $?" >> "$OUT/build.log"; fi
if has smoke; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke exit $?" >> "$OUT/smoke.log"; fi
if has tests; then timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > "$OUT/pytest_gpu.log" 2>&1; echo "pytest exit $?" >> "$OUT/pytest_gpu.log"; fi
if has bench; then timeout 900 python bench.py --workload "$WL" > "$OUT/bench_$WL.json" 2> "$OUT/bench_$WL.err"; echo "bench exit $?" >> "$OUT/bench_$WL.err"; fi
if has launches; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_$WL.csv" \
    python bench.py --workload "$WL" --steps 1 --warmup 1 --no-cpu-baseline > "$OUT/launches_$WL.log" 2>&1
  echo "ncu launches exit $?" >> "$OUT/launches_$WL.log"
fi
if has full; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:gemm|merge|attention|norm|logits" -s 40 -c 12 \
    -o "$OUT/full_$WL" python bench.py --workload "$WL" --steps 1 --warmup 1 --no-cpu-baseline > "$OUT/full_$WL.log" 2>&1
  echo "ncu full exit $?" >> "$OUT/full_$WL.log"
fi
ls -la "$OUT"
