#!/usr/bin/env bash
# Standard measurement pass on the GPU box (run under gpurun from the repo
# root).  Everything lands in gpurun_out/.  Each step is bounded by its own
# timeout so a hang cannot take the box down.
#   tools/gpu_check.sh [tests] [bench] [ncu] [smoke]
set -u
OUT=gpurun_out
mkdir -p "$OUT"
want() { [ $# -eq 0 ] && return 0; for a in "${ARGS[@]}"; do [ "$a" = "$1" ] && return 0; done; return 1; }
ARGS=("$@")
[ ${#ARGS[@]} -eq 0 ] && ARGS=(tests bench ncu)

nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv | tee "$OUT/gpu.txt"

if want smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke rc=$?"; tail -3 "$OUT/smoke.log"
fi
if want tests; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > "$OUT/tests_gpu.log" 2>&1
  echo "tests rc=$?"; tail -15 "$OUT/tests_gpu.log"
fi
if want bench; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench rc=$?"; cat "$OUT/bench.json"; tail -5 "$OUT/bench.err"
fi
if want ncu; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sub \
    > "$OUT/ncu_launches.log" 2>&1
  echo "ncu launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gains_tc \
    -s 1 -c 1 -o "$OUT/prof_gains_tc" -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sub \
    > "$OUT/ncu_full.log" 2>&1
  echo "ncu full rc=$?"; tail -3 "$OUT/ncu_full.log"
fi
