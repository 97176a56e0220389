#!/usr/bin/env bash
# K3-TC timing experiments at BASELINE config 4 (run under gpurun from the
# repo root): kernel time per EXEM_TC_DEBUG mask (1: no epilogue arithmetic,
# 4: no operand TMA, 5: both; 2 no MMA and 32 no TMEM drain need the extra
# branches of the r01 probe commit) and the CTA-0 timeline of the last launch.
# The masks exist only in a probe build (-DEXEM_TC_PROBE_BUILD); the script
# builds it, runs, and restores the normal build.
set -e
mkdir -p gpurun_out
EXEM_NVCC_FLAGS="-DEXEM_TC_PROBE_BUILD" python -c "from paper_2101_08763_b200.build import build; build(force=True)" > /dev/null
for d in ${DBGS:-0 1 4 5}; do
  echo "dbg=$d"
  EXEM_TC_DEBUG=$d timeout 300 python bench.py --no-e2e --no-cpu --steps 3 --warmup 3 \
    | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['roofline']['kernel_ms_avg'], j['clocks'])"
done
for d in 0 5; do
  EXEM_TC_DEBUG=$d EXEM_TC_TRACE=gpurun_out/k3_trace_$d.txt timeout 300 python bench.py \
    --no-e2e --no-cpu --steps 3 --warmup 3 > /dev/null
  python tools/tc_trace.py gpurun_out/k3_trace_$d.txt
done
python -c "from paper_2101_08763_b200.build import build; build(force=True)" > /dev/null
