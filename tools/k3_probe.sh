#!/usr/bin/env bash
# K3-TC timing experiments at BASELINE config 4 (run under gpurun from the
# repo root): kernel time per EXEM_TC_DEBUG mask (1: no epilogue arithmetic,
# 4: no operand TMA, 5: both) and the CTA-0 timeline of the last launch.
mkdir -p gpurun_out
for d in ${DBGS:-0 1 4 5}; do  # masks 2 and 32 need the probe build
  echo "dbg=$d"
  EXEM_TC_DEBUG=$d timeout 300 python bench.py --no-e2e --no-cpu --steps 3 --warmup 3 \
    | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['roofline']['kernel_ms_avg'], j['clocks'])"
done
for d in 0 5; do
  EXEM_TC_DEBUG=$d EXEM_TC_TRACE=gpurun_out/k3_trace_$d.txt timeout 300 python bench.py \
    --no-e2e --no-cpu --steps 3 --warmup 3 > /dev/null
  python tools/tc_trace.py gpurun_out/k3_trace_$d.txt
done
