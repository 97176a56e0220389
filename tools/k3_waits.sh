#!/usr/bin/env bash
# K3-TC issuer wait placement / epilogue polling sweep at config 4 (gpurun).
for w in 0 1 2 3 4 5 6 8 9 10 12; do
  echo -n "waits=$w "
  EXEM_TC_WAITS=$w timeout 300 python bench.py --no-e2e --no-cpu --steps 4 --warmup 3 \
    | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(round(j['roofline']['kernel_ms_avg'],2), j['clocks']['sm_mhz'])"
done
