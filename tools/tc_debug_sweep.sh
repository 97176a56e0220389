#!/usr/bin/env bash
# K3-TC debug-mask sweep (probe build: -DEXEM_TC_PROBE_BUILD), C4 bench kernel time per mask.
set -e
EXEM_NVCC_FLAGS="-DEXEM_TC_PROBE_BUILD" python -c "from paper_2101_08763_b200.build import build; build(force=True)" > /dev/null
for d in 0 1 2 4 3 5 6; do echo "dbg=$d"; EXEM_TC_DEBUG=$d timeout 300 python bench.py --no-e2e --no-cpu --steps 3 --warmup 3 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['roofline']['kernel_ms_avg'], j['clocks'])"; done
python -c "from paper_2101_08763_b200.build import build; build(force=True)" > /dev/null
