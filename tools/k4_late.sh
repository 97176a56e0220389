# K4-TC: next accumulator buffer acquired inside the tile (LATE=0) or after its commit (LATE=1)
for k in ${KS:-50}; do for d in ${DS:-100 256}; do for late in 0 1; do echo -n "late=$late "; EXEM_TCB_LATE=$late timeout 200 python tools/k4_probe.py --child --dims $d --ks $k --n 1000000 2>&1 | tail -1; done; done; done
