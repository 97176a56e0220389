for cg in 1 2; do for d in 100 256; do
  echo -n "cg=$cg "; EXEM_TCB_CG=$cg timeout 200 python tools/k4_probe.py --child --dims $d --ks 50 --n 1000000 2>&1 | tail -1
done; done
