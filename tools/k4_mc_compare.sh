for mc in 1 2 4; do for d in 100 256; do echo -n "mc=$mc "; EXEM_TCB_MC=$mc timeout 200 python tools/k4_probe.py --child --dims $d --ks 50 --n 1000000 2>&1 | tail -1; done; done
