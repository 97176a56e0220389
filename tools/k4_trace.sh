# K4-TC CTA-0 timelines (trace build), d = ${D:-100}, |S| = 50, several EXEM_TCB_DEBUG masks.
set -e
EXEM_NVCC_FLAGS="-DEXEM_TCB_TRACE_BUILD -DEXEM_TCB_PROBE_BUILD" python -c "from paper_2101_08763_b200.build import build; build(force=True)" > /dev/null
for dbg in ${DBGS:-0 7}; do
  EXEM_TCB_DEBUG=$dbg EXEM_TCB_TRACE=gpurun_out/k4_trace_$dbg.txt timeout 200 \
    python tools/k4_probe.py --child --dims ${D:-100} --ks ${K:-50} --n 1000000 --reps 2 | tail -1
done
python -c "from paper_2101_08763_b200.build import build; build(force=True)" > /dev/null
