#!/usr/bin/env bash
# ncu evidence for the two tcgen05 kernels (run under gpurun, one GPU):
#   launch list of a short C4 bench, one --set full capture of gains_tc_kernel
#   (C4 step) and of batch_tc_kernel (n=1M, d=256, l=4096, |S|=50).
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gains_tc \
  -s 1 -c 1 -o gpurun_out/prof_gains_tc -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu \
  > gpurun_out/ncu_full.log 2>&1
echo "gains_tc rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch_tc \
  -s 1 -c 1 -o gpurun_out/prof_batch_tc -f python tools/k4_probe.py --child --dims 256 --ks 50 \
  --n 1000000 --reps 1 > gpurun_out/ncu_full_b.log 2>&1
echo "batch_tc rc=$?"
