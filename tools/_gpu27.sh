set -u
mkdir -p gpurun_out
for d in 2 16 100; do
  for q in 2 4; do
  EXEM_K3_EPI=$q EXEM_LIB_PATH=paper_2101_08763_b200/_ab/libPROBE.so EXEM_TC_TRACE=gpurun_out/k3_trace_d${d}_q$q.txt timeout 300 python bench.py --points 100000 --dim $d --no-e2e --no-cpu --no-sub --steps 3 --warmup 3 > /dev/null 2>&1
  echo "d=$d q=$q"; python tools/tc_trace.py gpurun_out/k3_trace_d${d}_q$q.txt | tail -4
  done
done
