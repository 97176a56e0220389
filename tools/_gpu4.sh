set -u
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/epi_probe tools/epi_probe.cu && timeout 120 /tmp/epi_probe > gpurun_out/epi_probe.json; echo "epi rc=$?"; cat gpurun_out/epi_probe.json
timeout 300 python tools/k3_probe_data.py blobs 6; timeout 300 python tools/k3_probe_data.py gauss 6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gains_tc -s 2 -c 1 -o gpurun_out/k3_blobs -f python tools/k3_probe_data.py blobs 4 > gpurun_out/k3_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/k3_ncu.log
