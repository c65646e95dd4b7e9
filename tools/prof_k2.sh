#!/bin/bash
# ncu captures of the K2 variants on QFT-12 (one launch each, after warm-up).
TAG=${1:-r02}
for m in 3m 4m; do
  QSB_GEMM=$m timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm_ws -s 10 -c 1 \
     -o gpurun_out/${TAG}_k2ws_${m} -f python tools/quick_perf.py qft:12 > gpurun_out/${TAG}_ncu_${m}.log 2>&1
done
for m in 3m 4m; do QSB_GEMM=$m python tools/quick_perf.py qft:10 entangle:10 deutsch-jozsa:11 qft:12 > gpurun_out/${TAG}_perf_$m.log 2>&1; done
