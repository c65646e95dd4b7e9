#!/bin/bash
# Per-GEMM device times across one QFT-12 circuit for the 3M variants (ncu launch list).
TAG=${1:-r04}
for t in 4 5; do
  QSB_TILE=$t QSB_GEMM=3m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:zgemm -c 95 --csv \
     --log-file gpurun_out/${TAG}_layers_tile$t.csv python tools/quick_perf.py qft:12 > /dev/null 2>&1
  QSB_TILE=$t QSB_GEMM=3m python tools/quick_perf.py qft:10 entangle:10 deutsch-jozsa:11 qft:12 > gpurun_out/${TAG}_perf_tile$t.log 2>&1
done
QSB_GEMM=4m python tools/quick_perf.py qft:10 entangle:10 deutsch-jozsa:11 qft:12 > gpurun_out/${TAG}_perf_4m.log 2>&1
python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "tile" > gpurun_out/${TAG}_pytest_tiles.log 2>&1
