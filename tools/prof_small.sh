#!/bin/bash
# ncu captures of K2 at the small BASELINE sizes (Entangle-10, DJ-11) and QFT-12 for reference.
TAG=${1:-r16}
for spec in entangle:10 deutsch-jozsa:11; do
  name=${spec/:/}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm -s 2 -c 3 \
     -o gpurun_out/${TAG}_k2_${name} -f python tools/quick_perf.py $spec > gpurun_out/${TAG}_ncu_${name}.log 2>&1
done
