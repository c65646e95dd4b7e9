#!/bin/bash
# Runs on the GPU box (gpurun): bench lines, the ncu launch list of the bench
# command, and one full ncu capture of the K2 GEMM. Outputs land in gpurun_out/.
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt
python bench.py > gpurun_out/${TAG}_bench_qft12.json 2> gpurun_out/${TAG}_bench_qft12.err
python bench.py --workload entangle-10 --no-cpu-baseline > gpurun_out/${TAG}_bench_entangle10.json 2>&1
python bench.py --workload dj-11 --no-cpu-baseline > gpurun_out/${TAG}_bench_dj11.json 2>&1
python bench.py --workload qft-4 > gpurun_out/${TAG}_bench_qft4.json 2>&1
# launch list of the bench command (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_qft12.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# one full capture of the dominant kernel
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm -s 10 -c 1 \
    -o gpurun_out/${TAG}_k2_qft12 -f python tools/quick_perf.py qft:12 > gpurun_out/${TAG}_ncu_full.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:expand -c 1 \
    -o gpurun_out/${TAG}_k1_qft12 -f python tools/quick_perf.py qft:12 > /dev/null 2>&1
ls -la gpurun_out
