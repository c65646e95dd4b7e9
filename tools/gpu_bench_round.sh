#!/bin/bash
# Bench lines + the ncu launch list of the default bench command, and the
# row-block projections for the multi-GPU configurations (one shard on one GPU).
TAG=${1:-r21}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_qft12.json 2> gpurun_out/${TAG}_bench_qft12.err
timeout 600 python bench.py --workload qft-12 --virtual-ranks 8 --no-cpu-baseline > gpurun_out/${TAG}_bench_qft12_v8.json 2>&1
timeout 900 python bench.py --workload qft-14 --virtual-ranks 8 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_qft14_v8.json 2>&1
for w in entangle-10 dj-11 qft-4; do
  timeout 600 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_qft12.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
