#!/bin/bash
# Runs on the GPU box (gpurun): GPU tests, smoke, bench lines, the ncu launch
# list of the bench command and one full ncu capture of the production K2.
TAG=${1:-r08}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt
lscpu > gpurun_out/${TAG}_lscpu.txt; uname -m >> gpurun_out/${TAG}_lscpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_qft12.json 2> gpurun_out/${TAG}_bench_qft12.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${TAG}_bench_ref_qft12.json 2>&1
for w in entangle-10 dj-11 qft-4; do
  timeout 600 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_qft12.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm -s 10 -c 1 \
    -o gpurun_out/${TAG}_k2_qft12 -f python tools/quick_perf.py qft:12 > gpurun_out/${TAG}_ncu_full.log 2>&1
ls -la gpurun_out
