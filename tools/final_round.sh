#!/bin/bash
# Round-end evidence on one B200: GPU tests, smoke, bench lines for every
# backend and BASELINE config, the default command's ncu launch list, the
# 2/4/8-way QFT-14 projections, and the qubit sweep.
TAG=${1:-r53}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
bash tools/gpu_bench_round.sh ${TAG}
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${TAG}_bench_reference.json 2>&1
for w in qft-14 qft-12 entangle-10 dj-11; do timeout 300 python bench.py --backend structured --workload $w; done > gpurun_out/${TAG}_bench_structured.jsonl 2>&1
for w in qft-24 entangle-24; do timeout 300 python bench.py --backend fsv --workload $w; done > gpurun_out/${TAG}_bench_fsv.jsonl 2>&1
timeout 2000 python tools/sweep.py --out gpurun_out/${TAG}_sweep.md > gpurun_out/${TAG}_sweep.log 2>&1
