#!/bin/bash
# Round evidence: GPU tests, smoke, bench lines + launch list, reference arm,
# one ncu --set full capture of K2m (QFT-8), and the qubit sweep.
TAG=${1:-r84}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
bash tools/gpu_bench_round.sh ${TAG}
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/${TAG}_bench_reference.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mid_dmma -s 2 -c 1 \
    -o gpurun_out/${TAG}_k2m_qft8 python tools/mid_perf.py qft:8 > gpurun_out/${TAG}_k2m_ncu.log 2>&1
timeout 2400 python tools/sweep.py --out gpurun_out/${TAG}_sweep.md > gpurun_out/${TAG}_sweep.log 2>&1
