#!/bin/bash
# One gpurun call after a change: GPU tests, smoke, the default bench line and the
# BASELINE configs, and the default command's ncu launch list.
#   gpurun --timeout 3000 -- 'bash tools/gpu_validate.sh R2a'
TAG=${1:-R2}
O=gpurun_out/$TAG
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 1800 python -m pytest tests -m gpu -q -x -s -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
for w in entangle-10 dj-11 qft-4; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline; done > $O/bench_configs.jsonl 2> $O/bench_configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu exit $?"
