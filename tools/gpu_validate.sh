#!/bin/bash
# One gpurun call after a change: GPU tests, smoke, the default bench line and the
# BASELINE configs, and the default command's ncu launch list.
#   gpurun --timeout 3000 -- 'bash tools/gpu_validate.sh R2a'
TAG=${1:-R2}
O=gpurun_out/$TAG
mkdir -p $O
export PYTHONUNBUFFERED=1
# new persistent kernels first, under a short limit (a protocol bug would hang here, not later)
timeout 420 python -m pytest tests/test_parity_gpu.py -k chain -q -x -p no:cacheprovider > $O/pytest_chain.log 2>&1; echo "exit $?" >> $O/pytest_chain.log
tail -2 $O/pytest_chain.log
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
tail -1 $O/smoke.log
timeout 600 python bench.py ${BENCH_FLAGS:-} > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
for w in entangle-10 dj-11 qft-4; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline; done > $O/bench_configs.jsonl 2> $O/bench_configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu exit $?"
if [ -n "$CHAIN_AB" ]; then
  timeout 1200 python tools/env_ab.py ${CHAIN_AB} "base:" "chain:QSB_CHAIN=1" "c1:QSB_CHAIN=1,QSB_CHAIN_SPLITS=1" \
    "c2:QSB_CHAIN=1,QSB_CHAIN_SPLITS=2" "c4:QSB_CHAIN=1,QSB_CHAIN_SPLITS=4" > $O/chain_ab.txt 2>&1
  echo "chain ab exit $?"
fi
