#!/bin/bash
# Round-2 evidence refresh after the cold-path / NCCL-loading fixes: GPU tests, smoke,
# the default bench line, the BASELINE configs, the reference arm.
O=gpurun_out/R2n
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
for w in entangle-10 dj-11 qft-4; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5; done > $O/bench_configs.jsonl 2> $O/bench_configs.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref exit $?"
