#!/bin/bash
O=gpurun_out/R2l
mkdir -p $O
QSB_TRACE=1 timeout 600 python tools/host_call_perf.py qft:4,entangle:10,deutsch-jozsa:11,qft:10,qft:12 > $O/host_perf.txt 2> $O/host_trace.txt
cat $O/host_perf.txt
grep "memory check" $O/host_trace.txt | sort | uniq -c | sort -rn | head -8
for w in entangle-10 dj-11 qft-4; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline; done > $O/bench_configs.jsonl 2> $O/bench_configs.err
python - <<'PY'
import json
for line in open('gpurun_out/R2l/bench_configs.jsonl'):
    if line.startswith('{'):
        d=json.loads(line); e=d['e2e']; print(d['config']['workload'], d['value'], e['value'], e.get('value_plan_cached'))
PY
