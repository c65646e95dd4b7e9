#!/bin/bash
# Final evidence for the final code: GPU tests, smoke, the default bench line, configs,
# reference arm, launch list, the dominant K2 launch under ncu --set full.
O=gpurun_out/R2end
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
for w in entangle-10 dj-11 qft-4; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5; done > $O/bench_configs.jsonl 2> $O/bench_configs.err
timeout 900 python bench.py --workload qft-14 --virtual-ranks 8 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_qft14_v8.json 2> $O/bench_qft14_v8.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu exit $?"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
   -k 'regex:zgemm_ws_kernel<\(bool\)1, \(bool\)1, \(bool\)1, \(bool\)0>' -s 20 -c 1 -o $O/k2_3m_qft12 \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_3m.log 2>&1; echo "ncu full exit $?"
