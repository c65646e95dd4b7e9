#!/bin/bash
# Round-2 call F: the data-parallel-first stream-K order as default + the plan-cache key
# fix: GPU tests, smoke, A/B of both orders, one ncu --set full of the dominant 3M K2
# launch (DRAM bytes for roofline.traffic), the default bench line.
TAG=${1:-R2f}
O=gpurun_out/$TAG
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python tools/env_ab.py qft:10,qft:11,qft:12,entangle:11,entangle:12,deutsch-jozsa:11,deutsch-jozsa:12 "dp:" "sk:QSB_SK_DP=0" > $O/sk_dp_ab.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
   -k 'regex:zgemm_ws_kernel<\(bool\)1, \(bool\)1, \(bool\)1, \(bool\)0>' -s 20 -c 1 -o $O/k2_3m_qft12 \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_3m.log 2>&1; echo "ncu exit $?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
