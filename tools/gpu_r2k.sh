#!/bin/bash
O=gpurun_out/R2k
mkdir -p $O
timeout 900 python -m pytest tests/test_host_cache_gpu.py tests/test_parity_gpu.py -k "cache or registry or table or monomial or dj or deutsch or changed or mutation" -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
QSB_TRACE=1 timeout 600 python tools/host_call_perf.py qft:4,entangle:10,deutsch-jozsa:11,qft:10,qft:12 > $O/host_perf.txt 2> $O/host_trace.txt
cat $O/host_perf.txt
grep "qsb plan" $O/host_trace.txt | sort | uniq -c | sort -rn | head -20
