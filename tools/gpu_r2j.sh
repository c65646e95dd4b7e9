#!/bin/bash
O=gpurun_out/r2_sanitize5
mkdir -p $O
OUTDIR=$O SAN_TOOLS="synccheck memcheck" SAN_CASES="list:k2_splitk,k2_streamk" SAN_TIMEOUT=300 bash tools/gpu_pin_sanitize.sh san
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider -k "split or stream or tile" > $O/pytest_parity.log 2>&1; echo "exit $?" >> $O/pytest_parity.log
tail -2 $O/pytest_parity.log
timeout 600 python tools/env_ab.py qft:9,qft:10,qft:12,entangle:10,deutsch-jozsa:11 "base:" > $O/perf.txt 2>&1
cat $O/perf.txt
