#!/bin/bash
# Round-2 call D: row-block parts (QSB_PARTS) — tests, then the A/B against the default schedule.
cd "$(dirname "$0")/.."
O=gpurun_out/R2d
mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu.py -k "parts" -q -x -p no:cacheprovider > $O/pytest_parts.log 2>&1; echo "exit $?" >> $O/pytest_parts.log
tail -2 $O/pytest_parts.log
timeout 1200 python tools/env_ab.py qft:9,qft:10,qft:11,entangle:9,entangle:10,entangle:11,deutsch-jozsa:10,deutsch-jozsa:11,qft:12 \
  "base:" "p2:QSB_PARTS=2" "p4:QSB_PARTS=4" > $O/parts_ab.txt 2>&1
echo "ab exit $?"
