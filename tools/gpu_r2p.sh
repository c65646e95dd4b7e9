#!/bin/bash
O=gpurun_out/R2p
mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu.py -k "mid" -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 900 python tools/env_ab.py qft:6,qft:7,qft:8,entangle:7,entangle:8,deutsch-jozsa:7,deutsch-jozsa:8 "4m:QSB_MID_3M=0" "3m:QSB_MID_3M=1" > $O/mid3m_ab.txt 2>&1
cat $O/mid3m_ab.txt
