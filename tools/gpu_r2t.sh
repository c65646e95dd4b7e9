#!/bin/bash
O=gpurun_out/R2t
mkdir -p $O
timeout 900 python tools/env_ab.py entangle:10,qft:10,deutsch-jozsa:10,entangle:11,qft:11,deutsch-jozsa:11 "w0:QSB_SK_WAVES=0" "w1:QSB_SK_WAVES=1" "def:" > $O/waves_ab.txt 2>&1
cat $O/waves_ab.txt
