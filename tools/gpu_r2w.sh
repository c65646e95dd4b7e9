#!/bin/bash
# The reference's full QFT-12 simulate_full_state on an otherwise idle GPU box, all 16 host
# cores (round 2's first full run used 14 threads next to GPU tests), with the model beside it.
O=gpurun_out/R2w
mkdir -p $O
nproc > $O/nproc.txt
timeout 3300 python tools/cpu_pin.py qft-12 qft-11 > $O/cpu_pin.jsonl 2> $O/cpu_pin.err
echo "pin exit $?"
cat $O/cpu_pin.jsonl | cut -c1-300
