#!/bin/bash
O=gpurun_out/R2sweep
mkdir -p $O
timeout 3000 python tools/sweep.py --out $O/sweep.md > $O/sweep.log 2>&1; echo "sweep exit $?"
