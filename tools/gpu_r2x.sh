#!/bin/bash
O=gpurun_out/R2x
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
timeout 3000 python tools/sweep.py --out $O/sweep.md > $O/sweep.log 2>&1; echo "sweep exit $?"
