#!/bin/bash
O=gpurun_out/R2o
mkdir -p $O
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench exit $?"
timeout 600 python bench.py --workload dj-11 --steps 5 --warmup 3 > $O/bench_dj11.json 2> $O/bench_dj11.err; echo "bench dj exit $?"
tail -c 1500 $O/bench.json
tail -3 $O/bench.err
