#!/bin/bash
# Round-2 call C: the CPU-baseline pin on an otherwise idle box (all host cores),
# dense timings to the HBM limit (QFT-15 whole, QFT-16 one 8-way row shard), and
# one ncu --set full capture of the Entangle-10 K2 GEMM (the weakest BASELINE config).
cd "$(dirname "$0")/.."
O=gpurun_out/R2c
mkdir -p $O
timeout 900 python tools/cpu_pin.py qft-9 entangle-10 dj-10 dj-11 entangle-11 qft-10 qft-11 > $O/cpu_pin.jsonl 2> $O/cpu_pin.err
echo "pin exit $?"
timeout 2400 python tools/hbm_limit.py qft-15 qft-16/8 > $O/hbm_limit.jsonl 2> $O/hbm_limit.err
echo "hbm exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:zgemm_ws_kernel -s 40 -c 1 -o $O/k2_entangle10 \
  python bench.py --workload entangle-10 --steps 2 --warmup 5 --no-cpu-baseline > $O/ncu_entangle10.log 2>&1
echo "ncu exit $?"
