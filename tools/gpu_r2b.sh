#!/bin/bash
# Round-2 call B: the CPU-baseline pin (full reference runs, 14 threads, in the
# background) next to the GPU validation of the round's changes, then the
# sanitizer follow-up (K2c; racecheck on the one-launch chains, sv, registry).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/R2b gpurun_out/r2_sanitize2
(QSB_REF_THREADS=14 timeout 3400 python tools/cpu_pin.py qft-9 entangle-10 dj-10 dj-11 entangle-11 qft-10 qft-11 qft-12 \
   > gpurun_out/R2b/cpu_pin.jsonl 2> gpurun_out/R2b/cpu_pin.err) &
PIN=$!
BENCH_FLAGS=--no-cpu-baseline CHAIN_AB="qft:9,qft:10,qft:11,entangle:9,entangle:10,entangle:11,entangle:12,qft:12" bash tools/gpu_validate.sh R2b
OUTDIR=gpurun_out/r2_sanitize2 SAN_TOOLS="memcheck synccheck" SAN_CASES="list:k2c,k2_splitk4" SAN_TIMEOUT=300 bash tools/gpu_pin_sanitize.sh san
SAN_TOOLS="racecheck" SAN_CASES="list:k2m,k2s,k2_mat_all,registry,sv" SAN_TIMEOUT=300 OUTDIR=gpurun_out/r2_sanitize2 bash tools/gpu_pin_sanitize.sh san
wait $PIN
echo "pin exit $?"
