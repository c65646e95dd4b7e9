#!/bin/bash
# One gpurun call: (1) pin the CPU-baseline model to full reference runs on the
# box's host cores; (2) compute-sanitizer memcheck / racecheck / synccheck /
# initcheck over every kernel family at small shapes.
#   gpurun --timeout 3000 -- 'bash tools/gpu_pin_sanitize.sh [pin|san|all]'
set -u
cd "$(dirname "$0")/.."
OUT=${OUTDIR:-gpurun_out/r2_sanitize}
mkdir -p "$OUT"
WHAT=${1:-all}
nproc > "$OUT/nproc.txt"; lscpu | head -20 >> "$OUT/nproc.txt"
if [ "$WHAT" = pin ] || [ "$WHAT" = all ]; then
  timeout 1500 python tools/cpu_pin.py ${PIN_LIST:-qft-9 qft-10 entangle-10 entangle-11 dj-10 dj-11 qft-11} \
    > "$OUT/cpu_pin.jsonl" 2> "$OUT/cpu_pin.err"
  echo "cpu_pin rc=$?"
fi
if [ "$WHAT" = san ] || [ "$WHAT" = all ]; then
  CS=/usr/local/cuda/bin/compute-sanitizer
  CASES=$(python tools/sanitize_cases.py ${SAN_CASES:-list})
  for tool in ${SAN_TOOLS:-memcheck synccheck racecheck initcheck}; do
    for c in $CASES; do
      extra=""
      [ "$tool" = racecheck ] && extra="--racecheck-report all"
      t0=$(date +%s)
      timeout ${SAN_TIMEOUT:-420} $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
        python tools/sanitize_cases.py $c > "$OUT/${tool}_${c}.txt" 2>&1
      rc=$?
      echo "$tool $c rc=$rc $(( $(date +%s) - t0 ))s $(grep -m1 -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$OUT/${tool}_${c}.txt")" | tee -a "$OUT/summary.txt"
    done
  done
fi
