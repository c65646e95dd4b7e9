#!/bin/bash
# Round-2 call H: does racecheck model mbarrier arrive/wait? (a minimal correct kernel);
# initcheck over the kernel families; the split-K 4 synccheck case without PDL.
O=gpurun_out/r2_sanitize3
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
./tools/microbench/mbar_racecheck > $O/mbar_plain.txt 2>&1
$CS --tool racecheck --racecheck-report all ./tools/microbench/mbar_racecheck > $O/racecheck_mbar_micro.txt 2>&1; echo "micro rc=$?"
OUTDIR=$O SAN_TOOLS="initcheck" SAN_CASES="list:k2_streamk_3m,k2_splitk2,k2_mat_all,k2c_qft9,k2m_qft7,k2m_dj7,k2s_qft4,registry,sv" SAN_TIMEOUT=300 bash tools/gpu_pin_sanitize.sh san
OUTDIR=$O SAN_TOOLS="synccheck" SAN_CASES="list:k2_splitk4_nopdl" SAN_TIMEOUT=300 bash tools/gpu_pin_sanitize.sh san
echo done
