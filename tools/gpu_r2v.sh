#!/bin/bash
O=gpurun_out/r2_sanitize6
mkdir -p $O
OUTDIR=$O SAN_TOOLS="memcheck initcheck synccheck" SAN_CASES="list:k2_streamk,k2_splitk2,k2_n9,k2_mat,k2c_qft9,k2m_qft7,k2m_qft8,k2s_qft4" SAN_TIMEOUT=300 bash tools/gpu_pin_sanitize.sh san
echo done
