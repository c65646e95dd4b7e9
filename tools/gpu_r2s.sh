#!/bin/bash
O=gpurun_out/R2s
mkdir -p $O
timeout 900 python tools/env_ab.py qft:11,qft:12 "g16:" "g0:QSB_SK_GROUP=0" "g4:QSB_SK_GROUP=4" > $O/group_ab.txt 2>&1
cat $O/group_ab.txt
for g in 0 4 16; do
  QSB_SK_GROUP=$g timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
     --kernel-name-base demangled -k 'regex:zgemm_ws_kernel<\(bool\)1, \(bool\)1, \(bool\)1, \(bool\)0>' -s 10 -c 3 --csv \
     --log-file $O/dram_g$g.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
echo done
