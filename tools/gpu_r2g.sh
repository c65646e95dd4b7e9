#!/bin/bash
# Round-2 call G: grouped tile numbering for the data-parallel waves (QSB_SK_GROUP):
# tests, time A/B, DRAM bytes of the dominant 3M launch per grouping.
O=gpurun_out/R2g
mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_host_cache_gpu.py tests/test_multi_gpu.py -k "grouped or switch or allgather" -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 1200 python tools/env_ab.py qft:11,qft:12,deutsch-jozsa:12,entangle:12 "g0:QSB_SK_GROUP=0" "g8:QSB_SK_GROUP=8" "g16:QSB_SK_GROUP=16" "g32:QSB_SK_GROUP=32" > $O/group_ab.txt 2>&1
for g in 0 8 16 32; do
  QSB_SK_GROUP=$g timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
     --kernel-name-base demangled -k 'regex:zgemm_ws_kernel<\(bool\)1, \(bool\)1, \(bool\)1, \(bool\)0>' -s 10 -c 3 --csv \
     --log-file $O/dram_g$g.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
echo done
