#!/bin/bash
O=gpurun_out/R2u
mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 1200 python tools/env_ab.py qft:12,qft:11,qft:10,entangle:10,entangle:11,deutsch-jozsa:11,qft:12 "dense:QSB_MATB_DENSE=1" "skip:" > $O/zeroskip_ab.txt 2>&1
cat $O/zeroskip_ab.txt
for v in dense skip; do
  if [ $v = dense ]; then export QSB_MATB_DENSE=1; else unset QSB_MATB_DENSE; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
     --kernel-name-base demangled -k 'regex:zgemm_ws_kernel' -s 20 -c 8 --csv \
     --log-file $O/k2_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
echo done
