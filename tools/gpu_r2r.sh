#!/bin/bash
O=gpurun_out/R2r
mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -k "materiali or zero_tiles or stream or split" -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 900 python tools/env_ab.py qft:10,qft:11,qft:12,deutsch-jozsa:11 "dense:QSB_MATB_DENSE=1" "skip:" > $O/zeroskip_ab.txt 2>&1
cat $O/zeroskip_ab.txt
for v in dense skip; do
  if [ $v = dense ]; then export QSB_MATB_DENSE=1; else unset QSB_MATB_DENSE; fi
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
     --kernel-name-base demangled -k 'regex:zgemm_ws_kernel<\(bool\)1, \(bool\)1, \(bool\)1, \(bool\)0>' -s 10 -c 3 --csv \
     --log-file $O/dram_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
unset QSB_MATB_DENSE
echo done
