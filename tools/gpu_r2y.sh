#!/bin/bash
O=gpurun_out/R2y
mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_full_unitary_gpu.py -q -x -p no:cacheprovider -k "not qft14" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 1200 python tools/env_ab.py qft:10,qft:11,qft:12,deutsch-jozsa:11,qft:12 "dense:QSB_MATB_DENSE=1" "skip:" > $O/k1t_skip_ab.txt 2>&1
cat $O/k1t_skip_ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:expand_t -c 10 --csv --log-file $O/k1t.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu exit $?"
