#!/bin/bash
O=gpurun_out/R2m
mkdir -p $O
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_host_cache_gpu.py -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --workload entangle-10 > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err; echo "torchrun exit $?"
tail -1 $O/bench_torchrun1.json | cut -c1-300
