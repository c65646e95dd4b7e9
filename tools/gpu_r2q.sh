#!/bin/bash
O=gpurun_out/R2q
mkdir -p $O
export PYTHONUNBUFFERED=1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
tail -1 $O/smoke.log
timeout 900 python tools/env_ab.py qft:7,qft:8 "base:" > $O/mid.txt 2>&1; cat $O/mid.txt
