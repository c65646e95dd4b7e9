"""Quick K2 throughput probe: plans a named circuit, runs it with phase timing."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

import os
from paper_2305_14398_b200 import native as _n
sim = B200UnitarySimulator(gemm_mode={'4m': _n.GEMM_4M, '3m': _n.GEMM_3M}.get(os.environ.get('QSB_GEMM', ''), _n.GEMM_AUTO),
                           flags=int(os.environ.get('QSB_FLAGS', '0')))
for spec in sys.argv[1:] or ["qft:10", "qft:12"]:
    name, n = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    plan = sim.plan(c, reg)
    plan.set_timing(True)
    plan.execute(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    t0 = time.time()
    plan.execute(torch.cuda.current_stream().cuda_stream)
    total, gemm, mean = plan.last_timing()
    info = plan.info
    tf = info.gemm_flops / (gemm * 1e-3) / 1e12 if gemm > 0 else 0
    print(f"{spec}: gemms={info.n_gemms} total={total:.3f} ms gemm={gemm:.3f} ms mean={mean:.4f} ms "
          f"-> {tf:.2f} TFLOP/s (8N^3 credited), wall {time.time() - t0:.3f}s", flush=True)
    plan.close()
