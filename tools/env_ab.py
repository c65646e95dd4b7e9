"""A/B of plan-time switches: device time per circuit (CUDA events around plan
execution on a real stream) for each circuit under each environment variant.

    python tools/env_ab.py qft:9,qft:10 "base:" "mat0:QSB_MATERIALIZE=0" "sk1:QSB_STREAMK=1"
"""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

specs = sys.argv[1].split(",")
variants = []
for v in sys.argv[2:] or ["base:"]:
    name, _, env = v.partition(":")
    variants.append((name, dict(kv.split("=", 1) for kv in env.split(",") if kv)))
sim = B200UnitarySimulator()
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
keys = {k for _, e in variants for k in e}
for spec in specs:
    name, n = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    res = []
    for vname, env in variants:
        for k in keys:
            os.environ.pop(k, None)
        os.environ.update(env)
        plan = sim.plan(c, reg)
        for _ in range(3):
            plan.execute(s.cuda_stream)
        torch.cuda.synchronize()
        reps = max(3, min(50, int(2000 / max(1, 4 ** (int(n) - 8)))))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            plan.execute(s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        res.append(f"{vname} {e0.elapsed_time(e1) / reps:.4f} ms (tile {plan.info.gemm_tile}, splits {plan.info.gemm_splits}, launches {plan.info.n_launches})")
        plan.close()
    print(spec, " | ".join(res), flush=True)
