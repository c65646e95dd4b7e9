"""K2m (one cluster launch per chain) against the K2 GEMM chain (QSB_NO_MID=1,
N = 128 / 256) or the K2s row-resident kernel (QSB_SMALL_CLASSIC=1, N <= 64):
device time per circuit, CUDA events around plan execution."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

sim = B200UnitarySimulator()
s = torch.cuda.Stream()  # a real stream: stream 0 would make the plan use its own
torch.cuda.set_stream(s)
for spec in sys.argv[1:] or ["qft:3", "qft:4", "qft:5", "qft:6", "entangle:6", "deutsch-jozsa:6", "qft:7", "qft:8", "entangle:7", "entangle:8", "deutsch-jozsa:7", "deutsch-jozsa:8"]:
    name, n = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    out = []
    base = "k2s" if int(n) <= 6 else "k2"
    for mode in (base, "k2m"):
        os.environ.pop("QSB_NO_MID", None)
        os.environ.pop("QSB_SMALL_CLASSIC", None)
        if mode == "k2":
            os.environ["QSB_NO_MID"] = "1"
        elif mode == "k2s":
            os.environ["QSB_SMALL_CLASSIC"] = "1"
        plan = sim.plan(c, reg)
        for _ in range(3):
            plan.execute(s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(s)
        for _ in range(reps):
            plan.execute(s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        out.append((mode, e0.elapsed_time(e1) / reps, plan.info.n_launches, plan.info.n_gemms))
        plan.close()
    print(spec, "  ".join(f"{m}: {t * 1e3:.1f} us ({nl} launches, {g} gemms)" for m, t, nl, g in out),
          f"speed-up {out[0][1] / out[1][1]:.2f}x", flush=True)
