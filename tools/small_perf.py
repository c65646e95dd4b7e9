"""Device time per circuit for small plans (one launch), averaged over many
back-to-back executions on one stream, and host time per full C-ABI call."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

sim = B200UnitarySimulator()
stream = torch.cuda.Stream()
for spec in sys.argv[1:] or ["qft:4", "qft:5", "qft:6", "entangle:4"]:
    name, n = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    flat = native.flatten(c, reg)
    p = sim.plan(flat)
    for _ in range(3):
        p.execute(stream.cuda_stream)
    torch.cuda.synchronize()
    reps = 200
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        p.execute(stream.cuda_stream)
    b.record(stream)
    torch.cuda.synchronize()
    dev = a.elapsed_time(b) / reps * 1e3
    info = p.info
    p.close()
    ts = []
    for _ in range(50):
        t0 = time.perf_counter()
        sim.simulate_full_state(c, reg)
        ts.append(time.perf_counter() - t0)
    print(f"{spec}: launches {info.n_launches} gemm_tile {info.gemm_tile}: device {dev:.2f} us per execution "
          f"(back to back), host call median {1e6 * np.median(ts):.1f} us min {1e6 * min(ts):.1f} us", flush=True)
