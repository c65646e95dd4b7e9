"""Host-side phase timing of the dense path for one circuit: plan creation,
execute (graph / no graph), synchronisation, destruction."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

sim = B200UnitarySimulator()
for spec in sys.argv[1:] or ["qft:8", "qft:5", "entangle:10"]:
    name, n = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    flat = native.flatten(c, reg)
    for _ in range(3):
        t0 = time.perf_counter(); p = sim.plan(flat); t1 = time.perf_counter()
        p.execute(); t2 = time.perf_counter(); torch.cuda.synchronize(); t3 = time.perf_counter()
        p.execute(); t4 = time.perf_counter(); torch.cuda.synchronize(); t5 = time.perf_counter()
        p.close(); t6 = time.perf_counter()
    print(f"{spec}: plan {1e6*(t1-t0):.0f} us, first execute (graph capture) {1e6*(t2-t1):.0f} + sync {1e6*(t3-t2):.0f} us, "
          f"graph execute {1e6*(t4-t3):.0f} + sync {1e6*(t5-t4):.0f} us, close {1e6*(t6-t5):.0f} us, "
          f"tile {p.info.gemm_tile} splits {p.info.gemm_splits}", flush=True)
