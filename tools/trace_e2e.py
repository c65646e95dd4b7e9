import sys, time; sys.path.insert(0, ".")
import numpy as np
import paper_2305_14398_b200 as q
from paper_2305_14398_b200 import native
from paper_2305_14398_b200.simulator import B200UnitarySimulator
sim = B200UnitarySimulator()
c, reg = q.make_named_circuit("qft", 12)
flat = native.flatten(c, reg)
N = 4096
re = np.empty(N); im = np.empty(N)
for _ in range(3):
    t0 = time.perf_counter()
    native.check(native.lib().qsb_simulate_full_state(sim._h, flat.ptr, native.dptr(re), native.dptr(im)))
    print("call ms", (time.perf_counter() - t0) * 1e3, flush=True)
