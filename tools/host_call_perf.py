import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2305_14398_b200 as q
from paper_2305_14398_b200 import native
from paper_2305_14398_b200.simulator import B200UnitarySimulator, B200FsvSimulator, B200StructuredUnitarySimulator
for cls in (B200UnitarySimulator, B200StructuredUnitarySimulator, B200FsvSimulator):
    sim = cls()
    for name, n in [("qft", 4), ("qft", 5), ("entangle", 6), ("qft", 8)]:
        c, reg = q.make_named_circuit(name, n)
        flat = native.flatten(c, reg)
        N = 1 << n
        re = np.empty(N); im = np.empty(N)
        fn = {B200UnitarySimulator: native.lib().qsb_simulate_full_state,
              B200FsvSimulator: native.lib().qsb_fsv_simulate_full_state,
              B200StructuredUnitarySimulator: native.lib().qsb_structured_simulate_full_state}[cls]
        for _ in range(20): native.check(fn(sim._h, flat.ptr, native.dptr(re), native.dptr(im)))
        t0 = time.perf_counter()
        for _ in range(200): native.check(fn(sim._h, flat.ptr, native.dptr(re), native.dptr(im)))
        dt = (time.perf_counter() - t0) / 200 * 1e3
        print(f"{cls.__name__} {name}-{n}: {dt*1000:.1f} us per host call")
    sim.close()
