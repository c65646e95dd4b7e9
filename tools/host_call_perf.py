"""Host-API call latency (qsb_simulate_full_state with host buffers) of the dense
backend, cold (QSB_FLAG_NO_PLAN_CACHE: compile + upload every call) and with the
handle's plan cache (run_bench's repeated calls), next to the device time of the
plan's execution. Also times the fsv and structured backends' host calls.

    python tools/host_call_perf.py [qft:4,deutsch-jozsa:11,...]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import (B200FsvSimulator, B200StructuredUnitarySimulator,  # noqa: E402
                                             B200UnitarySimulator)

specs = (sys.argv[1] if len(sys.argv) > 1 else
         "qft:4,qft:6,entangle:8,deutsch-jozsa:8,deutsch-jozsa:10,deutsch-jozsa:11,entangle:10,qft:10").split(",")
L = native.lib()


def per_call(handle, fn, flat, N, budget_s=2.0):
    re, im = np.empty(N), np.empty(N)
    native.check(fn(handle, flat.ptr, native.dptr(re), native.dptr(im)))
    t0 = time.perf_counter()
    native.check(fn(handle, flat.ptr, native.dptr(re), native.dptr(im)))
    one = time.perf_counter() - t0
    reps = max(3, min(200, int(budget_s / max(one, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(reps):
        native.check(fn(handle, flat.ptr, native.dptr(re), native.dptr(im)))
    return (time.perf_counter() - t0) / reps * 1e6


cold = B200UnitarySimulator(flags=native.FLAG_NO_PLAN_CACHE)
warm = B200UnitarySimulator()
s = torch.cuda.Stream()
for spec in specs:
    name, n = spec.split(":")
    n = int(n)
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    N = 1 << n
    t_cold = per_call(cold._h, L.qsb_simulate_full_state, flat, N)
    t_warm = per_call(warm._h, L.qsb_simulate_full_state, flat, N)
    plan = warm.plan(flat)
    plan.execute(s.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record(s)
    for _ in range(reps):
        plan.execute(s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    dev = a.elapsed_time(b) / reps * 1e3
    plan.close()
    print(f"dense {name}-{n}: host call cold {t_cold:.1f} us, plan-cached {t_warm:.1f} us, "
          f"device {dev:.1f} us per execution ({t_warm / dev:.2f}x device cached, {t_cold / dev:.2f}x cold)",
          flush=True)
cold.close()
warm.close()
for cls, fn in ((B200FsvSimulator, L.qsb_fsv_simulate_full_state),
                (B200StructuredUnitarySimulator, L.qsb_structured_simulate_full_state)):
    sim = cls()
    for spec in specs[:3]:
        name, n = spec.split(":")
        c, reg = q.make_named_circuit(name, int(n))
        flat = native.flatten(c, reg)
        print(f"{cls.__name__} {name}-{n}: {per_call(sim._h, fn, flat, 1 << int(n)):.1f} us per host call", flush=True)
    sim.close()
