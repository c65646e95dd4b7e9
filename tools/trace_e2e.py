"""Host phases of the C-ABI call (QSB_TRACE=1 prints plan / enqueue / wait+copy)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

sim = B200UnitarySimulator()
for spec in sys.argv[1:] or ["qft:12"]:
    name, n = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    flat = native.flatten(c, reg)
    N = 1 << int(n)
    re = np.empty(N)
    im = np.empty(N)
    reps = 3 if int(n) >= 11 else 20
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        native.check(native.lib().qsb_simulate_full_state(sim._h, flat.ptr, native.dptr(re), native.dptr(im)))
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{spec}: call ms median {np.median(ts):.4f} min {min(ts):.4f}", flush=True)
