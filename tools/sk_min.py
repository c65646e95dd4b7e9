"""Minimal stream-K determinism cases: short chains, many repetitions."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.circuit import Circuit, GateType  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402


def make(kind, n):
    c = Circuit(n)
    for k in range(n):
        c.h(k)
    if kind == "hh":
        for k in range(n):
            c.h(k)
    elif kind == "hr":
        for k in range(n):
            c.add_gate(GateType.r(0.1 + k), k)
    elif kind == "hcr":
        for k in range(n - 1):
            c.add_control_gate(GateType.r(0.3 + k), k, k + 1)
    elif kind == "hhh":
        for _ in range(2):
            for k in range(n):
                c.h(k)
    return c


sim = B200UnitarySimulator()
reps = int(os.environ.get("SK_REPS", "50"))
for spec in sys.argv[1:]:
    kind, n, tile = spec.split(":")
    n = int(n)
    c = make(kind, n)
    flat = native.flatten(c, q.GateRegistry())
    os.environ["QSB_TILE"] = tile
    os.environ["QSB_STREAMK"] = "0"
    ref = sim.build_unitary(flat)
    os.environ["QSB_STREAMK"] = "1"
    p = sim.plan(flat)
    info = p.info
    p.close()
    nbad = 0
    for r in range(reps):
        a = sim.build_unitary(flat)
        d = np.abs(a[0] - ref[0]) + np.abs(a[1] - ref[1])
        bad = np.argwhere(d > 1e-12)
        if len(bad):
            nbad += 1
            if nbad <= 3:
                tiles = sorted({(int(i) // 64, int(j) // 64) for i, j in bad})
                print(spec, "run", r, "ndiff", len(bad), "tiles", tiles[:6], flush=True)
                for i, j in bad[:6]:
                    print("   ", int(i), int(j), a[0][i, j], ref[0][i, j], a[1][i, j], ref[1][i, j])
    print(spec, "gemms", info.n_gemms, "splits", info.gemm_splits, "bad runs", nbad, "of", reps, flush=True)
