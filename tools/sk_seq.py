"""Stream-K determinism in the test-suite order (one simulator, cached buffers)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

sim = B200UnitarySimulator()
os.environ.setdefault("QSB_STREAMK", "1")
for spec in sys.argv[1:]:
    name, n, tile = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    flat = native.flatten(c, reg)
    os.environ["QSB_TILE"] = tile
    p = sim.plan(flat)
    p.close()
    a = sim.build_unitary(flat)
    for r in range(1, int(os.environ.get("SK_REPS", "5"))):
        b = sim.build_unitary(flat)
        d = np.abs(a[0] - b[0]) + np.abs(a[1] - b[1])
        bad = np.argwhere(d > 0)
        tiles = sorted({(int(i) // 64, int(j) // 64) for i, j in bad[:100000]})
        if len(bad) or r % 20 == 0:
            print(spec, "run", r, "ndiff", len(bad), "max", float(d.max()), "tiles", len(tiles), tiles[:8], flush=True)
