import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2305_14398_b200 as q
from paper_2305_14398_b200 import native
from paper_2305_14398_b200.simulator import B200UnitarySimulator
sim = B200UnitarySimulator()
for spec in sys.argv[1:]:
    name, n = spec.split(":"); n = int(n)
    c, reg = q.make_named_circuit(name, n)
    out = sim.simulate_full_state(c, reg)
    out = sim.simulate_full_state(c, reg)
