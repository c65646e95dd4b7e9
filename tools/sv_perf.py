"""State-vector engine probe: times fsv (mode state) and structured-unitary
plans of named circuits with CUDA events; prints passes and achieved HBM GB/s."""
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import B200FsvSimulator, B200StructuredUnitarySimulator  # noqa: E402

fsv = B200FsvSimulator()
st = B200StructuredUnitarySimulator()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
for spec in sys.argv[1:] or ["fsv:qft:24", "fsv:qft:22", "fsv:entangle:24", "fsv:deutsch-jozsa:11", "u:qft:12", "u:qft:14", "u:entangle:14", "u:deutsch-jozsa:11", "u:qft:16"]:
    mode, name, n = spec.split(":")
    c, reg = q.make_named_circuit(name, int(n))
    flat = native.flatten(c, reg)
    plan = (fsv if mode == "fsv" else st).plan(flat)
    info = plan.info
    for _ in range(2):
        plan.execute(stream.cuda_stream)
    torch.cuda.synchronize()
    reps = 5
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        plan.execute(stream.cuda_stream)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{spec}: ops={info.n_ops} passes={info.n_passes} fnpasses={info.n_function_passes} "
          f"slab={info.slab_bits} maxT={info.max_batch_targets} {ms:.3f} ms "
          f"-> {info.bytes_per_run / (ms * 1e-3) / 1e9:.0f} GB/s (bytes/run {info.bytes_per_run / 1e9:.2f} GB)",
          flush=True)
    plan.close()
