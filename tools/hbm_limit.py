"""Dense timings up to the HBM limit of one B200 (BASELINE
north star "timed from 4 qubits up to the largest size that fits in HBM").

  * QFT-15 (32768^2 complex doubles, 141 GEMMs): the whole unitary on one GPU;
  * QFT-16 (65536^2, 160 GEMMs): rows [0, N/8) — one rank's share of the 8-GPU
    row-block decomposition (every rank's work is identical and independent) —
    and the full-size plan's guard / memory decision.

One plan execution each, CUDA events on the launching stream (no warm-up: at
these sizes one circuit is minutes and the first execution's host work is
negligible next to it). psi is checked against the DFT's column 0 (1/sqrt(N)).

    python tools/hbm_limit.py [qft-15] [qft-16/8]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import B200UnitarySimulator  # noqa: E402

PEAK = 37.1


def run(n, shards):
    N = 1 << n
    rows = N // shards
    c, reg = q.make_named_circuit("qft", n)
    flat = native.flatten(c, reg)
    sim = B200UnitarySimulator(device=0)
    s = torch.cuda.Stream()
    t0 = time.perf_counter()
    plan = sim.plan(flat, None, 0, rows)
    plan_s = time.perf_counter() - t0
    info = plan.info
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    plan.execute(s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    re = torch.empty(rows, dtype=torch.float64, device="cuda")
    im = torch.empty(rows, dtype=torch.float64, device="cuda")
    plan.copy_state(re.data_ptr(), im.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    want = 1.0 / np.sqrt(N)
    err = float(torch.sqrt(((re - want) ** 2 + im ** 2).sum() / (rows * want * want)).item())
    out = {"workload": f"qft-{n}", "rows": rows, "of_rows": N, "shards": shards, "ms": ms,
           "gemms": info.n_gemms, "v_planes": info.v_planes, "tile": native.TILE_NAMES.get(info.gemm_tile),
           "credited_tflops": info.gemm_flops / (ms * 1e-3) / 1e12,
           "hw_tflops": info.gemm_hw_flops / (ms * 1e-3) / 1e12,
           "hw_frac": info.gemm_hw_flops / (ms * 1e-3) / 1e12 / PEAK,
           "psi_rel_err_vs_dft_col0": err, "plan_s": plan_s,
           "guard": sim.qubit_guard(), "hbm_footprint_full_GB": native.lib().qsb_hbm_footprint(n) / 1e9}
    plan.close()
    sim.close()
    return out


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["qft-15", "qft-16/8"]:
        w, _, sh = arg.partition("/")
        print(json.dumps(run(int(w.split("-")[1]), int(sh or 1))), flush=True)
