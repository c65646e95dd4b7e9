"""Pin bench.py's CPU-baseline model to full reference runs.

For each workload, time the UNMODIFIED reference's whole
UnitarySimulator::simulate_full_state ("unitary-parallel", all host cores,
run_bench's method: bench.cpp:95-105 — warm-up, then timed full calls) and
the component model bench.py extrapolates from (cpu_sample_circuit), and print
one JSON line per workload with the model error. Run on the GPU box's host:

    python tools/cpu_pin.py qft-9 qft-10 qft-11 entangle-10 entangle-11 dj-10 dj-11
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402

NAMES = {"qft": "qft", "entangle": "entangle", "dj": "deutsch-jozsa"}


def main(argv):
    reps = int(os.environ.get("PIN_REPEATS", "1"))
    ref = oracle.Reference()
    for w in argv:
        short, n = w.rsplit("-", 1)
        name, n = NAMES[short], int(n)
        prog = ref.named(name, n)
        ref.L.refsh_set_worker_count(0)  # QSIM_THREADS unset: all host cores
        t0 = time.perf_counter()
        full = [ref.L.refsh_time_simulate(prog.h, b"unitary-parallel", n) for _ in range(reps)]
        wall = time.perf_counter() - t0
        model = bench.cpu_sample_circuit(name, n, 1)
        meas = min(full) * 1e3
        line = {"workload": f"{short}-{n}", "cores": os.cpu_count(), "measured_ms": meas,
                "measured_runs_ms": [t * 1e3 for t in full], "model_ms": model["value"],
                "model_error": model["value"] / meas - 1.0, "model_components_s": model.get("components_s"),
                "wall_s": wall}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
