"""Pin bench.py's CPU-baseline model to full reference runs.

For each workload, time the UNMODIFIED reference's whole
UnitarySimulator::simulate_full_state ("unitary-parallel", run_bench's way of
timing a full call: bench.cpp:95-105) and the component model bench.py
extrapolates from (cpu_sample_circuit with allow_full=False), on the same
threads, and print one JSON line per workload with the model's error. Run on
the GPU box's host:

    QSB_REF_THREADS=14 python tools/cpu_pin.py qft-9 qft-10 qft-11 entangle-10 entangle-11 dj-10 dj-11

QSB_REF_THREADS (default: every core) is the reference's worker count, so the
pin can share the box with GPU work on the remaining cores.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

NAMES = {"qft": "qft", "entangle": "entangle", "dj": "deutsch-jozsa"}


def main(argv):
    reps = int(os.environ.get("PIN_REPEATS", "1"))
    for w in argv:
        short, n = w.rsplit("-", 1)
        name, n = NAMES[short], int(n)
        t0 = time.perf_counter()
        model = bench.cpu_sample_circuit(name, n, 2, allow_full=False)
        t1 = time.perf_counter()
        full = [bench.cpu_full_run(name, n) for _ in range(reps)]
        wall = time.perf_counter() - t1
        meas = min(full)
        line = {"workload": f"{short}-{n}", "threads": bench.ref_cores(), "host_cores": os.cpu_count(),
                "measured_ms": meas, "measured_runs_ms": full, "model_ms": model["value"],
                "model_error": model["value"] / meas - 1.0, "model_components_s": model.get("components_s"),
                "model_sample_wall_s": t1 - t0, "full_wall_s": wall}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
