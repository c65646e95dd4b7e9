"""Time per circuit vs qubits (the paper's headline sweep, BASELINE.json metric)
for QFT, Fully Entangled and Deutsch-Jozsa circuits on one B200:

  * dense   — Algorithm 1 (the drop-in unitary-b200 path): device time of one
              plan execution (CUDA events), credited TFLOP/s of the GEMM chain;
  * struct  — unitary-structured-b200 (U[:,c] = fsv(e_c)), device time;
  * fsv     — fsv-b200, device time;
  * cpu     — the reference library (oracle/_ref) on this host's cores: measured
              directly for n <= 8, extrapolated from bounded component samples
              above (bench.cpu_sample), empty when oracle/_ref is absent.

    python tools/sweep.py [--max-dense 14] [--max-sv 16] [--cpu-max 12] [--out profiles/sweep.md]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402
from paper_2305_14398_b200.simulator import (B200FsvSimulator, B200StructuredUnitarySimulator,  # noqa: E402
                                             B200UnitarySimulator)


def time_plan(plan, stream, reps):
    plan.execute(stream.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        plan.execute(stream.cuda_stream)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def write_table(path, rows):
    with open(path, "w") as f:
        f.write("# Time per circuit vs qubits on one B200 (tools/sweep.py)\n\n")
        f.write("Device time per circuit (CUDA events, one plan execution; inputs resident). "
                "dense = Algorithm 1 (unitary-b200, FP64 tensor cores): hw frac = the FLOPs the DMMAs execute "
                "(6N^3 3M / 4N^3 real layer per GEMM) over the measured 37.1 TF/s DMMA peak; TFLOP/s credited "
                "8N^3 per GEMM (ZGEMM convention); struct = unitary-structured-b200; fsv = fsv-b200; cpu = the "
                f"reference library on the host's {os.cpu_count()} cores: the whole circuit run and timed where "
                "the component model predicts <= 300 s (m), else the model extrapolated from bounded samples (x; "
                "its error against full runs: profiles/cpu_pin.json).\n\n")
        f.write("| circuit | n | GEMMs | dense ms | dense hw frac | dense TFLOP/s (credited) | struct ms | fsv ms | "
                "cpu ms | dense speed-up vs cpu |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|\n")

        def fmt(v, p=3):
            return "" if v is None else (f"{v:.{p}g}" if isinstance(v, float) else str(v))

        for r in rows:
            sp = (r["cpu_ms"] / r["dense_ms"]) if r.get("cpu_ms") and r.get("dense_ms") else None
            cpu = fmt(r.get('cpu_ms'), 4)
            if cpu:
                cpu += " (m)" if r.get("cpu_full") else " (x)"
            f.write(f"| {r['circuit']} | {r['n']} | {fmt(r.get('gemms'))} | {fmt(r.get('dense_ms'), 4)} | "
                    f"{fmt(r.get('dense_hw_frac'))} | {fmt(r.get('dense_tflops'))} | {fmt(r.get('struct_ms'), 4)} | "
                    f"{fmt(r.get('fsv_ms'), 4)} | {cpu} | {fmt(sp)} |\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-dense", type=int, default=14)
    ap.add_argument("--max-sv", type=int, default=16)
    ap.add_argument("--cpu-max", type=int, default=12)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep.md"))
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dense, st, fsv = B200UnitarySimulator(), B200StructuredUnitarySimulator(), B200FsvSimulator()
    # DJ oracle registration (is_unitary, O(8^n)) on the GPU instead of the host
    from paper_2305_14398_b200 import circuit
    from paper_2305_14398_b200.simulator import gpu_unitarity_check

    circuit.set_unitarity_check(gpu_unitarity_check(dense))
    rows = []
    for name, key in [("qft", "qft"), ("entangle", "entangle"), ("deutsch-jozsa", "dj")]:  # noqa: B007
        for n in range(4, max(args.max_dense, args.max_sv) + 1):
            if name == "deutsch-jozsa" and n > 12:
                continue  # the registered oracle is a dense 2^n x 2^n matrix on the host
            c, reg = q.make_named_circuit(name, n)
            flat = native.flatten(c, reg)
            row = {"circuit": key, "n": n}
            if n <= args.max_dense:
                p = dense.plan(flat)
                ms = time_plan(p, stream, 1 if n >= 13 else 3)
                row["dense_ms"] = ms
                row["dense_tflops"] = p.info.gemm_flops / (ms * 1e-3) / 1e12 if p.info.n_gemms else None
                row["dense_hw_frac"] = (p.info.gemm_hw_flops / (ms * 1e-3) / 1e12 / bench.FP64_DMMA_PEAK_TFLOPS
                                        if p.info.n_gemms else None)
                row["gemms"] = p.info.n_gemms
                p.close()
            if n <= args.max_sv:
                p = st.plan(flat)
                row["struct_ms"] = time_plan(p, stream, 3)
                p.close()
                p = fsv.plan(flat)
                row["fsv_ms"] = time_plan(p, stream, 3)
                p.close()
            # the reference registers a DJ oracle with its O(8^n) host is_unitary: bounded at n = 10
            if n <= (min(args.cpu_max, 10) if key == "dj" else args.cpu_max) and bench.oracle_available():
                t0 = time.time()
                # a torch-free process, like the reference's own; the whole circuit is run where
                # the model predicts up to 5 minutes (QFT-11 included), the model above
                cb = bench.cpu_circuit_subprocess(name, n, full_limit_s=300.0)
                row["cpu_ms"] = cb["value"]
                row["cpu_full"] = cb.get("full_run", n <= 8)
                row["cpu_wall_s"] = time.time() - t0
            rows.append(row)
            print(row, flush=True)
            write_table(args.out, rows)  # after every row: a cut-off run still leaves its table
    print("wrote", args.out)


if __name__ == "__main__":
    main()
