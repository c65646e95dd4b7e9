"""Benchmark: unitary-simulation time per circuit on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload qft-12] [--impl ours|reference]

One step = one full circuit through the hot path (Algorithm 1: K1 expansion of
the first operator, one K2 DMMA GEMM per further layer, K3 application of
psi0). ``value`` is milliseconds per circuit with the circuit already resident
on the device (CUDA events on the launching stream, max over ranks); ``e2e`` is
the same circuit through the public C ABI with host buffers (descriptor H2D and
psi D2H inside the timed region). For N > 1 (torchrun, one process per GPU) the
unitary is sharded by row blocks; each rank computes its rows with no
communication and psi is all-gathered with NCCL.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref: the unmodified reference library compiled from its sources) on
this host's cores over a bounded sample of the same workload and extrapolates
the per-circuit time (the sample is stated in the JSON line).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "unitary-sim time (ms) per circuit vs qubits; FP64 TC TFLOPS %peak @1/2/4/8 GPU"
# FP64 tensor (DMMA) peak measured on this pool's B200: register-only
# mma.sync.m8n8k4.f64 loop over 148 SMs (tools/microbench/fp64_peak.cu,
# profiles/r01_fp64_peak.txt). MEASURED_PEAKS.json carries no FP64 figure.
FP64_DMMA_PEAK_TFLOPS = 37.1
WORKLOADS = {
    # name: (circuit, qubits) — BASELINE.json configs
    "qft-4": ("qft", 4),
    "entangle-10": ("entangle", 10),
    "dj-11": ("deutsch-jozsa", 11),
    "qft-12": ("qft", 12),
    "qft-14": ("qft", 14),
    "qft-16": ("qft", 16),
    # state-vector sizes (--backend fsv only)
    "qft-24": ("qft", 24),
    "entangle-24": ("entangle", 24),
}
DEFAULT_WORKLOAD = "qft-12"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gemm-mode", default="auto", choices=["auto", "4m", "3m"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU check of the multi-rank plumbing: the same launch (re-exec under torchrun for "
                         "--gpus N), rank-count checks, row_shard and the psi all-gather over gloo, with every "
                         "rank contributing index-valued rows instead of computed ones (no kernels)")
    ap.add_argument("--virtual-ranks", type=int, default=1,
                    help="with one GPU: time only rank 0's row block of a G-way shard (the work each of G "
                         "GPUs does, with no communication but the final psi all-gather) and report it "
                         "as a projection next to the measured line")
    ap.add_argument("--backend", default="dense", choices=["dense", "structured", "fsv"],
                    help="dense: Algorithm 1 on the FP64 tensor cores (the headline); structured: U built by "
                         "the state-vector engine (U[:,c] = fsv(e_c)); fsv: the full-state-vector backend")
    return ap.parse_args()


def mode_of(args) -> int:
    from paper_2305_14398_b200 import native

    return {"auto": native.GEMM_AUTO, "4m": native.GEMM_4M, "3m": native.GEMM_3M}[args.gemm_mode]


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------- CPU baseline

def oracle_available() -> bool:
    import oracle

    return oracle.reference_available()


def cpu_sample(workload: str, repeats: int = 2):
    """Reference CPU time of a named BASELINE workload (cpu_sample_circuit)."""
    name, n = WORKLOADS[workload]
    return cpu_sample_circuit(name, n, repeats)


FULL_RUN_LIMIT_S = 30.0  # model-predicted reference time under which the whole circuit is run instead
# reference worker threads (QSIM_THREADS semantics): 0 = every host core
REF_THREADS = int(os.environ.get("QSB_REF_THREADS", "0") or 0)


def ref_cores() -> int:
    return REF_THREADS if REF_THREADS > 0 else (os.cpu_count() or 1)


def cpu_full_run(name: str, n: int) -> float:
    """ms of one whole reference UnitarySimulator::simulate_full_state ("unitary-parallel")."""
    import oracle

    ref = oracle.Reference()
    prog = ref.named(name, n)
    ref.L.refsh_set_worker_count(REF_THREADS)
    return ref.L.refsh_time_simulate(prog.h, b"unitary-parallel", n) * 1e3


def cpu_sample_circuit(name: str, n: int, repeats: int = 2, allow_full: bool = True,
                       full_limit_s: float = FULL_RUN_LIMIT_S):
    """Time the reference CPU path (oracle/_ref: the unmodified reference library)
    on this host's cores for one circuit. When the component model below predicts
    at most FULL_RUN_LIMIT_S, the whole UnitarySimulator::simulate_full_state
    ("unitary-parallel", all cores) is run and timed — a measurement. Otherwise a
    bounded sample of the reference's own components is timed and extrapolated
    (SURVEY.md 8(d)):
      T = (steps + extra) * fold + steps * GEMM_par(N) + extra * GEMM_ser(N)
    per step: step_unitary folds every layer (unitary_backend.cpp:141-154) and
    multiplies a multi-layer step's layers serially (:151), then one parallel
    accumulate matmul (:211). GEMM_* come from the reference's own matmul on row
    slabs of N/4 (parallel) and N/16 (serial) rows (linalg.cpp:72-87 accepts
    rectangular shapes; smaller slabs mis-predict by up to 2x: thread start-up
    and cache effects), fold from step_unitary of a single-layer step; each
    component is the minimum of `repeats` timings. The model's error against full
    runs on the GPU box's host is committed in profiles/cpu_pin.json."""
    import oracle
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    workload = f"{name}-{n}"
    N = 1 << n
    cores = ref_cores()
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    orc = oracle.Oracle()
    n_steps = len(flat.step_offsets) - 1
    layers = [orc.step_layers(flat, s)[0] for s in range(n_steps)]
    extra = sum(l - 1 for l in layers)
    single = next(s for s in range(n_steps) if layers[s] == 1)
    if oracle.reference_available():
        ref = oracle.Reference()
        kind = "reference"
        prog = ref.named(name, n)
        if n <= 8:
            # small sizes: time the whole reference simulate_full_state directly
            t_full = []
            for _ in range(max(1, repeats)):
                ref.L.refsh_set_worker_count(REF_THREADS)
                t_full.append(ref.L.refsh_time_simulate(prog.h, b"unitary-parallel", n))
            t_par = min(t_full)
            ref.L.refsh_set_worker_count(1)
            t_ser = min(ref.L.refsh_time_simulate(prog.h, b"unitary", n) for _ in range(max(1, repeats)))
            ref.L.refsh_set_worker_count(REF_THREADS)
            best = min(t_par, t_ser)
            return {"value": best * 1e3, "unit": "ms", "cores": cores, "kind": kind,
                    "sample": f"full reference UnitarySimulator::simulate_full_state of {workload} "
                              f"(best of unitary / unitary-parallel, {repeats} run(s))"}
        rows_par = max(N // 4, 64)
        rows_ser = max(N // 16, 8)
        ref.L.refsh_set_worker_count(REF_THREADS)  # 0 = QSIM_THREADS unset: all host cores
        fold = min(ref.L.refsh_time_step_unitary(prog.h, single) for _ in range(max(1, repeats)))
        gemm_par = min(ref.L.refsh_time_matmul(rows_par, N, 1) for _ in range(max(1, repeats))) * N / rows_par
        # the serial layer product streams a 16 N^2-byte operand once per row on one thread:
        # memory-bound and the noisiest component on a shared (KVM) host, so one more sample
        ser_samples = ([ref.L.refsh_time_matmul(rows_ser, N, 0) * N / rows_ser for _ in range(max(1, repeats) + 1)]
                       if extra else [])
        gemm_ser = min(ser_samples) if ser_samples else 0.0
        total = (n_steps + extra) * fold + n_steps * gemm_par + extra * gemm_ser
        comps = {"fold": fold, "gemm_parallel": gemm_par, "gemm_serial": gemm_ser, "steps": n_steps,
                 "extra_layers": extra, "model_s": total, "gemm_serial_samples": ser_samples}
        if allow_full and total <= full_limit_s:
            return {"value": cpu_full_run(name, n), "unit": "ms", "cores": cores, "kind": kind,
                    "sample": f"full reference UnitarySimulator::simulate_full_state of {workload} "
                              f"(unitary-parallel, {cores} threads, one run)",
                    "components_s": comps, "full_run": True}
        sample = (f"reference step_unitary(single-layer step) + matmul({rows_par}x{N} . {N}x{N}, Parallel, "
                  f"{cores} threads) + matmul({rows_ser}x{N} . {N}x{N}, Serial), min of {repeats} ({repeats + 1} serial); "
                  f"extrapolated to {n_steps} steps + {extra} serial extra-layer GEMMs")
        return {"value": total * 1e3, "unit": "ms", "cores": cores, "kind": kind, "sample": sample,
                "components_s": comps, "full_run": False}
    kind = "port"
    orc.set_threads(cores)
    import numpy as np

    rows_par = max(N // 4, 64)
    rows_ser = max(N // 16, 8)
    a = np.random.default_rng(0).uniform(-1, 1, (rows_par, N)) * (1 + 0.5j)
    b = np.eye(N, dtype=complex)
    t0 = time.perf_counter()
    orc.layer_operator(flat, single, 0)
    fold = time.perf_counter() - t0
    t0 = time.perf_counter()
    orc.matmul(a, b)
    gemm_par = (time.perf_counter() - t0) * N / rows_par
    orc.set_threads(1)
    t0 = time.perf_counter()
    orc.matmul(a[:rows_ser], b)
    gemm_ser = (time.perf_counter() - t0) * N / rows_ser
    total = (n_steps + extra) * fold + n_steps * gemm_par + extra * gemm_ser
    return {"value": total * 1e3, "unit": "ms", "cores": cores, "kind": kind,
            "sample": "C oracle port (oracle/_ref absent): same components, extrapolated",
            "components_s": {"fold": fold, "gemm_parallel": gemm_par, "gemm_serial": gemm_ser,
                             "steps": n_steps, "extra_layers": extra, "model_s": total},
            "full_run": False}


def cpu_sample_subprocess(workload: str):
    """cpu_sample in a fresh process that never imports torch or touches the GPU (run
    before the bench initialises CUDA), like the reference's own process and the
    reference arm (--impl reference): in this container the reference's memory-bound
    serial product ran 1.26x slower after a torch import and matmul in the same process."""
    name, n = WORKLOADS[workload]
    return cpu_circuit_subprocess(name, n)


def cpu_circuit_subprocess(name: str, n: int, full_limit_s: float = FULL_RUN_LIMIT_S):
    code = ("import json, sys; sys.path.insert(0, %r); import bench; "
            "print(json.dumps(bench.cpu_sample_circuit(%r, %d, full_limit_s=%r)))" % (ROOT, name, n, full_limit_s))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=3600)
    if out.returncode != 0:
        raise RuntimeError(f"cpu baseline subprocess failed: {out.stderr[-2000:]}")
    return json.loads(out.stdout.strip().splitlines()[-1])


def model_validation(workload: str):
    """Measured error of the extrapolation model against full reference runs on a
    GPU box's host (tools/cpu_pin.py -> profiles/cpu_pin.json)."""
    path = os.path.join(ROOT, "profiles", "cpu_pin.json")
    try:
        with open(path) as f:
            pins = json.load(f)
    except Exception:
        return None
    rows = pins.get("runs", [])
    errs = [abs(r["model_error"]) for r in rows]
    first = {}
    for r in rows:  # the all-core runs on an idle box come first
        first.setdefault(r["workload"], round(r["model_error"], 4))
    out = {"source": "profiles/cpu_pin.json (tools/cpu_pin.py: full reference unitary-parallel "
                     "simulate_full_state vs the model, same host cores)",
           "workloads": first,
           "max_abs_error": max(errs) if errs else None,
           "model_used_when": f"the model predicts more than {FULL_RUN_LIMIT_S:.0f} s (QFT-11 and up); below "
                              "that the whole reference circuit is run and timed"}
    if workload in out["workloads"]:
        out["this_workload_error"] = out["workloads"][workload]
    return out


def run_reference(args):
    """The reference's own CPU path (oracle/_ref: the unmodified reference library)
    on this host's cores. n <= 8: the whole simulate_full_state, timed --steps
    times after --warmup runs. Larger n: one timed sample of the model's components
    (one single-layer step_unitary, a parallel and a serial matmul row slab),
    extrapolated ONCE to the circuit (extrapolated: true) — the model's error
    against full reference runs is stated from profiles/cpu_pin.json."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    name, n = WORKLOADS[args.workload]
    t0 = time.perf_counter()
    first = cpu_sample(args.workload)
    if n <= 8 or first.get("full_run"):
        # the whole circuit is affordable: time it --steps times (bounded to ~2 minutes)
        per = first["value"] / 1e3
        reps = max(1, min(args.steps, int(120.0 / max(per, 1e-6))))
        vals = [first["value"]] + [cpu_full_run(name, n) if first.get("full_run") else cpu_sample(args.workload)["value"]
                                   for _ in range(reps - 1)]
        value = statistics.mean(vals)
        runs = vals
        last = first
        extrapolated, timed = False, len(runs)
    else:
        last = first  # one timed sample of the components, extrapolated once
        value = last["value"]
        extrapolated, timed = True, 1
    wall = time.perf_counter() - t0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "deterministic circuit (synthetic)",
        "config": {"workload": args.workload, "circuit": name, "qubits": n, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "ms", "cores": last["cores"], "kind": last["kind"],
                         "sample": last["sample"], "extrapolated": extrapolated, "samples_timed": timed,
                         "model_validation": model_validation(args.workload) if extrapolated else None},
        "e2e": {"value": value, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated": extrapolated,
        "wall_s": wall,
    }
    if "components_s" in last:
        line["cpu_baseline"]["components_s"] = last["components_s"]
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, tag: str = "bench"):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{tag}_{device}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].isdigit():
                    rows.append(parts)
        note = None
        if not rows:
            # a timed region shorter than the 200 ms sampling period: one query right after it
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                for line in out.stdout.splitlines():
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= 9 and parts[1].isdigit():
                        rows.append(parts)
                note = "timed region shorter than the sampling period: sampled right after it"
            except Exception:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][2]), "reasons": reasons,
               "samples": len(rows)}
        powers = [float(r[3]) for r in rows if r[3] not in ("", "[N/A]")]
        if powers:
            out["power_w_max"] = max(powers)
        if note:
            out["note"] = note
        return out


# --------------------------------------------------------------- our arm

def run_ours(args, cpu_baseline=None):
    import torch
    import torch.distributed as dist

    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.sharding import gather_state, row_shard
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    rank, world, local = dist_env()
    if world != max(1, args.gpus):
        raise SystemExit(f"bench: --gpus {args.gpus} but {world} rank(s)")
    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench: rank {rank} has LOCAL_RANK {local} but only {torch.cuda.device_count()} GPU(s)")
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator ranks are visible in the log
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        if dist.get_world_size() != args.gpus:
            raise SystemExit(f"bench: process group has {dist.get_world_size()} ranks, --gpus {args.gpus}")
    torch.cuda.set_device(local)
    name, n = WORKLOADS[args.workload]
    N = 1 << n
    mode = mode_of(args)
    sim = B200UnitarySimulator(device=local, gemm_mode=mode)
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    vr = args.virtual_ranks if world == 1 and args.virtual_ranks > 1 else 1
    begin, count = row_shard(N, world * vr, rank)
    # A dedicated stream: every launch of the plan, the all-gather and the
    # timing events share it (the legacy default stream has handle 0).
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    s_ptr = stream.cuda_stream
    plan = sim.plan(flat, None, begin, count) if count > 0 else None
    psi_re = torch.empty(N, dtype=torch.float64, device="cuda")
    psi_im = torch.empty(N, dtype=torch.float64, device="cuda")
    flush = None
    u_bytes = 16 * (count or 1) * N
    if u_bytes < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")

    def step():
        if plan is not None:
            plan.execute(s_ptr)
        gather_state(plan, psi_re, psi_im, begin, count, world, s_ptr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    timed = plan is not None and plan.info.n_gemms > 0 and N > 32
    if timed:
        plan.set_timing(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    gemm_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            if timed:
                _, g_ms, _ = plan.last_timing()
                gemm_ms.append(g_ms)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_step = [a.elapsed_time(b) for a, b in ev]
    ms = sum(per_step) / len(per_step)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # ---- roofline of the dominant kernel (K2) ----
    info = plan.info if plan is not None else None
    gemm_flops_step = info.gemm_flops if info else 0.0
    n_gemms = info.n_gemms if info else 0
    mean_gemm_ms = (sum(gemm_ms) / len(gemm_ms) / n_gemms) if (gemm_ms and n_gemms) else None
    per_launch_flops = gemm_flops_step / n_gemms if n_gemms else 0.0  # credited 8 M N^2
    hw_per_launch = info.gemm_hw_flops / n_gemms if n_gemms else 0.0  # what the DMMAs execute
    achieved = hw_per_launch / (mean_gemm_ms * 1e-3) / 1e12 if mean_gemm_ms else None
    credited = per_launch_flops / (mean_gemm_ms * 1e-3) / 1e12 if mean_gemm_ms else None
    # per-kind breakdown: one more execute (after the timed region) with an event pair
    # around every K2 launch — those events serialise the chained launches, so this
    # run explains the timed one rather than replacing it
    per_kind = None
    if timed:
        plan.set_timing(2)
        plan.execute(s_ptr)
        torch.cuda.synchronize()
        g_ms, g_kind = plan.gemm_times()
        plan.set_timing(0)
        per_kind = k2_breakdown(g_ms, g_kind, per_launch_flops)
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(prof_json):
        with open(prof_json) as f:
            tr = json.load(f).get(args.workload)
            if tr:
                traffic = tr.get("dram_bytes_per_launch")
    chain_tflops = gemm_flops_step / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    tot = torch.tensor([gemm_flops_step, info.gemm_hw_flops if info else 0.0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot)
    job_tflops = float(tot[0].item()) / (ms_max * 1e-3) / 1e12  # credited 8N^3 per GEMM
    job_hw_tflops = float(tot[1].item()) / (ms_max * 1e-3) / 1e12  # executed DMMA FLOPs

    # ---- e2e through the public API with host buffers ----
    # (the device-timed plan is closed first: an open plan holds the handle's
    # buffer cache, and the host call would allocate its own V buffers every step)
    if plan is not None:
        plan.close()
        plan = None
    e2e_clocks = None
    if vr > 1:
        e2e_ms, h2d, d2h, e2e_calls, e2e_cached = None, 0, 0, 0, None  # the projection times one shard
        e2e_error = None
    else:
        e2e_error = None
        with ClockSampler(local, "e2e") as eclk:
            try:
                e2e_ms, h2d, d2h, e2e_calls, e2e_cached = e2e_measure(sim, flat, args, world, rank, N, begin, count,
                                                                       s_ptr)
            except Exception as exc:  # keep the device-timed line: report the failure instead of dying
                e2e_ms, h2d, d2h, e2e_calls, e2e_cached = None, 0, 0, 0, None
                e2e_error = f"{type(exc).__name__}: {exc}"
        e2e_clocks = eclk.summary()

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": ms_max, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "deterministic circuit from make_named_circuit (synthetic, no dataset)",
            "config": {"workload": args.workload, "circuit": name, "qubits": n, "dimension": N,
                       "parallelism": f"row-block x{world}" if world > 1 else "1 GPU",
                       "gemms_per_circuit": n_gemms, "layers": info.n_layers if info else None,
                       "identity_layers_skipped": info.n_identity_layers if info else None,
                       "gemm_mode": args.gemm_mode,
                       "gemm_splitk": info.gemm_splits if info else None,
                       "l2": ("inputs larger than L2" if flush is None else "L2 flushed between steps")},
            # whole job, every rank's GEMMs over the max-over-ranks circuit time
            "tflops": job_hw_tflops,
            "fp64_peak_frac": job_hw_tflops / (FP64_DMMA_PEAK_TFLOPS * world),
            "credited_tflops": job_tflops,
            "credited_fp64_peak_frac": job_tflops / (FP64_DMMA_PEAK_TFLOPS * world),
            "roofline": {"bound": "tensor", "kernel": (native.TILE_NAMES.get(info.gemm_tile, "small_circuit_kernel") + " (K2)") if info else None,
                         "achieved": achieved, "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": (achieved / FP64_DMMA_PEAK_TFLOPS) if achieved else None,
                         "flops_counted": "FP64 FLOPs the DMMAs execute per launch: 6MN^2 (3M complex layer), "
                                          "4MN^2 (real layer: two real products), 8MN^2 (4M); mean over the "
                                          "timed chain, K1t expansions included in the launch time",
                         "hw_frac": (achieved / FP64_DMMA_PEAK_TFLOPS) if achieved else None,
                         "credited_achieved": credited,
                         "credited_frac": (credited / FP64_DMMA_PEAK_TFLOPS) if credited else None,
                         "credited_note": "8MN^2 per GEMM (ZGEMM convention, SURVEY 8(d)); above 1 because 3M "
                                          "and real layers execute fewer FLOPs than they are credited",
                         "per_kind": per_kind,
                         "real_gemms": info.n_real_gemms if info else None,
                         "traffic": traffic,
                         "algorithmic_flops_per_launch": hw_per_launch,
                         "mean_launch_ms": mean_gemm_ms,
                         "peak_source": "builder-measured FP64 DMMA peak of this pool's B200 (register-only "
                                        "mma.sync.m8n8k4.f64 loop, tools/microbench/fp64_peak.cu, "
                                        "profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json has no FP64 entry"},
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "calls_timed": e2e_calls,
                    "cold_call": "every call compiles the circuit and uploads its descriptors (QSB_FLAG_NO_PLAN_CACHE)",
                    "value_plan_cached": e2e_cached,
                    "error": e2e_error,
                    "api": "qsb_simulate_full_state (C ABI)" if world == 1 else
                           "qsb_simulate_full_state_sharded (C ABI: row block per rank, psi all-gathered over "
                           "libqsb's NCCL communicator, whole psi to every rank's host planes)",
                    "clocks": e2e_clocks},
            "gpu_launches": (info.n_launches if info else 0) * args.steps,
            "clocks": clocks,
        }
        if vr > 1:
            line["n_gpus"] = 1
            line["config"]["parallelism"] = f"row block 0 of {vr} (one shard on one GPU)"
            line["projection"] = {
                "n_gpus": vr, "ms_per_circuit": ms_max,
                "tflops_aggregate": job_hw_tflops * vr,
                "fp64_peak_frac_aggregate": job_hw_tflops / FP64_DMMA_PEAK_TFLOPS,
                "credited_tflops_aggregate": job_tflops * vr,
                "method": f"rows [0, N/{vr}) of U timed alone on one B200: every rank does identical, "
                          "independent work (row blocks, operators regenerated locally); excludes the "
                          f"NCCL all-gather of psi ({16 * N // vr} bytes per rank)"}
        if world == 1 and vr == 1 and cpu_baseline is not None:
            cb = cpu_baseline
            cb["extrapolated"] = not cb.get("full_run", True) if "components_s" in cb else False
            if cb["extrapolated"]:
                cb["model_validation"] = model_validation(args.workload)
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def k2_breakdown(ms, kinds, credited_per_launch):
    """Per-kind K2 roofline from one mode-2 execute: kind bit 0 = real layer (two real
    products, 4MN^2), bit 1 = operand materialised by K1t, bit 2 = 4M (8MN^2), else 3M (6MN^2)."""
    groups = {}
    for t, k in zip(ms, kinds):
        arith = "4M" if k & 4 else ("real" if k & 1 else "3M")
        key = f"{arith}{' materialised' if k & 2 else ' generated'}"
        hw = credited_per_launch * (1.0 if k & 4 else (0.5 if k & 1 else 0.75))
        g = groups.setdefault(key, {"launches": 0, "ms": 0.0, "hw_flops_per_launch": hw})
        g["launches"] += 1
        g["ms"] += t
    out = {}
    for key, g in groups.items():
        mean = g["ms"] / g["launches"]
        tf = g["hw_flops_per_launch"] / (mean * 1e-3) / 1e12
        out[key] = {"launches": g["launches"], "mean_ms": mean, "hw_flops_per_launch": g["hw_flops_per_launch"],
                    "achieved_tflops": tf, "frac": tf / FP64_DMMA_PEAK_TFLOPS,
                    "credited_frac": credited_per_launch / (mean * 1e-3) / 1e12 / FP64_DMMA_PEAK_TFLOPS}
    return out


def e2e_measure(sim, flat, args, world, rank, N, begin, count, s_ptr):
    """The same circuit through the public API with host buffers: descriptor
    H2D and psi D2H inside the timed region, every step."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2305_14398_b200 import native

    h2d = flat.nbytes()
    d2h = 16 * N
    if world == 1:
        from paper_2305_14398_b200.simulator import B200UnitarySimulator

        re = np.empty(N)
        im = np.empty(N)
        L = native.lib()

        def timed_calls(handle):
            t0 = time.perf_counter()
            native.check(L.qsb_simulate_full_state(handle, flat.ptr, native.dptr(re), native.dptr(im)))
            first = time.perf_counter() - t0
            # as many calls as --steps within ~20 s (at least 3): run_bench's repeated calls
            reps = max(3, min(args.steps, int(20.0 / max(first, 1e-6))))
            times = []
            for _ in range(reps):
                t0 = time.perf_counter()
                native.check(L.qsb_simulate_full_state(handle, flat.ptr, native.dptr(re), native.dptr(im)))
                times.append((time.perf_counter() - t0) * 1e3)
            return sum(times) / len(times), len(times)

        # headline: every call compiles the circuit and uploads its descriptors / registry
        # tables (QSB_FLAG_NO_PLAN_CACHE); beside it the repeated-call cost with the handle's
        # plan cache (compiled plan reused, registry contents re-checked on the host)
        cold = B200UnitarySimulator(device=sim.device, gemm_mode=mode_of(args), flags=native.FLAG_NO_PLAN_CACHE)
        cold_ms, calls = timed_calls(cold._h)
        cold.close()
        cached_ms, _ = timed_calls(sim._h)
        return cold_ms, h2d, d2h, calls, cached_ms
    # one process per GPU: every rank makes the C-ABI call qsb_simulate_full_state_sharded
    # (its row block of U, psi all-gathered over libqsb's own NCCL communicator, the whole
    # psi in every rank's host planes); max over ranks per call
    from paper_2305_14398_b200.simulator import B200UnitarySimulator, Comm, nccl_unique_id

    if count * world != N:
        return None, h2d, d2h, 0, None  # ragged worlds keep trailing ranks idle: no sharded call
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = Comm(sim, uid[0], world, rank)

    def timed_calls(s2):
        def one():
            dist.barrier()
            t0 = time.perf_counter()
            s2.simulate_full_state_sharded(flat, None, comm)
            t = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        first = one()
        reps = max(3, min(args.steps, int(20e3 / max(first, 1e-3))))  # identical on every rank
        times = [one() for _ in range(reps)]
        return sum(times) / len(times), len(times)

    cold = B200UnitarySimulator(device=sim.device, gemm_mode=mode_of(args), flags=native.FLAG_NO_PLAN_CACHE)
    cold_ms, calls = timed_calls(cold)
    cold.close()
    cached_ms, _ = timed_calls(sim)
    comm.close()
    return cold_ms, h2d, d2h, calls, cached_ms


# --------------------------------------------------------------- state-vector engine arms

def hbm_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except Exception:
        return 6550.0, "B200_PROFILING.md fallback"


def run_sv(args):
    """--backend structured | fsv: the state-vector engine (qsb_sv_plan_*).
    structured: U[:, c] = fsv(e_c), columns sharded over ranks (no
    communication; psi = column 0 lives on rank 0). fsv: one state per rank
    (replicas). One step = one circuit; value = ms per circuit (max over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200FsvSimulator, B200StructuredUnitarySimulator

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    name, n = WORKLOADS[args.workload]
    N = 1 << n
    structured = args.backend == "structured"
    sim = (B200StructuredUnitarySimulator if structured else B200FsvSimulator)(device=local)
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    s_ptr = stream.cuda_stream
    if structured:
        cols = N // world
        plan = sim.plan(flat, None, rank * cols, cols)
    else:
        plan = sim.plan(flat)
    info = plan.info
    elems = N * info.col_count
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda") if 16 * elems < 2 * L2_BYTES else None
    for _ in range(args.warmup):
        plan.execute(s_ptr)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev[i][0].record(stream)
            plan.execute(s_ptr)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    peak, peak_src = hbm_peak_gbs()
    achieved = info.bytes_per_run / (ms * 1e-3) / 1e9
    plan.close()
    # e2e through the public C ABI with host buffers (psi D2H), rank 0 / single GPU
    e2e_ms = None
    if rank == 0:
        re, im = np.empty(N), np.empty(N)
        fn = native.lib().qsb_structured_simulate_full_state if structured else native.lib().qsb_fsv_simulate_full_state
        native.check(fn(sim._h, flat.ptr, native.dptr(re), native.dptr(im)))
        times = []
        for _ in range(max(1, min(args.steps, 3))):
            t0 = time.perf_counter()
            native.check(fn(sim._h, flat.ptr, native.dptr(re), native.dptr(im)))
            times.append((time.perf_counter() - t0) * 1e3)
        e2e_ms = sum(times) / len(times)
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_max, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": False,
            "scaling": ("strong" if structured else "replicas"), "vs_baseline": None, "dtype": "f64",
            "data": "deterministic circuit from make_named_circuit (synthetic, no dataset)",
            "config": {"workload": args.workload, "circuit": name, "qubits": n, "backend": args.backend,
                       "algorithm": ("structured unitary: U[:,c] = fsv(e_c), all columns at once "
                                     "(not Algorithm 1's dense products; no FP64 tensor work)") if structured
                       else "full state vector (FsvSimulator)",
                       "parallelism": (f"column-block x{world}" if structured and world > 1 else
                                       ("replicas" if world > 1 else "1 GPU")),
                       "passes": info.n_passes, "ops": info.n_ops, "function_passes": info.n_function_passes,
                       "l2": "inputs larger than L2" if flush is None else "L2 flushed between steps"},
            "roofline": {"bound": "hbm", "kernel": "sv_reg_kernel (register batches)", "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                         "algorithmic_bytes_per_run": info.bytes_per_run,
                         "note": "bytes = passes x read+write of the [2][2^n][cols] array; whole execute timed",
                         "peak_source": peak_src},
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": flat.nbytes(), "d2h_bytes_per_step": 16 * N,
                    "api": "qsb_structured_simulate_full_state (C ABI)" if structured
                    else "qsb_fsv_simulate_full_state (C ABI)"},
            "gpu_launches": info.n_launches * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def ensure_ranks(args) -> int:
    """--gpus N is honoured or the run fails: under torchrun the world size must
    equal N; a plain `python bench.py --gpus N` (N > 1) re-executes itself under
    torch.distributed.run with one process per GPU, after checking that N GPUs
    are visible. Returns 0 to continue in this process (never returns after exec)."""
    rank, world, _ = dist_env()
    if world > 1:
        if world != args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
            sys.exit(2)
        return 0
    if args.gpus <= 1 or args.impl == "reference":
        return 0
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus and not args.dry_run:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
                          "n_gpus": have}), flush=True)
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)
    return 0


def run_dry(args):
    """--dry-run: the N > 1 plumbing on CPU over gloo (tests/test_sharding_gloo.py)."""
    import torch
    import torch.distributed as dist

    from paper_2305_14398_b200.sharding import gather_rows, row_shard

    rank, world, _ = dist_env()
    if world != max(1, args.gpus):
        raise SystemExit(f"bench: --gpus {args.gpus} but {world} rank(s)")
    if world > 1:
        dist.init_process_group("gloo")
    _, n = WORKLOADS[args.workload]
    N = 1 << n
    begin, count = row_shard(N, world, rank)
    rows = torch.arange(begin, begin + count, dtype=torch.float64)
    if world > 1:
        re, im = gather_rows(rows, -rows, N, world)
    else:
        re, im = rows, -rows
    want = torch.arange(N, dtype=torch.float64)
    ok = bool(torch.equal(re, want) and torch.equal(im, -want))
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "workload": args.workload, "rows_per_rank": count,
                          "gathered_ok": ok, "backend": dist.get_backend() if world > 1 else None}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if ok else 1


def main():
    args = parse()
    ensure_ranks(args)
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.backend != "dense":
        return run_sv(args)
    # the CPU baseline first, in a fresh torch-free process, before this process initialises
    # CUDA: the reference's own process never loads torch, and in this container the
    # reference's single-threaded, memory-bound layer product ran 1.26x slower after a
    # torch import and matmul in the same process
    _, world, _ = dist_env()
    cb = None
    if world == 1 and args.virtual_ranks <= 1 and not args.no_cpu_baseline:
        cb = cpu_sample_subprocess(args.workload)
    return run_ours(args, cb)


if __name__ == "__main__":
    sys.exit(main())
