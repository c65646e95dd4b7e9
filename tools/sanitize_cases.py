"""Small-shape cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) over every synchronisation-heavy kernel family.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py <case>

Each case runs one circuit through the C ABI (libqsb.so) under the plan-time
switch that selects the kernel variant, then checks psi against the C oracle
(test infrastructure, the checker only). Exit 0 = results correct.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2305_14398_b200 as q  # noqa: E402
from paper_2305_14398_b200 import native  # noqa: E402


def k2_circuit(n):
    """Four layers -> three K2 GEMMs covering every operand kind: a dense
    non-monomial layer (H on every qubit: K1t-materialised), a complex monomial
    layer (controlled phase: materialised), a real monomial (X: generated), a
    real non-monomial (H on one qubit: generated)."""
    c = q.Circuit(n)
    for k in range(n):
        c.h(k)
    c.cr(np.pi / 2, 1, 0)
    c.x(0)  # each op overlaps the previous one: its own step
    c.h(0)
    return c, None


# case -> (circuit builder, qubits, environment, gemm mode)
CASES = {
    # K2 warp-specialised, 3M sum plane, stream-K (N = 1024: 256 tiles >= 148)
    "k2_streamk_3m": (k2_circuit, 10, {}, native.GEMM_AUTO),
    "k2_streamk_4m": (k2_circuit, 10, {}, native.GEMM_4M),
    # cluster split-K through DSMEM
    "k2_splitk2": (k2_circuit, 10, {"QSB_STREAMK": "0", "QSB_SPLITK": "2"}, native.GEMM_AUTO),
    "k2_splitk4": (k2_circuit, 10, {"QSB_STREAMK": "0", "QSB_SPLITK": "4"}, native.GEMM_AUTO),
    "k2_splitk8": (k2_circuit, 10, {"QSB_STREAMK": "0", "QSB_SPLITK": "8"}, native.GEMM_AUTO),
    "k2_splitk4_nopdl": (k2_circuit, 10, {"QSB_STREAMK": "0", "QSB_SPLITK": "4", "QSB_NO_PDL": "1"}, native.GEMM_AUTO),
    "k2_n9_default": (k2_circuit, 9, {}, native.GEMM_AUTO),
    # every layer materialised / every layer generated
    "k2_mat_all": (k2_circuit, 9, {"QSB_MATERIALIZE": "1"}, native.GEMM_AUTO),
    "k2_mat_none": (k2_circuit, 9, {"QSB_MATERIALIZE": "0"}, native.GEMM_AUTO),
    # v1 tiles (zgemm_gen_kernel)
    "k2_gen_128x64": (k2_circuit, 9, {"QSB_TILE": "0"}, native.GEMM_AUTO),
    "k2_gen_64x64": (k2_circuit, 9, {"QSB_TILE": "1"}, native.GEMM_AUTO),
    "k2_gen_32x32": (k2_circuit, 8, {"QSB_TILE": "2"}, native.GEMM_AUTO),
    # K2c: the whole chain in one persistent dataflow launch (k-splits 1 / 2 / 4)
    "k2c_qft9": ("qft", 9, {"QSB_CHAIN": "1"}, native.GEMM_AUTO),
    "k2c_entangle10": ("entangle", 10, {"QSB_CHAIN": "1"}, native.GEMM_AUTO),
    "k2c_qft10_s4": ("qft", 10, {"QSB_CHAIN": "1", "QSB_CHAIN_SPLITS": "4"}, native.GEMM_AUTO),
    # K2m cluster chains (N = 64 / 128 / 256), with and without double-buffered operators
    "k2m_qft6": ("qft", 6, {}, native.GEMM_AUTO),
    "k2m_qft7": ("qft", 7, {}, native.GEMM_AUTO),
    "k2m_qft8": ("qft", 8, {}, native.GEMM_AUTO),
    "k2m_entangle8_nodbuf": ("entangle", 8, {"QSB_MID_NODBUF": "1"}, native.GEMM_AUTO),
    "k2m_dj7": ("deutsch-jozsa", 7, {}, native.GEMM_AUTO),
    # K2s one-CTA chains
    "k2s_qft4": ("qft", 4, {}, native.GEMM_AUTO),
    "k2s_qft5": ("qft", 5, {}, native.GEMM_AUTO),
    "k2s_fma_qft2": ("qft", 2, {}, native.GEMM_AUTO),
}


def run_case(name):
    import oracle

    build, n, env, mode = CASES[name]
    os.environ.update(env)
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    if callable(build):
        c, reg = build(n)
    else:
        c, reg = q.make_named_circuit(build, n)
    flat = native.flatten(c, reg)
    sim = B200UnitarySimulator(device=0, gemm_mode=mode)
    out = sim.simulate_full_state(flat)
    sim.close()
    re, im = oracle.Oracle().fsv(flat)
    err = np.sqrt(np.sum((out.re - re) ** 2 + (out.im - im) ** 2)) / np.sqrt(np.sum(re ** 2 + im ** 2))
    print(f"{name}: rel err {err:.2e}", flush=True)
    return 0 if err <= 1e-10 else 1


def run_registry():
    """gram_kernel (TMA + DMMA, dim multiple of 64) and gram_small_kernel."""
    from paper_2305_14398_b200.simulator import B200UnitarySimulator, is_unitary

    sim = B200UnitarySimulator(device=0)
    rng = np.random.default_rng(7)
    ok = True
    for d in (16, 128):
        a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        u, _ = np.linalg.qr(a)
        good, dev = is_unitary(sim, u, 1e-9)
        ok = ok and good
        print(f"gram dim {d}: unitary={good} dev={dev:.2e}", flush=True)
    sim.close()
    return 0 if ok else 1


def run_sv():
    """State-vector engine: register batches (NVRTC and interpreted), slab batches."""
    import oracle
    from paper_2305_14398_b200.simulator import B200FsvSimulator, B200StructuredUnitarySimulator

    orc = oracle.Oracle()
    ok = True
    for cls, name, n in ((B200FsvSimulator, "qft", 9), (B200StructuredUnitarySimulator, "qft", 6),
                         (B200FsvSimulator, "deutsch-jozsa", 7)):
        c, reg = q.make_named_circuit(name, n)
        flat = native.flatten(c, reg)
        s = cls(device=0)
        out = s.simulate_full_state(flat)
        s.close()
        re, im = orc.fsv(flat)
        same = np.array_equal(out.re, re) and np.array_equal(out.im, im)
        ok = ok and same
        print(f"sv {cls.__name__} {name}({n}): bit-exact={same}", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    which = sys.argv[1]
    if which == "list":
        print(" ".join(list(CASES) + ["registry", "sv"]))
        sys.exit(0)
    if which.startswith("list:"):  # cases whose name starts with one of the comma-separated prefixes
        pre = which[5:].split(",")
        print(" ".join(c for c in list(CASES) + ["registry", "sv"] if any(c.startswith(p) for p in pre)))
        sys.exit(0)
    if which == "registry":
        sys.exit(run_registry())
    if which == "sv":
        sys.exit(run_sv())
    sys.exit(run_case(which))
