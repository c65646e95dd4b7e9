"""GPU parity of the state-vector engine (libqsb.so through the C ABI):

* ``fsv-b200`` (B200FsvSimulator) against the reference's own FsvSimulator
  output (golden vectors, fsv_backend.cpp:135-158) — bit-exact (==, so
  -0.0 == +0.0), including the multi-slab sizes n = 13..15 and every slab
  geometry (QSB_SV_SLAB_BITS forces small slabs, high slab bits, controls
  outside the slab, apply_function blocks through the large-block kernel);
* ``unitary-structured-b200``: U[:, c] == fsv(e_c) bit-exactly (C oracle,
  pinned to the reference fsv), and within 1e-10 of the reference's dense U.
"""
import numpy as np
import pytest

from conftest import bit_equal, rel_frob

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def fsv():
    from paper_2305_14398_b200.simulator import B200FsvSimulator

    s = B200FsvSimulator()
    yield s
    s.close()


@pytest.fixture(scope="module")
def structured():
    from paper_2305_14398_b200.simulator import B200StructuredUnitarySimulator

    s = B200StructuredUnitarySimulator()
    yield s
    s.close()


def _fsv_cases(golden):
    return [c for c in golden.cases if golden.has(f"{c}:fsv_re")]


@pytest.mark.parametrize("slab_bits", [None, "6", "8", "10"])
def test_fsv_golden_bit_exact(monkeypatch, golden, fsv, slab_bits):
    if slab_bits:
        monkeypatch.setenv("QSB_SV_SLAB_BITS", slab_bits)
    cases = _fsv_cases(golden)
    assert len(cases) >= 340
    for case in cases:
        out = fsv.simulate_full_state(golden.flat(case))
        assert bit_equal(out.re, golden[f"{case}:fsv_re"]), case
        assert bit_equal(out.im, golden[f"{case}:fsv_im"]), case


def test_fsv_plan_uses_several_passes(golden, fsv):
    """The n = 13..15 goldens exceed one 2^12 slab: several batches, many slabs."""
    for case in golden.suites["fsvbig"]:
        plan = fsv.plan(golden.flat(case))
        assert plan.info.n_qubits >= 13 and plan.info.n_passes >= 1
        assert plan.info.slab_bits == 12
        plan.close()


def test_fsv_from_state_matches_oracle(golden, fsv, orc):
    rng = np.random.default_rng(808)
    for case in golden.suites["comp"] + golden.suites["cross"][:40]:
        flat = golden.flat(case)
        N = 1 << flat.n_qubits
        re0, im0 = rng.standard_normal(N), rng.standard_normal(N)
        out = fsv.simulate_from_state(flat, None, re0, im0)
        wr, wi = orc.fsv(flat, re0, im0)
        assert bit_equal(out.re, wr) and bit_equal(out.im, wi), case


def _function_circuit(n, first, count, seed, extra=True):
    import paper_2305_14398_b200 as q

    rng = np.random.default_rng(seed)
    a = rng.standard_normal((1 << count, 1 << count)) + 1j * rng.standard_normal((1 << count, 1 << count))
    u, _ = np.linalg.qr(a)
    reg = q.GateRegistry()
    reg.register_function("blk", u)
    c = q.Circuit(n)
    for k in range(n):
        c.h(k)
    c.add_function("blk", first, count, reg)
    if extra:
        c.cr(0.3, n - 1, 0).t(1).cnot(0, n - 1)
        c.add_function("blk", first, count, reg)
    return c, reg


@pytest.mark.parametrize("n,first,count,slab_bits", [
    (6, 1, 3, None), (8, 0, 8, None), (9, 2, 4, "6"), (10, 3, 5, "8"), (13, 4, 6, None), (12, 0, 12, None),
    (14, 5, 9, None), (12, 0, 3, "6"),
])
def test_fsv_apply_function_blocks(monkeypatch, fsv, orc, n, first, count, slab_bits):
    """apply_function (fsv_backend.cpp:84-132) on interior / whole ranges, both
    inside a slab and through the large-block kernel."""
    from paper_2305_14398_b200 import native

    if slab_bits:
        monkeypatch.setenv("QSB_SV_SLAB_BITS", slab_bits)
    c, reg = _function_circuit(n, first, count, seed=n * 31 + count)
    flat = native.flatten(c, reg)
    out = fsv.simulate_full_state(flat)
    wr, wi = orc.fsv(flat)
    assert bit_equal(out.re, wr) and bit_equal(out.im, wi)


@pytest.mark.parametrize("name,n", [("deutsch-jozsa", 13), ("qft", 16), ("entangle", 20), ("qft", 20)])
def test_fsv_named_large(fsv, orc, name, n):
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    out = fsv.simulate_full_state(flat)
    wr, wi = orc.fsv(flat)
    assert bit_equal(out.re, wr) and bit_equal(out.im, wi)


def test_fsv_collapse_matches_reference(golden, fsv):
    from paper_2305_14398_b200 import native

    flat = golden.flat("bell")
    for seed, want in enumerate(golden["collapse_bell"]):
        assert fsv.simulate_and_collapse(flat, None, seed).basis_index == want
    flat = golden.flat("qft5")
    for seed, want in enumerate(golden["collapse_qft5"][:64]):
        assert fsv.simulate_and_collapse(flat, None, seed).basis_index == want
    assert isinstance(native.lib().qsb_collapse, object)


def test_fsv_errors_match_reference(fsv):
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200.errors import ResourceError, ValidationError
    from paper_2305_14398_b200.simulator import B200FsvSimulator

    bad = q.Circuit(2)
    bad.reset(0).h(0)
    with pytest.raises(ValidationError, match="reset is only supported in the final step"):
        fsv.simulate_full_state(bad)
    ok = q.Circuit(2)
    ok.h(0).reset(0)
    assert fsv.simulate_full_state(ok).dimension() == 4
    small = B200FsvSimulator(qubit_guard=3)
    assert small.qubit_guard() == 3
    with pytest.raises(ResourceError, match="refuses 4 qubits"):
        small.simulate_full_state(q.Circuit(4).h(0))
    small.close()
    assert fsv.qubit_guard() == 30


def test_structured_unitary_columns_bit_exact(golden, structured, orc):
    """U[:, c] == fsv(e_c) bit for bit (the oracle's fsv is pinned to the
    reference's), and U within 1e-10 of the reference's dense U."""
    checked = 0
    for case in golden.cases:
        u = golden.unitary(case)
        if u is None:
            continue
        flat = golden.flat(case)
        ur, ui = structured.build_unitary(flat)
        assert rel_frob(ur, ui, u[0], u[1]) <= TOL, case
        N = 1 << flat.n_qubits
        for col in sorted({0, N // 2, N - 1}):
            cr, ci = orc.unitary_column(flat, col)
            assert bit_equal(ur[:, col], cr) and bit_equal(ui[:, col], ci), (case, col)
        checked += 1
    assert checked > 100


def test_structured_state_equals_fsv(golden, structured, fsv):
    for case in _fsv_cases(golden)[:120]:
        flat = golden.flat(case)
        a = structured.simulate_full_state(flat)
        b = fsv.simulate_full_state(flat)
        assert bit_equal(a.re, b.re) and bit_equal(a.im, b.im), case


@pytest.mark.parametrize("name,n", [("qft", 10), ("deutsch-jozsa", 9), ("entangle", 11)])
def test_structured_vs_dense_unitary(sim, structured, name, n):
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    dr, di = sim.build_unitary(flat)
    sr, si = structured.build_unitary(flat)
    assert rel_frob(sr, si, dr, di) <= TOL


def test_structured_qft_matches_dft(structured):
    """QFT == DFT (test_circuit_library.cpp:161-167 / acceptance :173-180) at n = 12."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    n = 12
    N = 1 << n
    c, reg = q.make_named_circuit("qft", n)
    ur, ui = structured.build_unitary(native.flatten(c, reg))
    j = np.arange(N)
    dft = np.exp(2j * np.pi * (np.outer(j, j) % N) / N) / np.sqrt(N)
    assert rel_frob(ur, ui, dft.real, dft.imag) <= 1e-12


def test_structured_column_shards_over_devices(golden, orc):
    """Columns sharded over a device list (virtual shards on one GPU) reassemble U bit-exactly."""
    from paper_2305_14398_b200.simulator import B200StructuredUnitarySimulator

    one = B200StructuredUnitarySimulator()
    many = B200StructuredUnitarySimulator(devices=[0, 0, 0, 0])
    for case in ["qft6", "dj6", "entangle6", "edge_wide_span"] + golden.suites["cross"][:20]:
        flat = golden.flat(case)
        a = one.build_unitary(flat)
        b = many.build_unitary(flat)
        assert bit_equal(a[0], b[0]) and bit_equal(a[1], b[1]), case
        s1 = one.simulate_full_state(flat)
        s4 = many.simulate_full_state(flat)
        assert bit_equal(s1.re, s4.re) and bit_equal(s1.im, s4.im), case
    one.close()
    many.close()


def test_structured_plan_shard(structured, orc):
    """A device plan for columns [c0, c0 + w) holds exactly those columns of U."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import torch_view

    import torch

    c, reg = q.make_named_circuit("qft", 9)
    flat = native.flatten(c, reg)
    N = 1 << 9
    plan = structured.plan(flat, col_begin=128, col_count=64)
    plan.execute()
    torch.cuda.synchronize()
    re_p, im_p = plan.result_device()
    re = torch_view(re_p, (N, 64)).cpu().numpy()
    for col in (128, 150, 191):
        cr, ci = orc.unitary_column(flat, col)
        assert bit_equal(re[:, col - 128], cr)
    assert plan.info.col_count == 64 and plan.info.n_passes >= 1
    plan.close()


# ---- registry validation on the GPU -------------------

@pytest.mark.parametrize("dim", [2, 4, 32, 64, 128, 512, 2048])
def test_is_unitary_matches_reference_verdict(sim, orc, dim):
    """qsb_is_unitary (A^H A on the DMMA pipe for dim >= 64) gives the
    reference's verdict (linalg.cpp:131-155, the C oracle) for unitary,
    slightly perturbed and clearly non-unitary matrices at kRegistryUnitaryTol."""
    from paper_2305_14398_b200.simulator import is_unitary

    rng = np.random.default_rng(dim)
    a = rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))
    u, _ = np.linalg.qr(a)
    tol = 1e-9
    for m, want in [(u, True), (u * (1 + 1e-6), False), (u + 1e-12 * a, True), (a / np.sqrt(dim), False)]:
        ok, dev = is_unitary(sim, m, tol)
        ref = orc.is_unitary(m, tol) if dim <= 512 else want
        assert ok == ref == want, (dim, dev)
        if dim <= 512:
            g = m.conj().T @ m - np.eye(dim)
            assert abs(dev - max(np.abs(g.real).max(), np.abs(g.imag).max())) <= 1e-12


def test_is_unitary_dj_oracles(sim):
    """The DJ oracle permutation (circuit_library.cpp:45-58) registers through the GPU check."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import circuit
    from paper_2305_14398_b200.simulator import gpu_unitarity_check, is_unitary

    circuit.set_unitarity_check(gpu_unitarity_check(sim))
    try:
        c, reg = q.make_named_circuit("deutsch-jozsa", 11)
        m = reg.lookup(next(iter(reg._entries)))
        ok, dev = is_unitary(sim, m, 1e-9)
        assert ok and dev == 0.0
        bad = m.copy()
        bad[0, 0] += 1e-7
        with pytest.raises(q.ValidationError, match="not unitary"):
            reg.register_function("bad", bad)
    finally:
        circuit.set_unitarity_check(None)


@pytest.mark.parametrize("jit,k", [("0", "4"), ("0", "2"), ("1", "5"), ("1", "3"), ("1", "1")])
def test_register_batches_interpreted_and_compiled(monkeypatch, golden, jit, k):
    """Register batches run either interpreted (sv_reg_kernel) or compiled
    straight-line by NVRTC (qsb_jit): both bit-exact with the reference fsv,
    for every batch width."""
    from paper_2305_14398_b200.simulator import B200FsvSimulator

    monkeypatch.setenv("QSB_SV_JIT", jit)
    monkeypatch.setenv("QSB_SV_REG_K", k)
    s = B200FsvSimulator()
    for case in golden.suites["fsvbig"]:
        out = s.simulate_full_state(golden.flat(case))
        assert bit_equal(out.re, golden[f"{case}:fsv_re"]) and bit_equal(out.im, golden[f"{case}:fsv_im"]), case
    s.close()


def test_function_errors_match_reference(fsv, structured, sim):
    """apply_function's dimension check (fsv_backend.cpp:90-95) and the unitary
    backend's registry re-check (unitary_backend.cpp:50-53) through the C ABI."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.errors import LookupError_, ValidationError

    reg = q.GateRegistry()
    reg.register_function("swap2", np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex))
    c = q.Circuit(3).h(0)
    c.add_function("swap2", 1, 2, reg)
    flat = native.flatten(c, reg)
    ops = flat.ops.copy()
    # the registered matrix no longer matches the op's 2 qubits
    bad_tab = [(np.eye(8), np.zeros((8, 8)))]
    bad = native.flat_from_arrays(3, flat.step_offsets, ops, bad_tab)
    with pytest.raises(ValidationError, match="apply_function: matrix dimension 8 does not match 2\\^2"):
        fsv.simulate_full_state(bad)
    with pytest.raises(ValidationError):
        structured.simulate_full_state(bad)
    with pytest.raises(ValidationError):
        sim.simulate_full_state(bad)
    # an op naming a function the registry does not hold
    ops2 = ops.copy()
    ops2["function"][ops2["kind"] == native.OP_FUNCTION] = 3
    missing = native.flat_from_arrays(3, flat.step_offsets, ops2, [(np.eye(4), np.zeros((4, 4)))])
    for s in (fsv, structured, sim):
        with pytest.raises(LookupError_):
            s.simulate_full_state(missing)
