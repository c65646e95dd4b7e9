"""GPU parity: the B200 path (libqsb.so, through the C ABI) against the golden
vectors recorded from the reference and against the C oracle.

Bars (BASELINE.json north_star):
  * operator entries / permutation indexing: bit-exact (==, as the reference's
    ComplexMatrix::operator==, so -0.0 == +0.0);
  * amplitudes and U: ||delta||_F / ||ref||_F <= 1e-10.
"""
import numpy as np
import pytest

from conftest import bit_equal, rel_frob

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _named_cases(golden):
    return [c for c in golden.cases
            if not c.split("_")[0] in ("cross", "fsv", "fsvbig", "norm", "steps", "par", "det", "comp")
            and golden.has(f"{c}:psi_re")]


def test_named_circuits_state(golden, sim):
    worst = 0.0
    for case in _named_cases(golden):
        flat = golden.flat(case)
        out = sim.simulate_full_state(flat)
        re, im = golden.psi(case)
        err = rel_frob(out.re, out.im, re, im)
        worst = max(worst, err)
        assert err <= TOL, (case, err)
    print(f"named circuits: worst relative L2 error {worst:.3e}")


def test_named_circuits_unitary(golden, sim):
    for case in _named_cases(golden):
        u = golden.unitary(case)
        if u is None:
            continue
        ur, ui = sim.build_unitary(golden.flat(case))
        assert rel_frob(ur, ui, u[0], u[1]) <= TOL, case


@pytest.fixture(scope="module", params=["4m", "3m"])
def sim_mode(request):
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    s = B200UnitarySimulator(gemm_mode=native.GEMM_4M if request.param == "4m" else native.GEMM_3M)
    yield s
    s.close()


@pytest.mark.parametrize("suite", ["cross", "fsv", "norm", "steps", "par", "det", "comp"])
def test_random_suites(golden, sim_mode, suite):
    sim = sim_mode
    worst = 0.0
    for case in golden.suites[suite]:
        flat = golden.flat(case)
        out = sim.simulate_full_state(flat)
        re, im = golden.psi(case)
        err = rel_frob(out.re, out.im, re, im)
        worst = max(worst, err)
        assert err <= TOL, (case, err)
        u = golden.unitary(case)
        if u is not None:
            ur, ui = sim.build_unitary(flat)
            assert rel_frob(ur, ui, u[0], u[1]) <= TOL, case
    print(f"{suite}: worst {worst:.3e}")


def test_layer_operators_bit_exact(golden, sim, orc):
    """K1 expansion == kronecker_fold(fill_layer(layer)) entrywise, and for
    single-layer steps == the reference's step_unitary."""
    from paper_2305_14398_b200.simulator import step_layer_count

    checked = 0
    for case in golden.cases:
        steps = golden.steps(case)
        if not steps:
            continue
        flat = golden.flat(case)
        for s, (sr, si) in enumerate(steps):
            nl = step_layer_count(flat, None, s)
            for layer in range(nl):
                gr, gi = sim.layer_operator(flat, None, s, layer)
                orr, ori = orc.layer_operator(flat, s, layer)
                assert bit_equal(gr, orr) and bit_equal(gi, ori), (case, s, layer)
                checked += 1
            if nl == 1:
                gr, gi = sim.layer_operator(flat, None, s, 0)
                assert bit_equal(gr, sr) and bit_equal(gi, si), (case, s)
    assert checked > 100


def test_initial_state(golden, sim):
    """test_unitary_backend.cpp:143-153: U applied to random states."""
    for case in golden.suites["comp"]:
        flat = golden.flat(case)
        r0, i0 = golden[f"{case}:state_re"], golden[f"{case}:state_im"]
        out = sim.simulate_from_state(flat, None, r0, i0)
        ur, ui = golden.unitary(case)
        u = ur + 1j * ui
        want = u @ (r0 + 1j * i0)
        assert rel_frob(out.re, out.im, want.real, want.imag) <= TOL
        assert abs(np.sum(out.re ** 2 + out.im ** 2) - 1.0) < 1e-9


def test_probabilities_and_collapse(golden, sim):
    for key in ["comp_0", "comp_1"]:
        re, im = golden[f"{key}:state_re"], golden[f"{key}:state_im"]
        p, norm = sim.probabilities(re, im)
        assert bit_equal(p, golden[f"{key}:probs"])  # p_i bit-exact (state.cpp:58-65)
        assert abs(norm - float(golden[f"{key}:norm"])) < 1e-14
    flat = golden.flat("bell")
    for seed, want in enumerate(golden["collapse_bell"]):
        assert sim.simulate_and_collapse(flat, None, seed).basis_index == int(want)
    flat = golden.flat("qft5")
    for seed, want in enumerate(golden["collapse_qft5"][:50]):
        assert sim.simulate_and_collapse(flat, None, seed).basis_index == int(want)


def test_errors_match_reference(sim):
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    bad = q.Circuit(2)
    bad.reset(0).h(0)
    with pytest.raises(q.ValidationError):
        sim.simulate_full_state(bad)
    ok = q.Circuit(2)
    ok.h(0).reset(0)
    assert sim.simulate_full_state(ok).dimension() == 4
    small = B200UnitarySimulator(qubit_guard=3)
    with pytest.raises(q.ResourceError) as e:
        small.simulate_full_state(q.Circuit(4))
    assert "estimated memory 2176 bytes" in str(e.value)  # memory_estimate(4) (unitary_backend.cpp:156-166)
    # the reference's message word for word (unitary_backend.cpp:197-205), this backend's name
    assert str(e.value).endswith("unitary-b200 backend refuses 4 qubits (guard 3): estimated memory 2176 bytes "
                                 "(2.18 kB at 8 bytes per complex; engine-accurate 12.54 kB)"), str(e.value)
    assert small.simulate_full_state(q.Circuit(3)).dimension() == 8
    small.close()


def test_hbm_guard(sim):
    assert sim.qubit_guard() >= 15  # 2 x 16 x 4^15 B = 34 GB fits any B200


@pytest.mark.parametrize("name,n", [("qft", 10), ("entangle", 10), ("deutsch-jozsa", 10), ("qft", 11)])
def test_large_against_oracle_fsv(sim, orc, name, n):
    """Beyond the dense oracle: psi vs the reference's fsv restatement, and
    sampled columns of U vs fsv(e_c)."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    out = sim.simulate_full_state(flat)
    re, im = orc.fsv(flat)
    assert rel_frob(out.re, out.im, re, im) <= TOL
    ur, ui = sim.build_unitary(flat)
    rng = np.random.default_rng(7)
    for col in rng.choice(1 << n, size=4, replace=False):
        cr, ci = orc.unitary_column(flat, int(col))
        assert rel_frob(ur[:, col], ui[:, col], cr, ci) <= TOL


def test_row_shards_match_full(monkeypatch, sim):
    """Row-block sharding (the multi-GPU decomposition) on one GPU: G virtual
    shards computed separately reproduce the full U and psi exactly (for a
    fixed summation order: no split-K)."""
    import torch

    monkeypatch.setenv("QSB_SPLITK", "1")
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit("qft", 9)
    flat = native.flatten(c, reg)
    full_re, full_im = sim.build_unitary(flat)
    N = 1 << 9
    for G in (2, 4, 8):
        rows = N // G
        for r in range(G):
            plan = sim.plan(flat, None, r * rows, rows)
            plan.execute()
            torch.cuda.synchronize()
            re_p, im_p = plan.unitary_device()
            got = np.empty((rows, N))
            gim = np.empty((rows, N))
            native_copy(re_p, got)
            native_copy(im_p, gim)
            assert bit_equal(got, full_re[r * rows:(r + 1) * rows])
            assert bit_equal(gim, full_im[r * rows:(r + 1) * rows])
            plan.close()


def native_copy(dev_ptr, host):
    from paper_2305_14398_b200.simulator import torch_view

    host[...] = torch_view(dev_ptr, host.shape).cpu().numpy()


@pytest.mark.parametrize("tile", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("name,n", [("qft", 8), ("deutsch-jozsa", 9), ("entangle", 9)])
def test_every_gemm_tile_variant(monkeypatch, sim, orc, tile, name, n):
    """Force each K2 variant (v1 128x64 / 64x64 / 32x32, warp-specialised 4M / 3M)
    through the QSB_TILE debug switch and check it against the oracle."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    monkeypatch.setenv("QSB_TILE", str(tile))
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    ur, ui = sim.build_unitary(flat)
    orr, ori = orc.circuit_unitary(flat)
    assert rel_frob(ur, ui, orr, ori) <= TOL


@pytest.mark.parametrize("mode", ["4m", "3m"])
def test_qft12_modes_against_dft_columns(mode, orc):
    """n = 12 through the production tiles (both arithmetic modes): psi and
    sampled columns of U against the fsv restatement."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    s = B200UnitarySimulator(gemm_mode=native.GEMM_4M if mode == "4m" else native.GEMM_3M)
    c, reg = q.make_named_circuit("qft", 12)
    flat = native.flatten(c, reg)
    ur, ui = s.build_unitary(flat)
    for col in (0, 1, 777, 4095):
        cr, ci = orc.unitary_column(flat, col)
        assert rel_frob(ur[:, col], ui[:, col], cr, ci) <= TOL
    # QFT == DFT: U[j, k] = exp(2 pi i jk / N) / sqrt(N)
    N = 1 << 12
    j = np.arange(N)[:, None]
    k = np.arange(0, N, 97)[None, :]
    dft = np.exp(2j * np.pi * ((j * k) % N) / N) / np.sqrt(N)
    assert rel_frob(ur[:, ::97], ui[:, ::97], dft.real, dft.imag) <= TOL
    s.close()


@pytest.mark.parametrize("tile", [3, 4, 5])
def test_random_circuits_through_warp_specialised_tiles(monkeypatch, golden, sim, orc, tile):
    """The production K2 (warp-specialised, tile-prefix operator generation)
    on every golden random circuit it can tile (n >= 6), against the reference."""
    monkeypatch.setenv("QSB_TILE", str(tile))
    checked = 0
    for suite in ("cross", "det", "fsv", "norm"):
        for case in golden.suites[suite]:
            flat = golden.flat(case)
            if flat.n_qubits < 6 or (tile == 3 and flat.n_qubits < 7):  # tile rows: 4M 128, 3M 64
                continue
            out = sim.simulate_full_state(flat)
            re, im = golden.psi(case)
            assert rel_frob(out.re, out.im, re, im) <= TOL, (case, tile)
            checked += 1
    assert checked > 40


def test_layer_entries_through_tiles_bit_exact(monkeypatch, sim, orc):
    """Every K2 product here multiplies by a permutation, so the 4M path must
    reproduce the reference bit-for-bit: U = X(1) CNOT(0,n-1) L with L a mixed
    single-layer step. Row form: V = X[rows]; V <- V*CNOT; V <- V*L, and V*L
    picks exactly one generated entry of L per output (1*x + 0*y + ... = x),
    so K2's tile-prefix operator generation is checked entry by entry."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    monkeypatch.setenv("QSB_TILE", "3")
    for n in (7, 8, 9, 10):
        c = q.Circuit(n)
        c.h(1).t(0).cr(0.3, n - 1, 2)   # step 0: one layer, CR spans qubits 2..n-1
        c.cnot(0, n - 1).x(1)           # step 1: two permutation layers
        flat = native.flatten(c)
        ur, ui = sim.build_unitary(flat)
        orr, ori = orc.circuit_unitary(flat)
        assert np.array_equal(ur, orr) and np.array_equal(ui, ori), n


@pytest.mark.parametrize("mode", ["4m", "3m"])
def test_host_api_row_blocks_over_devices(monkeypatch, golden, orc, mode):
    """qsb_options.devices: the host API shards U by row blocks over the listed
    devices (repeats = virtual shards on one GPU); psi and U rows land at their
    host offsets. 4M results are bit-identical to one device (same k order);
    3M within 1e-10."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    monkeypatch.setenv("QSB_SPLITK", "1")  # bit-identity needs one summation order for every shard size
    gm = native.GEMM_4M if mode == "4m" else native.GEMM_3M
    one = B200UnitarySimulator(gemm_mode=gm)
    for G in (2, 4, 8):
        many = B200UnitarySimulator(gemm_mode=gm, devices=[0] * G)
        for name, n in [("qft", 9), ("deutsch-jozsa", 10), ("entangle", 8), ("qft", 5)]:
            c, reg = q.make_named_circuit(name, n)
            flat = native.flatten(c, reg)
            a = one.simulate_full_state(flat)
            b = many.simulate_full_state(flat)
            if mode == "4m":
                assert np.array_equal(a.re, b.re) and np.array_equal(a.im, b.im), (name, n, G)
            assert rel_frob(b.re, b.im, a.re, a.im) <= TOL
            ua = one.build_unitary(flat)
            ub = many.build_unitary(flat)
            assert rel_frob(ub[0], ub[1], ua[0], ua[1]) <= TOL
        many.close()
    one.close()


@pytest.mark.parametrize("splits", ["1", "2", "4", "8"])
@pytest.mark.parametrize("tile", ["3", "5"])
@pytest.mark.parametrize("name,n", [("qft", 10), ("entangle", 10), ("deutsch-jozsa", 10), ("qft", 11)])
def test_cluster_split_k(monkeypatch, sim, orc, splits, tile, name, n):
    """K2 split-K over a thread-block cluster (partials summed through DSMEM in
    rank order): within 1e-10 of the fsv restatement, and deterministic."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    monkeypatch.setenv("QSB_SPLITK", splits)
    monkeypatch.setenv("QSB_TILE", tile)
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    plan = sim.plan(flat)
    assert plan.info.gemm_splits == int(splits) and plan.info.gemm_tile == int(tile)
    plan.close()
    a = sim.build_unitary(flat)
    b = sim.build_unitary(flat)
    assert bit_equal(a[0], b[0]) and bit_equal(a[1], b[1])
    for col in (0, 5, (1 << n) - 1):
        cr, ci = orc.unitary_column(flat, col)
        assert rel_frob(a[0][:, col], a[1][:, col], cr, ci) <= TOL
    out = sim.simulate_full_state(flat)
    re, im = orc.fsv(flat)
    assert rel_frob(out.re, out.im, re, im) <= TOL


def test_split_k_chosen_for_small_grids(sim):
    """Small grids take their parallelism from the K split (N = 512: 64 tiles x 2
    ranks); grids of at least one wave run stream-K (gemm_splits -1); N <= 64 runs
    row-resident in one launch."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit("qft", 9)
    plan = sim.plan(native.flatten(c, reg))
    assert plan.info.gemm_splits == 2 and plan.info.gemm_tile == 5
    plan.close()
    c, reg = q.make_named_circuit("qft", 6)
    plan = sim.plan(native.flatten(c, reg))
    assert plan.info.gemm_tile == -1 and plan.info.n_launches == 1
    plan.close()
    c, reg = q.make_named_circuit("qft", 12)
    plan = sim.plan(native.flatten(c, reg))
    assert plan.info.gemm_splits == -1
    plan.close()


@pytest.mark.parametrize("dense", [False, True])
def test_registry_table_layouts(monkeypatch, golden, sim, dense):
    """Registered matrices reach the generator compactly (per-row column + value
    when every row has one nonzero, e.g. DJ oracles) or as dense tables
    (QSB_DENSE_TABLES): identical operator entries, same results."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    if dense:
        monkeypatch.setenv("QSB_DENSE_TABLES", "1")
    for case in [c for c in golden.cases if c.startswith("dj")]:
        flat = golden.flat(case)
        out = sim.simulate_full_state(flat)
        re, im = golden.psi(case)
        assert rel_frob(out.re, out.im, re, im) <= TOL, case
        steps = golden.steps(case)
        for st, (sr, si) in enumerate(steps):
            from paper_2305_14398_b200.simulator import step_layer_count

            if step_layer_count(flat, None, st) == 1:
                lr, li = sim.layer_operator(flat, None, st, 0)
                assert bit_equal(lr, sr) and bit_equal(li, si), (case, st)
    rng = np.random.default_rng(3)
    for n in (9, 11):
        for spec in ["balanced-mask:5", "constant1"]:
            c, reg = q.make_named_circuit("deutsch-jozsa", n, spec)
            flat = native.flatten(c, reg)
            ur, ui = sim.build_unitary(flat)
            for col in rng.choice(1 << n, 3, replace=False):
                cr, ci = orc_col(flat, int(col))
                assert rel_frob(ur[:, col], ui[:, col], cr, ci) <= TOL


def orc_col(flat, col):
    import oracle

    return oracle.Oracle().unitary_column(flat, col)


@pytest.mark.parametrize("name,n", [("qft", 10), ("entangle", 10), ("deutsch-jozsa", 10), ("qft", 11)])
def test_monomial_tiles_match_general_generator(monkeypatch, sim, name, n):
    """Monomial layers (CR, CNOT, X, DJ oracle) are generated as zeros plus one
    nonzero per operator row; the operator entries are the same bits as the
    general generator's, so U is bit-identical with QSB_NO_MONOMIAL."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    for tile in ("3", "5"):
        monkeypatch.setenv("QSB_TILE", tile)
        monkeypatch.delenv("QSB_NO_MONOMIAL", raising=False)
        a = sim.build_unitary(flat)
        monkeypatch.setenv("QSB_NO_MONOMIAL", "1")
        b = sim.build_unitary(flat)
        assert bit_equal(a[0], b[0]) and bit_equal(a[1], b[1]), tile


@pytest.mark.parametrize("tile", ["3", "4", "5"])
@pytest.mark.parametrize("name,n", [("deutsch-jozsa", 10), ("qft", 10), ("entangle", 9)])
def test_materialised_operator_matches_generated(monkeypatch, sim, orc, tile, name, n):
    """A layer materialised by K1t (transposed planes) and streamed to K2 by TMA
    carries the same operator bits as the shared-memory generator: U is
    bit-identical (== semantics) with every layer generated, and matches the oracle."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    monkeypatch.setenv("QSB_TILE", tile)
    monkeypatch.setenv("QSB_SPLITK", "1")
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    monkeypatch.setenv("QSB_MATERIALIZE", "1")
    plan = sim.plan(flat)
    assert plan.info.n_launches == 2 + 2 * plan.info.n_gemms
    plan.close()
    a = sim.build_unitary(flat)
    monkeypatch.setenv("QSB_MATERIALIZE", "0")
    b = sim.build_unitary(flat)
    assert bit_equal(a[0], b[0]) and bit_equal(a[1], b[1])
    for col in (0, (1 << n) - 1):
        cr, ci = orc.unitary_column(flat, col)
        assert rel_frob(a[0][:, col], a[1][:, col], cr, ci) <= TOL


def test_materialise_flag_and_dense_layer_choice(sim, orc):
    """QSB_FLAG_MATERIALIZE materialises every layer; by default only dense,
    non-monomial layers are (DJ's H on every qubit)."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    c, reg = q.make_named_circuit("deutsch-jozsa", 11)
    flat = native.flatten(c, reg)
    plan = sim.plan(flat)
    assert plan.info.n_launches == 2 + plan.info.n_gemms + 1  # one layer (X + H on 10 qubits) materialised
    plan.close()
    mat = B200UnitarySimulator(flags=native.FLAG_MATERIALIZE)
    plan = mat.plan(flat)
    assert plan.info.n_launches == 2 + 2 * plan.info.n_gemms
    plan.close()
    a = mat.simulate_full_state(flat)
    b = sim.simulate_full_state(flat)
    assert rel_frob(a.re, a.im, b.re, b.im) <= TOL
    re, im = orc.fsv(flat)
    assert rel_frob(a.re, a.im, re, im) <= TOL
    mat.close()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_single_layer_and_tiny_circuits(sim, orc, n):
    """One-layer and few-layer circuits through the one-CTA path (N <= 32) and
    the first tiled sizes: every gate kind, controls above / below targets."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    rng = np.random.default_rng(n)
    gates = [q.GateType.h(), q.GateType.x(), q.GateType.y(), q.GateType.z(), q.GateType.s(), q.GateType.t(),
             q.GateType.r(0.3)]
    for trial in range(40):
        c = q.Circuit(n)
        for _ in range(1 + trial % 4):
            g = gates[rng.integers(len(gates))]
            if n > 1 and rng.random() < 0.5:
                a, b = rng.choice(n, 2, replace=False)
                c.add_control_gate(g, int(a), int(b))
            else:
                c.add_gate(g, int(rng.integers(n)))
        flat = native.flatten(c, None)
        out = sim.simulate_full_state(flat)
        re, im = orc.unitary_simulate(flat, guard=n)
        assert rel_frob(out.re, out.im, re, im) <= TOL, (n, trial)
        ur, ui = sim.build_unitary(flat)
        orr, ori = orc.circuit_unitary(flat)
        assert rel_frob(ur, ui, orr, ori) <= TOL, (n, trial)


@pytest.mark.parametrize("name,n", [("deutsch-jozsa", 11), ("entangle", 10), ("qft", 10)])
def test_real_layers_as_two_real_gemms(monkeypatch, sim, orc, name, n):
    """Layers with an exactly-zero imaginary plane (H, X, CNOT, DJ oracle) run as
    two real GEMMs on the 3M tiles; U matches the full-3M run and the oracle."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    a = sim.build_unitary(flat)
    monkeypatch.setenv("QSB_NO_REAL", "1")
    b = sim.build_unitary(flat)
    assert rel_frob(a[0], a[1], b[0], b[1]) <= TOL
    for col in (0, 3, (1 << n) - 1):
        cr, ci = orc.unitary_column(flat, col)
        assert rel_frob(a[0][:, col], a[1][:, col], cr, ci) <= TOL


def test_concurrent_host_calls_on_one_handle(golden):
    """simulate_full_state is const and reentrant (simulator.hpp:44-45): calls from
    several host threads on one handle serialise internally and stay correct."""
    import threading

    from paper_2305_14398_b200.simulator import (B200FsvSimulator, B200StructuredUnitarySimulator,
                                                 B200UnitarySimulator)

    cases = ["qft9", "dj9", "entangle10", "qft5", "edge_wide_span"] + golden.suites["cross"][:10]
    # the npz archive is not thread-safe: load every input and expectation up front
    data = {case: (golden.flat(case), golden.psi(case)) for case in cases}
    for cls in (B200UnitarySimulator, B200StructuredUnitarySimulator, B200FsvSimulator):
        s = cls()
        errors = []

        def worker(k):
            try:
                for case in cases[k::3] * 3:
                    flat, (re, im) = data[case]
                    out = s.simulate_full_state(flat)
                    if rel_frob(out.re, out.im, re, im) > TOL:
                        errors.append((cls.__name__, case))
            except Exception as e:  # noqa: BLE001
                errors.append((cls.__name__, repr(e)))

        threads = [threading.Thread(target=worker, args=(k,)) for k in range(3)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        s.close()
        assert not errors, errors[:3]


def test_qft14_row_shard_matches_dft(sim):
    """The north-star size: rows [0, N/8) of the QFT-14 unitary (one rank's
    shard of the 8-GPU decomposition, 16384 x 2048 complex) equal the DFT
    matrix within 1e-10 relative (QFT == DFT: test_circuit_library.cpp:161-167,
    acceptance_main.cpp:173-180)."""
    import torch

    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import torch_view

    n = 14
    N = 1 << n
    rows = N // 8
    c, reg = q.make_named_circuit("qft", n)
    plan = sim.plan(native.flatten(c, reg), None, 0, rows)
    plan.execute()
    torch.cuda.synchronize()
    re_p, im_p = plan.unitary_device()
    ur = torch_view(re_p, (rows, N))
    ui = torch_view(im_p, (rows, N))
    j = torch.arange(rows, device=ur.device, dtype=torch.int64)[:, None]
    k = torch.arange(N, device=ur.device, dtype=torch.int64)[None, :]
    ang = (2.0 * np.pi / N) * ((j * k) % N).to(torch.float64)
    dr = torch.cos(ang) / np.sqrt(N)
    di = torch.sin(ang) / np.sqrt(N)
    num = torch.sqrt(((ur - dr) ** 2 + (ui - di) ** 2).sum()).item()
    den = torch.sqrt((dr ** 2 + di ** 2).sum()).item()
    plan.close()
    assert num / den <= TOL, num / den


def test_hbm_limit_plans_fall_back_to_two_planes(sim):
    """QFT-16 (65536^2): two 3-plane V buffers (206 GB) do not fit a B200, so the
    plan keeps re/im planes only (in-register 3M sums) and generates every
    operator instead of materialising (memory_estimate / guard:
    unitary_backend.cpp:156-192)."""
    import torch

    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    free, _ = torch.cuda.mem_get_info()
    if free < 150e9:
        pytest.skip("needs ~140 GB of free HBM")
    c, reg = q.make_named_circuit("qft", 16)
    plan = sim.plan(native.flatten(c, reg))
    assert plan.info.v_planes == 2 and plan.info.gemm_tile == 4
    assert plan.info.n_launches == 2 + plan.info.n_gemms  # no K1t launches
    plan.close()
    c, reg = q.make_named_circuit("qft", 17)
    with pytest.raises(q.ResourceError, match="refuses 17 qubits"):
        sim.simulate_full_state(c, reg)


@pytest.mark.parametrize("tile", ["3", "4", "5"])
@pytest.mark.parametrize("name,n", [("entangle", 10), ("qft", 10), ("deutsch-jozsa", 11), ("qft", 11)])
def test_stream_k_schedule(monkeypatch, sim, orc, tile, name, n):
    """Stream-K (persistent CTAs sharing the tile x k-tile iterations; a split
    tile's owner adds the published partials in k order): deterministic, within
    1e-10 of the oracle and of the whole-tile schedule."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    monkeypatch.setenv("QSB_TILE", tile)
    monkeypatch.setenv("QSB_STREAMK", "1")
    plan = sim.plan(flat)
    assert plan.info.gemm_splits == -1
    plan.close()
    a = sim.build_unitary(flat)
    for _ in range(3):
        b = sim.build_unitary(flat)
        assert bit_equal(a[0], b[0]) and bit_equal(a[1], b[1])
    monkeypatch.setenv("QSB_STREAMK", "0")
    ref = sim.build_unitary(flat)
    assert rel_frob(a[0], a[1], ref[0], ref[1]) <= TOL
    for col in (0, (1 << n) - 1):
        cr, ci = orc.unitary_column(flat, col)
        assert rel_frob(a[0][:, col], a[1][:, col], cr, ci) <= TOL


def test_stream_k_chosen_where_waves_quantise(sim):
    """Grids of at least one wave run stream-K (Entangle-10: 256 tiles on 148 SMs,
    QFT-12: 4096 tiles); QFT-9 (64 tiles) keeps the cluster split-K grid."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit("entangle", 10)
    plan = sim.plan(native.flatten(c, reg))
    assert plan.info.gemm_splits == -1
    plan.close()
    c, reg = q.make_named_circuit("qft", 12)
    plan = sim.plan(native.flatten(c, reg))
    assert plan.info.gemm_splits == -1
    plan.close()
    c, reg = q.make_named_circuit("qft", 9)
    plan = sim.plan(native.flatten(c, reg))
    assert plan.info.gemm_splits == 2
    plan.close()


def test_stage_release_regression(monkeypatch, sim):
    """H^n H^n = I through one materialised real GEMM under stream-K, repeated:
    every run bit-identical and within 1e-12 of I. Before stages were released
    after a block boundary, a consumer warp's last shared load could be
    overwritten by the producer's TMA refill (one wrong k-tile, ~30 % of runs)."""
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.circuit import Circuit, GateRegistry

    n = 11
    c = Circuit(n)
    for _ in range(2):
        for k in range(n):
            c.h(k)
    flat = native.flatten(c, GateRegistry())
    monkeypatch.setenv("QSB_TILE", "5")
    monkeypatch.setenv("QSB_STREAMK", "1")
    first = sim.build_unitary(flat)
    assert np.abs(first[0] - np.eye(1 << n)).max() < 1e-12 and np.abs(first[1]).max() < 1e-12
    for _ in range(15):
        u = sim.build_unitary(flat)
        assert bit_equal(u[0], first[0]) and bit_equal(u[1], first[1])


@pytest.mark.parametrize("G", [1, 2, 4])
def test_column_blocks(orc, G):
    """QSB_FLAG_COLUMN_BLOCKS: U[:, cols] <- S_k U[:, cols] in
    application order — the reference's own association — sharded by column
    blocks; psi is the sum of the shards' shares. U and psi within 1e-10 of the
    row-block form and of the oracle; general psi0 and the collapse path too."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    rows = B200UnitarySimulator()
    cols = B200UnitarySimulator(flags=native.FLAG_COLUMN_BLOCKS, devices=[0] * G if G > 1 else None)
    rng = np.random.default_rng(808)
    for name, n in [("qft", 4), ("qft", 6), ("qft", 7), ("entangle", 8), ("deutsch-jozsa", 9), ("qft", 10)]:
        c, reg = q.make_named_circuit(name, n)
        flat = native.flatten(c, reg)
        N = 1 << n
        ua = rows.build_unitary(flat)
        ub = cols.build_unitary(flat)
        assert rel_frob(ub[0], ub[1], ua[0], ua[1]) <= TOL, (name, n, G)
        for col in (0, N - 1):
            cr, ci = orc.unitary_column(flat, col)
            assert rel_frob(ub[0][:, col], ub[1][:, col], cr, ci) <= TOL
        a = rows.simulate_full_state(flat)
        b = cols.simulate_full_state(flat)
        assert rel_frob(b.re, b.im, a.re, a.im) <= TOL
        x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        x /= np.linalg.norm(x)
        a = rows.simulate_from_state(flat, None, x.real.copy(), x.imag.copy())
        b = cols.simulate_from_state(flat, None, x.real.copy(), x.imag.copy())
        assert rel_frob(b.re, b.im, a.re, a.im) <= TOL
    cols.close()
    rows.close()


@pytest.mark.parametrize("name,n", [("qft", 7), ("qft", 8), ("entangle", 7), ("entangle", 8),
                                    ("deutsch-jozsa", 7), ("deutsch-jozsa", 8)])
def test_mid_cluster_chain(monkeypatch, sim, orc, name, n):
    """K2m (N = 128, 256): the whole chain in one cluster launch. U within 1e-10
    of the K2 GEMM chain (QSB_NO_MID) and of the oracle's columns; psi from a
    general psi0; one launch per plan; row blocks over virtual devices."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    N = 1 << n
    plan = sim.plan(flat)
    if (name, n) == ("deutsch-jozsa", 8):  # dense H-on-every-qubit layers keep K2 at N = 256
        assert plan.info.gemm_tile >= 0 and plan.info.n_launches > 1
    else:
        assert plan.info.gemm_tile == -1 and plan.info.n_launches == 1
    plan.close()
    ur, ui = sim.build_unitary(flat)
    for col in (0, 3, N - 1):
        cr, ci = orc.unitary_column(flat, col)
        assert rel_frob(ur[:, col], ui[:, col], cr, ci) <= TOL
    x = np.random.default_rng(n).standard_normal(N) + 1j * np.random.default_rng(n + 1).standard_normal(N)
    x /= np.linalg.norm(x)
    got = sim.simulate_from_state(flat, None, x.real.copy(), x.imag.copy())
    want = (ur + 1j * ui) @ x
    assert rel_frob(got.re, got.im, want.real, want.imag) <= TOL
    monkeypatch.setenv("QSB_NO_MID", "1")
    kr, ki = sim.build_unitary(flat)
    assert rel_frob(ur, ui, kr, ki) <= TOL
    monkeypatch.delenv("QSB_NO_MID")
    multi = B200UnitarySimulator(devices=[0, 0, 0, 0])
    mr, mi = multi.build_unitary(flat)
    multi.close()
    if (name, n) == ("deutsch-jozsa", 8):  # K2: the split-K order depends on the shard height
        assert rel_frob(mr, mi, ur, ui) <= TOL
    else:  # K2m computes every row block alike
        assert bit_equal(mr, ur) and bit_equal(mi, ui)


def test_mid_cluster_chain_random_golden(golden, sim):
    """Every golden circuit of 7 or 8 qubits (63 recorded from the reference) through K2m."""
    seen = 0
    for case in golden.cases:
        if not golden.has(f"{case}:psi_re"):
            continue
        flat = golden.flat(case)
        if flat.n_qubits not in (7, 8):
            continue
        out = sim.simulate_full_state(flat)
        re, im = golden.psi(case)
        assert rel_frob(out.re, out.im, re, im) <= TOL, case
        seen += 1
    assert seen >= 60


@pytest.mark.parametrize("n", [5, 6, 7])
def test_small_k2m_matches_row_resident(monkeypatch, sim, orc, n):
    """N = 64 runs K2m (clusters of 2 CTAs, K over 8 warp groups; N = 32 keeps
    K2s); the K2s row-resident kernel (QSB_SMALL_CLASSIC) stays selectable. Both
    within 1e-10 of the oracle and of each other, for chains short enough to
    stage every descriptor in shared memory and long enough to need the ring."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    rng = np.random.default_rng(100 + n)
    gates = [q.GateType.h(), q.GateType.y(), q.GateType.s(), q.GateType.r(0.7), q.GateType.t()]
    circuits = [q.make_named_circuit(name, n) for name in ("qft", "entangle", "deutsch-jozsa")]
    for layers in (1, 5, 40, 600):
        c = q.Circuit(n)
        for _ in range(layers):
            g = gates[rng.integers(len(gates))]
            a, b = rng.choice(n, 2, replace=False)
            c.add_control_gate(g, int(a), int(b)) if rng.random() < 0.5 else c.add_gate(g, int(a))
        circuits.append((c, None))
    for c, reg in circuits:
        flat = native.flatten(c, reg)
        out = sim.simulate_full_state(flat)
        ur, ui = sim.build_unitary(flat)
        orr, ori = orc.circuit_unitary(flat)
        assert rel_frob(ur, ui, orr, ori) <= TOL
        re, im = orc.unitary_simulate(flat, guard=n)
        assert rel_frob(out.re, out.im, re, im) <= TOL
        # the other paths: K2s (N <= 64) or the K2 chain (N = 128), and K2m without
        # double-buffered operators
        for env in ("QSB_SMALL_CLASSIC" if n <= 6 else "QSB_NO_MID", "QSB_MID_NODBUF"):
            monkeypatch.setenv(env, "1")
            kr, ki = sim.build_unitary(flat)
            monkeypatch.delenv(env)
            assert rel_frob(ur, ui, kr, ki) <= TOL, env


@pytest.mark.parametrize("splits", ["", "1", "2", "4", "8"])
@pytest.mark.parametrize("name,n", [("qft", 9), ("entangle", 10), ("qft", 10), ("entangle", 9)])
def test_chain_kernel(monkeypatch, sim, orc, splits, name, n):
    """K2c (QSB_CHAIN=1): every GEMM of the chain in one persistent launch, dataflow
    between GEMMs by row block, real and complex layers mixed, k-split partials summed
    in a fixed order. psi and U against the oracle (1e-10), U against the per-GEMM
    path (1e-12), and bit-identical across repeated runs (deterministic)."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    per_gemm = sim.build_unitary(flat)
    monkeypatch.setenv("QSB_CHAIN", "1")
    if splits:
        monkeypatch.setenv("QSB_CHAIN_SPLITS", splits)
    s = B200UnitarySimulator(device=0)
    plan = s.plan(flat)
    assert plan.info.gemm_tile == 6 and plan.info.n_launches == 3, plan.info.gemm_tile
    if splits:
        assert plan.info.gemm_splits == int(splits)
    plan.close()
    a = s.build_unitary(flat)
    b = s.build_unitary(flat)
    out = s.simulate_full_state(flat)
    s.close()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert rel_frob(a[0], a[1], per_gemm[0], per_gemm[1]) <= 1e-12
    re, im = orc.fsv(flat)
    assert rel_frob(out.re, out.im, re, im) <= TOL
    for col in (0, 5, (1 << n) - 1):
        cr, ci = orc.unitary_column(flat, col)
        assert rel_frob(a[0][:, col], a[1][:, col], cr, ci) <= TOL


def test_chain_kernel_row_shards(monkeypatch, orc):
    """K2c on row shards (M < N): each shard's rows equal the full unitary's."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    monkeypatch.setenv("QSB_CHAIN", "1")
    c, reg = q.make_named_circuit("qft", 10)
    flat = native.flatten(c, reg)
    s = B200UnitarySimulator(devices=[0, 0, 0, 0])
    ur, ui = s.build_unitary(flat)
    psi = s.simulate_full_state(flat)
    s.close()
    re, im = orc.fsv(flat)
    assert rel_frob(psi.re, psi.im, re, im) <= TOL
    assert rel_frob(ur[:, 0], ui[:, 0], re, im) <= TOL


@pytest.mark.parametrize("parts", ["2", "4"])
@pytest.mark.parametrize("name,n", [("qft", 9), ("entangle", 10), ("deutsch-jozsa", 10), ("qft", 11)])
def test_row_block_parts(monkeypatch, sim, orc, parts, name, n):
    """QSB_PARTS: a plan's rows split into independent sub-plans whose chains run
    concurrently on one device (fork / join streams, captured in the plan's CUDA
    graph on reuse). psi, U (host API and the assembled device U) against the single
    plan (1e-12) and the oracle (1e-10); psi0 != |0...0>; timing API."""
    import torch

    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator, torch_view

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    N = 1 << n
    whole = sim.build_unitary(flat)
    monkeypatch.setenv("QSB_PARTS", parts)
    s = B200UnitarySimulator(device=0)
    u1 = s.build_unitary(flat)
    u2 = s.build_unitary(flat)  # the cached plan (graph of the fork / join)
    psi = s.simulate_full_state(flat)
    assert np.array_equal(u1[0], u2[0]) and np.array_equal(u1[1], u2[1])
    assert rel_frob(u1[0], u1[1], whole[0], whole[1]) <= 1e-12
    re, im = orc.fsv(flat)
    assert rel_frob(psi.re, psi.im, re, im) <= TOL
    rng = np.random.default_rng(n)
    v = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    v /= np.linalg.norm(v)
    gen = s.simulate_from_state(flat, None, v.real, v.imag)
    ore, oim = orc.fsv(flat, np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag))
    assert rel_frob(gen.re, gen.im, ore, oim) <= TOL
    # device plan: assembled U rows, psi rows, timing
    plan = s.plan(flat)
    plan.set_timing(True)
    plan.execute()
    total, chain, mean = plan.last_timing()
    assert total > 0 and chain > 0
    plan.set_timing(False)
    plan.execute()
    torch.cuda.synchronize()
    pr, pi = plan.unitary_device()
    ur = torch_view(pr, (N, N)).cpu().numpy()
    ui = torch_view(pi, (N, N)).cpu().numpy()
    assert rel_frob(ur, ui, whole[0], whole[1]) <= 1e-12
    dre = torch.empty(N, dtype=torch.float64, device="cuda")
    dim = torch.empty(N, dtype=torch.float64, device="cuda")
    plan.copy_state(dre.data_ptr(), dim.data_ptr())
    torch.cuda.synchronize()
    assert rel_frob(dre.cpu().numpy(), dim.cpu().numpy(), re, im) <= TOL
    plan.close()
    s.close()


@pytest.mark.parametrize("group", ["5", "16"])
@pytest.mark.parametrize("name,n", [("qft", 11), ("deutsch-jozsa", 11), ("entangle", 11)])
def test_grouped_tile_numbering(monkeypatch, sim, orc, group, name, n):
    """QSB_SK_GROUP: the data-parallel / stream-K tiles numbered group by group of row
    blocks (a short last group with 5) — U within 1e-12 of the row-major numbering,
    psi against the oracle."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    monkeypatch.setenv("QSB_SK_GROUP", "0")
    base = sim.build_unitary(flat)
    monkeypatch.setenv("QSB_SK_GROUP", group)
    s = B200UnitarySimulator(device=0)
    u = s.build_unitary(flat)
    psi = s.simulate_full_state(flat)
    s.close()
    assert rel_frob(u[0], u[1], base[0], base[1]) <= 1e-12
    re, im = orc.fsv(flat)
    assert rel_frob(psi.re, psi.im, re, im) <= TOL


@pytest.mark.parametrize("name,n", [("qft", 6), ("qft", 7), ("qft", 8), ("deutsch-jozsa", 7)])
def test_mid_cluster_chain_3m(monkeypatch, sim, orc, name, n):
    """K2m with complex layers as 3M (QSB_MID_3M=1: three DMMAs, sums in registers)
    against the 4M K2m (1e-12) and the oracle (1e-10)."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    monkeypatch.setenv("QSB_MID_3M", "0")
    a = sim.build_unitary(flat)
    monkeypatch.setenv("QSB_MID_3M", "1")
    b = sim.build_unitary(flat)
    psi = sim.simulate_full_state(flat)
    assert rel_frob(b[0], b[1], a[0], a[1]) <= 1e-12
    re, im = orc.fsv(flat)
    assert rel_frob(psi.re, psi.im, re, im) <= TOL


@pytest.mark.parametrize("name,n", [("qft", 10), ("qft", 11), ("deutsch-jozsa", 10)])
def test_materialised_zero_tiles_skipped(monkeypatch, sim, orc, name, n):
    """Materialised operands: structurally zero B tiles are cleared in shared memory
    instead of loaded — bit-identical U to loading every tile (QSB_MATB_DENSE=1),
    with every layer materialised as well as with the default choice."""
    import paper_2305_14398_b200 as q
    from paper_2305_14398_b200 import native

    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    for mat in (None, "1"):
        if mat:
            monkeypatch.setenv("QSB_MATERIALIZE", mat)
        monkeypatch.setenv("QSB_MATB_DENSE", "1")
        dense = sim.build_unitary(flat)
        monkeypatch.delenv("QSB_MATB_DENSE")
        skip = sim.build_unitary(flat)
        assert bit_equal(skip[0], dense[0]) and bit_equal(skip[1], dense[1])
    re, im = orc.fsv(flat)
    assert rel_frob(skip[0][:, 0], skip[1][:, 0], re, im) <= TOL
