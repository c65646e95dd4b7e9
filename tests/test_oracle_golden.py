"""Pins the C oracle (oracle/qsim_oracle.c) to golden vectors recorded from the
unmodified reference library (tests/golden/make_golden.py). CPU only.

The oracle restates the reference's arithmetic operation for operation with no
FMA contraction, so it must reproduce the reference BIT-EXACTLY.
"""
import numpy as np
import pytest

from conftest import bit_equal


def test_every_case_state_bit_exact(golden, orc):
    for case in golden.cases:
        flat = golden.flat(case)
        if flat.n_qubits > 8:
            continue
        re, im = orc.unitary_simulate(flat, guard=flat.n_qubits)
        gr, gi = golden.psi(case)
        assert bit_equal(re, gr) and bit_equal(im, gi), case


def test_every_case_unitary_bit_exact(golden, orc):
    n = 0
    for case in golden.cases:
        u = golden.unitary(case)
        if u is None:
            continue
        re, im = orc.circuit_unitary(golden.flat(case))
        assert bit_equal(re, u[0]) and bit_equal(im, u[1]), case
        n += 1
    assert n > 150


def test_step_unitaries_bit_exact(golden, orc):
    n = 0
    for case in golden.cases:
        steps = golden.steps(case)
        flat = golden.flat(case) if steps else None
        for s, (sr, si) in enumerate(steps):
            re, im = orc.step_unitary(flat, s)
            assert bit_equal(re, sr) and bit_equal(im, si), (case, s)
            n += 1
    assert n > 100


def test_single_layer_steps_equal_layer_operator(golden, orc):
    for case in golden.cases:
        steps = golden.steps(case)
        if not steps:
            continue
        flat = golden.flat(case)
        for s, (sr, si) in enumerate(steps):
            nl, _ = orc.step_layers(flat, s)
            if nl == 1:
                re, im = orc.layer_operator(flat, s, 0)
                assert bit_equal(re, sr) and bit_equal(im, si)


def test_multilayer_steps_exist_and_factor(golden, orc):
    """QFT packs H(k+1) inside the CR(n-1 -> k) span: the
    first-fit layering must split those steps (unitary_backend.cpp:63-91)."""
    flat = golden.flat("qft4")
    layers = [orc.step_layers(flat, s)[0] for s in range(len(flat.step_offsets) - 1)]
    assert sum(layers) == 16 and len(layers) == 13
    flat = golden.flat("edge_span_overlap")
    assert orc.step_layers(flat, 0) == (2, [0, 1])


def test_large_named_states(golden, orc):
    """n = 9, 10: oracle (fsv restatement) within 1e-12 of the reference unitary path."""
    for case in ["qft9", "entangle9", "entangle10", "dj9"]:
        flat = golden.flat(case)
        re, im = orc.fsv(flat)
        gr, gi = golden.psi(case)
        assert np.max(np.hypot(re - gr, im - gi)) < 1e-12, case


def test_fsv_restatement_agrees(golden, orc):
    for case in golden.suites["cross"][:80]:
        flat = golden.flat(case)
        re, im = orc.fsv(flat)
        gr, gi = golden.psi(case)
        assert np.max(np.hypot(re - gr, im - gi)) < 1e-9


def test_splitmix_and_collapse(golden, orc):
    for seed, bits in enumerate(golden["splitmix_bits"]):
        assert np.float64(orc.splitmix64_unit(seed)).view(np.uint64) == bits
    for seed, bits in enumerate(golden["splitmix_bits_3"]):
        assert np.float64(orc.splitmix64_unit(seed, 3)).view(np.uint64) == bits
    re, im = golden.psi("bell")
    for seed, want in enumerate(golden["collapse_bell"]):
        assert orc.collapse(re, im, seed) == want
    re, im = golden.psi("qft5")
    for seed, want in enumerate(golden["collapse_qft5"]):
        assert orc.collapse(re, im, seed) == want
    for key in ["comp_0", "comp_1"]:
        re, im = golden[f"{key}:state_re"], golden[f"{key}:state_im"]
        assert bit_equal(orc.probabilities(re, im), golden[f"{key}:probs"])
        assert orc.norm_squared(re, im) == float(golden[f"{key}:norm"])
        for seed, want in enumerate(golden[f"{key}:collapse"]):
            assert orc.collapse(re, im, seed) == want


def test_memory_accounting(golden, orc):
    for n in range(1, 31):
        assert orc.memory_estimate(n, 0) == golden["mem_unitary"][n - 1]
        assert orc.memory_estimate(n, 1) == golden["mem_fsv"][n - 1]
    for n in range(1, 30):
        assert orc.engine_memory_estimate(n, 0) == golden["engine_unitary"][n - 1]
    for b, s in golden.index["format_bytes"]:
        assert orc.format_bytes(int(b)) == s


def test_guard_and_reset_errors(golden, orc):
    import oracle

    flat = golden.flat("qft5")
    with pytest.raises(oracle.OracleError) as e:
        orc.unitary_simulate(flat, guard=4)
    assert e.value.code == 1 and "estimated memory 8448 bytes" in str(e.value)


def test_gate_and_controlled_kats(orc):
    """test_gates.cpp:40-107 known answers."""
    s = np.sqrt(0.5)
    assert bit_equal(orc.gate_matrix(0), np.array([[s, s], [s, -s]], dtype=complex))
    assert bit_equal(orc.gate_matrix(1), np.array([[0, 1], [1, 0]], dtype=complex))
    assert bit_equal(orc.gate_matrix(2), np.array([[0, -1j], [1j, 0]]))
    cx = orc.controlled_unitary(orc.gate_matrix(1), 0, 1, 2)
    assert bit_equal(cx, np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex))
    m = orc.controlled_unitary(orc.gate_matrix(1), 1, 0, 2)
    assert m[0, 0] == 1 and m[3, 1] == 1 and m[2, 2] == 1 and m[1, 3] == 1 and m.sum() == 4
    # brute-force permutation oracle, spans 2..3 (acceptance_main.cpp:133-168)
    for span in (2, 3):
        dim = 1 << span
        for c in range(span):
            for t in range(span):
                if c == t:
                    continue
                m = orc.controlled_unitary(orc.gate_matrix(1), c, t, span)
                cm, tm = 1 << (span - 1 - c), 1 << (span - 1 - t)
                want = np.zeros((dim, dim), dtype=complex)
                for col in range(dim):
                    want[col ^ tm if col & cm else col, col] = 1
                assert bit_equal(m, want)


def test_matmul_matches_naive(orc):
    """test_linalg.cpp:74-81: matmul vs std::complex naive at 1e-12."""
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (7, 5)) + 1j * rng.uniform(-1, 1, (7, 5))
    b = rng.uniform(-1, 1, (5, 3)) + 1j * rng.uniform(-1, 1, (5, 3))
    assert np.max(np.abs(orc.matmul(a, b) - a @ b)) <= 1e-12
    h = orc.gate_matrix(0)
    assert bit_equal(orc.kronecker(h, np.eye(2, dtype=complex)),
                     np.kron(h, np.eye(2)))


def test_fsv_restatement_bit_exact_with_reference_fsv(golden, orc):
    """The C oracle's fsv (fsv_backend.cpp:40-158 restated) reproduces the
    reference's own FsvSimulator output bit for bit on every recorded circuit,
    including the multi-slab sizes (n = 13..15)."""
    checked = 0
    for case in golden.cases:
        if not golden.has(f"{case}:fsv_re"):
            continue
        re, im = orc.fsv(golden.flat(case))
        assert bit_equal(re, golden[f"{case}:fsv_re"]) and bit_equal(im, golden[f"{case}:fsv_im"]), case
        checked += 1
    assert checked >= 340
