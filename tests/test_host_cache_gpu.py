"""The host-API plan cache (run_bench calls one circuit 51
times, bench.cpp:95-105): a call with the same circuit structure reuses the last
call's compiled plans, uploaded tables and buffers, and checks the registry
matrices' contents against kept copies while the GPU runs. Results must be those
of a fresh handle in every case, including a registry matrix that changed under
an identical structure."""
import numpy as np
import pytest

import paper_2305_14398_b200 as q
from paper_2305_14398_b200 import native
from paper_2305_14398_b200.simulator import B200UnitarySimulator

pytestmark = pytest.mark.gpu


def fresh(flat, **kw):
    s = B200UnitarySimulator(device=0, **kw)
    out = s.simulate_full_state(flat)
    s.close()
    return out


@pytest.mark.parametrize("name,n", [("qft", 4), ("qft", 7), ("deutsch-jozsa", 8), ("qft", 10), ("deutsch-jozsa", 11)])
def test_repeated_calls_identical(name, n):
    c, reg = q.make_named_circuit(name, n)
    flat = native.flatten(c, reg)
    want = fresh(flat)
    s = B200UnitarySimulator(device=0)
    for _ in range(4):
        out = s.simulate_full_state(flat)
        assert np.array_equal(out.re, want.re) and np.array_equal(out.im, want.im)
    s.close()


@pytest.mark.parametrize("n", [5, 9, 11])
def test_changed_registry_matrix_is_detected(orc, n):
    """Same ops, same function dimension, different oracle contents: the reused
    plan's result is discarded and the call is redone from the new matrix."""
    s = B200UnitarySimulator(device=0)
    for spec in ("balanced-bit:0", "constant0", "balanced-bit:1", "constant1", "balanced-bit:0"):
        c, reg = q.make_named_circuit("deutsch-jozsa", n, spec)
        flat = native.flatten(c, reg)
        out = s.simulate_full_state(flat)
        re, im = orc.fsv(flat)
        err = np.sqrt(np.sum((out.re - re) ** 2 + (out.im - im) ** 2))
        assert err <= 1e-10, (spec, err)
    s.close()


def test_in_place_mutation_of_registry_matrix(orc):
    """The caller's matrix storage itself is edited between two calls (same pointers)."""
    c, reg = q.make_named_circuit("deutsch-jozsa", 6, "balanced-bit:0")
    flat = native.flatten(c, reg)
    s = B200UnitarySimulator(device=0)
    a = s.simulate_full_state(flat)
    re0, im0 = flat.fn_planes[0]
    re0[:] = np.eye(re0.shape[0])[::-1]  # another permutation, written in place
    b = s.simulate_full_state(flat)
    want_re, want_im = orc.fsv(flat)
    assert np.allclose(b.re, want_re, atol=1e-12) and np.allclose(b.im, want_im, atol=1e-12)
    assert not np.array_equal(a.re, b.re)
    s.close()


@pytest.mark.parametrize("n", [4, 8, 10])
def test_initial_state_then_zero_state_on_cached_plan(orc, n):
    c, reg = q.make_named_circuit("qft", n)
    flat = native.flatten(c, reg)
    rng = np.random.default_rng(n)
    N = 1 << n
    v = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    v /= np.linalg.norm(v)
    s = B200UnitarySimulator(device=0)
    zero = s.simulate_full_state(flat)
    gen = s.simulate_from_state(flat, None, v.real, v.imag)
    zero2 = s.simulate_full_state(flat)
    assert np.array_equal(zero.re, zero2.re) and np.array_equal(zero.im, zero2.im)
    ore, oim = orc.fsv(flat, np.ascontiguousarray(v.real), np.ascontiguousarray(v.imag))
    assert np.sqrt(np.sum((gen.re - ore) ** 2 + (gen.im - oim) ** 2)) <= 1e-10
    ur, ui = s.build_unitary(flat)  # same plan, U downloaded instead of psi
    assert np.array_equal(ur[:, 0], zero.re) and np.array_equal(ui[:, 0], zero.im)
    s.close()


def test_other_paths_drop_the_cache(orc):
    """fsv / structured / layer_operator / is_unitary calls on the same handle free the
    kept dense plan first; the next dense call rebuilds it correctly."""
    from paper_2305_14398_b200.simulator import is_unitary

    c, reg = q.make_named_circuit("qft", 9)
    flat = native.flatten(c, reg)
    s = B200UnitarySimulator(device=0)
    a = s.simulate_full_state(flat)
    s.layer_operator(flat, None, 0, 0)
    ok, _ = is_unitary(s, np.eye(64), 1e-9)
    assert ok
    b = s.simulate_full_state(flat)
    assert np.array_equal(a.re, b.re) and np.array_equal(a.im, b.im)
    s.close()


def test_plan_switch_change_is_a_new_plan():
    """A QSB_* plan-time switch changed between calls must not reuse a plan built
    under the old setting (the cache key carries the QSB_* environment), and a
    QSB_FLAG_NO_PLAN_CACHE handle compiles every call (the bench's cold e2e)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import os, sys; sys.path.insert(0, %r)\n"
        "import paper_2305_14398_b200 as q\n"
        "from paper_2305_14398_b200 import native\n"
        "from paper_2305_14398_b200.simulator import B200UnitarySimulator\n"
        "c, reg = q.make_named_circuit('qft', 9); f = native.flatten(c, reg)\n"
        "s = B200UnitarySimulator(device=0)\n"
        "s.simulate_full_state(f); s.simulate_full_state(f)\n"
        "os.environ['QSB_SPLITK'] = '4'\n"
        "s.simulate_full_state(f); s.simulate_full_state(f)\n"
        "s.close()\n"
        "cold = B200UnitarySimulator(device=0, flags=native.FLAG_NO_PLAN_CACHE)\n"
        "cold.simulate_full_state(f); cold.simulate_full_state(f)\n"
        "cold.close()\n" % root)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, QSB_TRACE="1"))
    assert r.returncode == 0, r.stderr
    kinds = [ln.split()[3] for ln in r.stderr.splitlines() if ln.startswith("qsb trace:")]
    assert kinds == ["new", "cached", "new", "cached", "new", "new"], r.stderr
