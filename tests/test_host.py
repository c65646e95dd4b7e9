"""CPU-only tests of the host side: the reference-interface mirror (circuit
model, packing, gate library, generators), the ABI flattening, the C-ABI
library (loads, exports every symbol of include/qsb.h, host-only entry points)
— no GPU compute calls."""
import ctypes
import subprocess

import numpy as np
import pytest

import paper_2305_14398_b200 as q
from paper_2305_14398_b200 import native
from conftest import bit_equal

NAMED = [("qft", n, f"qft{n}") for n in range(1, 10)] + \
        [("entangle", n, f"entangle{n}") for n in range(2, 11)] + \
        [("deutsch-jozsa", n, f"dj{n}") for n in range(2, 10)] + [("bell", 2, "bell")]


# ---- circuit model (test_circuit.cpp:62-121) ----

def test_new_circuits_bounded():
    assert q.Circuit(1).steps() == []
    assert q.Circuit(2).qubit_count() == 2
    with pytest.raises(q.ArgumentError):
        q.Circuit(0)
    with pytest.raises(q.ArgumentError):
        q.Circuit(25)
    assert q.Circuit(25, 30).qubit_count() == 25


def test_greedy_last_step_packing():
    assert len(q.Circuit(2).h(0).cnot(0, 1).steps()) == 2
    c = q.Circuit(2).h(0).x(1)
    assert len(c.steps()) == 1 and len(c.steps()[0].operations) == 2
    assert len(q.Circuit(2).h(0).x(0).steps()) == 2
    c = q.Circuit(2).measure(0)
    c.h(1)
    assert len(c.steps()) == 1
    assert len(q.Circuit(2).h(0).measure(0).steps()) == 2
    # control gates only claim control and target, so a gate inside the span packs
    c = q.Circuit(3).cnot(0, 2).x(1)
    assert len(c.steps()) == 1


def test_argument_validation():
    c = q.Circuit(4)
    for f in (lambda: c.h(4), lambda: c.cnot(1, 1), lambda: c.cnot(0, 7), lambda: c.reset(5)):
        with pytest.raises(q.ArgumentError):
            f()
    c.cnot(0, 3)
    assert len(c.steps()) == 1
    with pytest.raises(q.ArgumentError):
        q.GateType.r(float("inf"))


def test_function_insertion_validates():
    reg = q.GateRegistry()
    reg.register_function("oracle", np.eye(16))
    assert len(q.Circuit(4).add_function("oracle", 0, 4, reg).steps()) == 1
    with pytest.raises(q.ValidationError):
        q.Circuit(4).add_function("oracle", 0, 3, reg)
    with pytest.raises(q.LookupError_):
        q.Circuit(4).add_function("nope", 0, 1, reg)
    with pytest.raises(q.ArgumentError):
        q.Circuit(4).add_function("oracle", 2, 4, reg)
    with pytest.raises(q.ValidationError):
        reg.register_function("bad", np.ones((4, 4)))
    with pytest.raises(q.ValidationError):
        reg.register_function("bad", np.eye(3))


def test_gate_matrices_bit_exact_with_oracle(orc):
    for tag in range(6):
        assert bit_equal(q.gate_matrix(q.GateType(q.GateTag(tag))), orc.gate_matrix(tag))
    for phi in [0.0, 0.3, -2.5, np.pi / 7, np.ldexp(np.pi, -13)]:
        assert bit_equal(q.gate_matrix(q.GateType.r(phi)), orc.gate_matrix(6, phi))


def test_controlled_unitary_matches_oracle(orc):
    rng = np.random.default_rng(1)
    for span in range(2, 6):
        for c in range(span):
            for t in range(span):
                if c == t:
                    continue
                u = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
                assert bit_equal(q.controlled_unitary(u, c, t, span), orc.controlled_unitary(u, c, t, span))


@pytest.mark.parametrize("name,n,case", NAMED)
def test_mirror_flattens_like_reference(golden, name, n, case):
    """The Python mirror of Circuit/gate_matrix/circuit_library produces the
    exact bytes the reference's own circuits serialise to."""
    c, reg = q.make_named_circuit(name, n)
    mine = native.flatten(c, reg)
    ref = golden.flat(case)
    assert mine.ops.tobytes() == ref.ops.tobytes()
    assert mine.step_offsets.tobytes() == ref.step_offsets.tobytes()
    assert len(mine.fn_planes) == len(ref.fn_planes)
    for (a, b), (x, y) in zip(mine.fn_planes, ref.fn_planes):
        assert bit_equal(a, x) and bit_equal(b, y)


def test_dj_variants_and_oracle_specs(golden):
    for spec in ["constant0", "constant1", "balanced-mask:5", "balanced-bit:2"]:
        c, reg = q.make_named_circuit("deutsch-jozsa", 5, spec)
        mine = native.flatten(c, reg)
        ref = golden.flat(f"dj5_{spec.replace(':', '_')}")
        assert mine.ops.tobytes() == ref.ops.tobytes()
        assert bit_equal(mine.fn_planes[0][0], ref.fn_planes[0][0])
    for bad in ["balanced-bit:9", "balanced-mask:0", "balanced-mask:zz"]:
        with pytest.raises(q.ArgumentError):
            q.parse_oracle_spec(bad, 4)
    with pytest.raises(q.ValidationError):
        q.parse_oracle_spec("nope", 4)
    with pytest.raises(q.LookupError_):
        q.make_named_circuit("nope", 3)


def test_qft_structure():
    """QFT step/GEMM counts."""
    want = {4: 13, 6: 24, 8: 39, 10: 58, 11: 68, 12: 81, 13: 93, 14: 108}
    for n, steps in want.items():
        assert len(q.qft(n).steps()) == steps


# ---- the C-ABI library, no GPU ----

def test_library_exports_every_header_symbol():
    L = native.lib()
    names = native.exported_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True, text=True).stdout
    for name in names:
        assert f" T {name}" in out, name
    assert L.qsb_abi_version() == 1


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass        # K2 runs on the FP64 tensor pipe
    assert "UTMALDG" in sass           # A tiles staged by TMA


def test_layer_count_matches_oracle(golden, orc):
    from paper_2305_14398_b200.simulator import step_layer_count

    for case in golden.cases[:120]:
        flat = golden.flat(case)
        for s in range(len(flat.step_offsets) - 1):
            assert step_layer_count(flat, None, s) == orc.step_layers(flat, s)[0]


def test_memory_estimates_match_reference(golden):
    from paper_2305_14398_b200.simulator import memory_estimate

    for n in range(1, 31):
        assert memory_estimate(n, 0) == golden["mem_unitary"][n - 1]
        assert memory_estimate(n, 1) == golden["mem_fsv"][n - 1]


def test_no_cpu_fallback_without_gpu():
    """Without a CUDA device the product path fails loudly (DeviceError)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    with pytest.raises(q.DeviceError):
        B200UnitarySimulator()


def test_abi_struct_layout():
    assert native.OP_DTYPE.itemsize == 104
    assert ctypes.sizeof(native.QsbCircuit) == 40
    assert ctypes.sizeof(native.QsbOptions) == 32
    assert ctypes.sizeof(native.QsbFunction) == 24
    assert ctypes.sizeof(native.QsbPlanInfo) == 80


def test_abi_rejects_bad_circuits():
    """Host validation runs before any device work (layer count is host-only)."""
    L = native.lib()
    c = q.Circuit(3).h(0)
    flat = native.flatten(c)
    n = ctypes.c_int32()
    assert L.qsb_step_layer_count(flat.ptr, 5, ctypes.byref(n)) == 4  # ARGUMENT
    flat.c.n_qubits = 0
    assert L.qsb_step_layer_count(flat.ptr, 0, ctypes.byref(n)) == 4


def test_state_planes_reject_mismatched_lengths():
    """The C ABI carries no lengths: short or mismatched psi planes raise ShapeError
    in the binding (the reference's matvec ShapeError, linalg.cpp:89-94) instead of
    becoming a host out-of-bounds read."""
    import numpy as np
    import pytest

    from paper_2305_14398_b200.errors import ShapeError
    from paper_2305_14398_b200.simulator import _state_planes

    re, im = _state_planes(np.ones(8), np.zeros(8), 8)
    assert re.dtype == np.float64 and len(im) == 8
    with pytest.raises(ShapeError, match="matvec: 8x8 times vector of length 4"):
        _state_planes(np.ones(4), np.zeros(4), 8)
    with pytest.raises(ShapeError):
        _state_planes(np.ones(8), np.zeros(7))


def test_gather_state_rejects_column_block_plans():
    """Column-block shares are summed, not gathered."""
    import pytest

    from paper_2305_14398_b200.sharding import gather_state

    class ColumnPlan:
        columns = True

    with pytest.raises(ValueError, match="row-block"):
        gather_state(ColumnPlan(), None, None, 0, 4, 2)


def test_nccl_loaded_before_torch_keeps_torch_importable():
    """libqsb opens NCCL at first use; loading the system libnccl.so.2 before torch would
    make torch's libtorch_cuda bind to it (same soname) and fail on its newer symbols.
    The binding points libqsb at torch's NCCL wheel, so a later `import torch` works."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k != "QSB_NCCL_LIB"}
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2305_14398_b200.simulator import nccl_version\n"
            "v = nccl_version()\n"
            "import torch, torch.distributed\n"
            "print(v, torch.cuda.nccl.version() if hasattr(torch.cuda, 'nccl') else '')\n" % root)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.split()[0]) >= 22000


def test_bench_reference_arm_line():
    """`bench.py --impl reference` (the driver's reference arm) prints one JSON line
    with the contract's keys, timing the unmodified reference library on this host."""
    import json
    import os
    import subprocess
    import sys

    import oracle

    if not oracle.reference_available():
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--workload", "qft-4",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "ms"
    assert line["higher_is_better"] is False and line["config"]["workload"] == "qft-4"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["extrapolated"] is False
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
