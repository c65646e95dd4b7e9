"""Record golden vectors from the UNMODIFIED reference library.

Runs in the build container, where oracle/_ref/libqsim_refshim.so is compiled
from /root/reference (oracle/Makefile). Every expected value below is produced
by the reference's own code: make_named_circuit / test::random_circuit build
the circuits, UnitarySimulator ("unitary", serial) / test::circuit_unitary /
step_unitary / collapse produce the outputs. The circuits are stored in the ABI
layout (include/qsb.h) exactly as the reference flattens them.

    python tests/golden/make_golden.py      # rewrites tests/golden/golden.npz

Seeds and loops replicate the reference tests they cite (paths relative to
/root/reference/proj).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

ref = oracle.Reference()
L = ref.L
data = {}
index = {"cases": [], "suites": {}}


def put_circuit(key, prog, psi=True, unitary_max_n=6, steps_max_n=0, backend="unitary", fsv=True):
    n, offs, ops, fns = ref.serialize(prog)
    data[f"{key}:n"] = np.array(n)
    data[f"{key}:offs"] = offs
    data[f"{key}:ops"] = ops
    for i, (r, im) in enumerate(fns):
        data[f"{key}:fn{i}_re"] = r
        data[f"{key}:fn{i}_im"] = im
    data[f"{key}:nfn"] = np.array(len(fns))
    if psi:
        re, im = ref.simulate(prog, backend, guard=n)
        data[f"{key}:psi_re"] = re
        data[f"{key}:psi_im"] = im
    if fsv:  # FsvSimulator::simulate_full_state (fsv_backend.cpp:135-158)
        re, im = ref.simulate(prog, "fsv", guard=n)
        data[f"{key}:fsv_re"] = re
        data[f"{key}:fsv_im"] = im
    if n <= unitary_max_n:
        ur, ui = ref.circuit_unitary(prog)
        data[f"{key}:u_re"] = ur
        data[f"{key}:u_im"] = ui
    if n <= steps_max_n:
        for s in range(len(offs) - 1):
            sr, si = ref.step_unitary(prog, s)
            data[f"{key}:step{s}_re"] = sr
            data[f"{key}:step{s}_im"] = si
    index["cases"].append(key)
    return n


t0 = time.time()
# -- named circuits: the BASELINE workloads (circuit_library.cpp:152-179) --------
for n in range(1, 10):
    put_circuit(f"qft{n}", ref.named("qft", n), unitary_max_n=6, steps_max_n=5,
                backend="unitary" if n <= 8 else "unitary-parallel")
for n in range(2, 11):
    put_circuit(f"entangle{n}", ref.named("entangle", n), unitary_max_n=6, steps_max_n=5,
                backend="unitary" if n <= 8 else "unitary-parallel")
for n in range(2, 10):
    put_circuit(f"dj{n}", ref.named("deutsch-jozsa", n), unitary_max_n=6, steps_max_n=5,
                backend="unitary" if n <= 8 else "unitary-parallel")
for spec in ["constant0", "constant1", "balanced-mask:5", "balanced-bit:2"]:
    put_circuit(f"dj5_{spec.replace(':', '_')}", ref.named("deutsch-jozsa", 5, spec), unitary_max_n=6)
put_circuit("bell", ref.named("bell", 2), steps_max_n=2)

# -- hand-built edge cases (test_unitary_backend.cpp:29-47, :86-102, :114-118, :223-231) --
def build(n, ops):
    p = oracle.RefProgram(ref, L.refsh_circuit_new(n))
    for op in ops:
        kind = op[0]
        if kind == "g":
            assert L.refsh_add_gate(p.h, op[1], op[2], op[3]) == 0
        elif kind == "c":
            assert L.refsh_add_control(p.h, op[1], op[2], op[3], op[4]) == 0
        elif kind == "i":
            assert L.refsh_add_instruction(p.h, op[1], op[2]) == 0
    return p


H, X, Y, Z, S, T, R = range(7)
put_circuit("edge_measure_only", build(2, [("i", 0, 0)]), steps_max_n=2)
put_circuit("edge_span_overlap", build(3, [("c", X, 0.0, 0, 2), ("g", X, 0.0, 1)]), steps_max_n=3)
put_circuit("edge_terminal_reset", build(2, [("g", H, 0.0, 0), ("i", 1, 0)]), steps_max_n=2)
put_circuit("edge_empty", build(3, []), steps_max_n=3)
put_circuit("edge_ctrl_below", build(4, [("c", R, 0.7, 3, 0), ("g", Y, 0.0, 1), ("c", X, 0.0, 2, 1),
                                         ("g", S, 0.0, 2), ("c", R, -1.3, 1, 3), ("g", T, 0.0, 0)]), steps_max_n=4)
put_circuit("edge_wide_span", build(6, [("c", R, 2.1, 0, 5), ("g", H, 0.0, 2), ("g", Z, 0.0, 3),
                                        ("c", X, 0.0, 4, 1), ("g", H, 0.0, 5)]), steps_max_n=6)

# -- random suites replaying the reference tests' seeds ----------------------------
def suite(name, seed, count, sequence, unitary_max_n=5, steps_max_n=0):
    rng = L.refsh_rng_new(seed)
    keys = []
    for i in range(count):
        p = sequence(rng)
        key = f"{name}_{i}"
        put_circuit(key, p, unitary_max_n=unitary_max_n, steps_max_n=steps_max_n)
        keys.append(key)
    L.refsh_rng_free(rng)
    index["suites"][name] = keys


def seq_pick_then_circuit(qlo, qhi, olo, ohi):
    def f(rng):
        n = L.refsh_rng_uniform_size(rng, qlo, qhi)
        ops = L.refsh_rng_uniform_size(rng, olo, ohi)
        return oracle.RefProgram(ref, L.refsh_random_circuit(rng, n, ops))
    return f


def seq_fixed(n, ops):
    return lambda rng: oracle.RefProgram(ref, L.refsh_random_circuit(rng, n, ops))


# acceptance_main.cpp:80-110 (seed 20260810: 200 circuits, 2..8 qubits, 1..30 ops)
suite("cross", 20260810, 200, seq_pick_then_circuit(2, 8, 1, 30), unitary_max_n=4)
# test_unitary_backend.cpp:172-185 (seed 31415: 20 circuits, 2..6 qubits, 1..25 ops)
suite("fsv", 31415, 20, seq_pick_then_circuit(2, 6, 1, 25))
# test_unitary_backend.cpp:132-142 (seed 555: 12 circuits, 2..6 qubits, 1..50 ops)
suite("norm", 555, 12, seq_pick_then_circuit(2, 6, 1, 50))
# test_unitary_backend.cpp:75-84 (seed 31337: 10 x random_circuit(rng, 5, 12), step unitaries)
suite("steps", 31337, 10, seq_fixed(5, 12), steps_max_n=5)
# test_unitary_backend.cpp:155-170 (seed 4242: 8 x random_circuit(rng, 5, 16))
suite("par", 4242, 8, seq_fixed(5, 16))
# acceptance_main.cpp:270-292 (seed 777: 50 x random_circuit(rng, qubit_pick(rng), op_pick(rng)))
rng = L.refsh_rng_new(777)
keys = []
for i in range(50):
    p = oracle.RefProgram(ref, L.refsh_random_circuit_args(rng, 2, 6, 1, 20))
    put_circuit(f"det_{i}", p, unitary_max_n=4)
    keys.append(f"det_{i}")
L.refsh_rng_free(rng)
index["suites"]["det"] = keys

# test_unitary_backend.cpp:143-153 (seed 808: random_circuit(rng, 4, 15) then random_state(rng, 4))
rng = L.refsh_rng_new(808)
keys = []
for i in range(6):
    p = oracle.RefProgram(ref, L.refsh_random_circuit(rng, 4, 15))
    key = f"comp_{i}"
    put_circuit(key, p, unitary_max_n=4)
    re, im = np.empty(16), np.empty(16)
    assert L.refsh_random_state(rng, 4, re.ctypes.data, im.ctypes.data) == 0
    data[f"{key}:state_re"] = re
    data[f"{key}:state_im"] = im
    keys.append(key)
L.refsh_rng_free(rng)
index["suites"]["comp"] = keys

# -- fsv backend beyond one shared-memory slab (2^12 amplitudes): states only -----
put_circuit("fsvbig_qft13", ref.named("qft", 13), psi=False, unitary_max_n=0)
put_circuit("fsvbig_entangle14", ref.named("entangle", 14), psi=False, unitary_max_n=0)
rng = L.refsh_rng_new(4711)
keys = ["fsvbig_qft13", "fsvbig_entangle14"]
for i, (n, ops) in enumerate([(13, 60), (13, 120), (14, 90), (15, 40)]):
    p = oracle.RefProgram(ref, L.refsh_random_circuit(rng, n, ops))
    put_circuit(f"fsvbig_{i}", p, psi=False, unitary_max_n=0)
    keys.append(f"fsvbig_{i}")
L.refsh_rng_free(rng)
index["suites"]["fsvbig"] = keys

# -- state.cpp: SplitMix64 draws, collapse outcomes, probabilities ---------------
seeds = np.arange(0, 64, dtype=np.uint64)
data["splitmix_bits"] = np.array([L.refsh_splitmix64_unit_bits(int(s), 1) for s in seeds], dtype=np.uint64)
data["splitmix_bits_3"] = np.array([L.refsh_splitmix64_unit_bits(int(s), 3) for s in seeds], dtype=np.uint64)
bell_re = data["bell:psi_re"]
bell_im = data["bell:psi_im"]
data["collapse_bell"] = np.array([ref.collapse(bell_re, bell_im, int(s)) for s in seeds], dtype=np.uint64)
qre, qim = data["qft5:psi_re"], data["qft5:psi_im"]
data["collapse_qft5"] = np.array([ref.collapse(qre, qim, int(s)) for s in range(200)], dtype=np.uint64)
for key in ["comp_0", "comp_1"]:
    re, im = data[f"{key}:state_re"], data[f"{key}:state_im"]
    p, norm = np.empty(16), np.array(0.0)
    assert L.refsh_probabilities(4, re.ctypes.data, im.ctypes.data, p.ctypes.data, norm.ctypes.data) == 0
    data[f"{key}:probs"] = p
    data[f"{key}:norm"] = norm.copy()
    data[f"{key}:collapse"] = np.array([ref.collapse(re, im, s) for s in range(64)], dtype=np.uint64)

# -- unitary_backend.cpp:156-192: memory accounting --------------------------------
data["mem_unitary"] = np.array([L.refsh_memory_estimate(n, 0) for n in range(1, 31)], dtype=np.uint64)
data["mem_fsv"] = np.array([L.refsh_memory_estimate(n, 1) for n in range(1, 31)], dtype=np.uint64)
data["engine_unitary"] = np.array([L.refsh_engine_memory_estimate(n, 0) for n in range(1, 30)], dtype=np.uint64)
buf = __import__("ctypes").create_string_buffer(64)
fmt = []
for b in [0, 1, 999, 1000, 1234567, 8796101410816, 8388608, 137438953472, 2**63]:
    L.refsh_format_bytes(b, buf, 64)
    fmt.append([str(b), buf.value.decode()])
index["format_bytes"] = fmt
data["index_json"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)

np.savez_compressed(OUT, **data)
print(f"wrote {OUT}: {len(index['cases'])} circuits, {os.path.getsize(OUT) / 1e6:.2f} MB, {time.time() - t0:.1f} s")
