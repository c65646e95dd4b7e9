"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the parity checkers.

* :class:`Oracle`   — liboracle.so, the plain-C restatement (qsim_oracle.c).
* :class:`Reference`— _ref/libqsim_refshim.so over the UNMODIFIED reference
  library compiled from /root/reference (oracle/Makefile). Present wherever it
  was built (this container; it travels to the GPU box as a prebuilt .so).

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs may import this package. The product (libqsb.so) never links it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")
REFSHIM_SO = os.path.join(REF_DIR, "libqsim_refshim.so")

P, I32, I64, U64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double


def build(reference: bool = True) -> None:
    """Compile the oracle (always) and, when /root/reference exists, oracle/_ref."""
    targets = ["oracle"]
    if reference and os.path.isdir("/root/reference/proj"):
        targets += ["ref", "dropin"]
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """The C restatement; circuits are native.FlatCircuit objects (the ABI layout)."""

    def __init__(self) -> None:
        if not os.path.exists(ORACLE_SO):
            build(reference=False)
        L = ctypes.CDLL(ORACLE_SO)
        sig = {
            "orc_last_error": (ctypes.c_char_p, []),
            "orc_set_threads": (None, [ctypes.c_int]),
            "orc_gate_matrix": (ctypes.c_int, [I32, D, P, P]),
            "orc_controlled_unitary": (ctypes.c_int, [P, P, I64, I64, I64, P, P]),
            "orc_kronecker": (ctypes.c_int, [P, P, I64, I64, P, P, I64, I64, P, P]),
            "orc_matmul": (ctypes.c_int, [P, P, P, P, I64, I64, I64, P, P]),
            "orc_matvec": (ctypes.c_int, [P, P, I64, I64, P, P, P, P]),
            "orc_step_layers": (ctypes.c_int, [P, I32, P, P]),
            "orc_layer_operator": (ctypes.c_int, [P, I32, I32, P, P]),
            "orc_step_unitary": (ctypes.c_int, [P, I32, P, P]),
            "orc_circuit_unitary": (ctypes.c_int, [P, P, P]),
            "orc_validate_instruction_placement": (ctypes.c_int, [P]),
            "orc_unitary_simulate": (ctypes.c_int, [P, I32, P, P]),
            "orc_fsv_apply": (ctypes.c_int, [P, P, P]),
            "orc_splitmix64_next": (U64, [P]),
            "orc_splitmix64_unit": (D, [P]),
            "orc_norm_squared": (D, [P, P, I64]),
            "orc_probabilities": (None, [P, P, I64, P]),
            "orc_collapse": (U64, [P, P, I64, U64]),
            "orc_memory_estimate": (U64, [I32, I32]),
            "orc_engine_memory_estimate": (U64, [I32, I32]),
            "orc_format_bytes": (None, [U64, ctypes.c_char_p, ctypes.c_size_t]),
            "orc_is_unitary": (ctypes.c_int, [P, P, I64, D]),
            "orc_max_entry_diff": (D, [P, P, P, P, I64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self.L = L

    def _check(self, rc: int) -> None:
        if rc:
            raise OracleError(rc, self.L.orc_last_error().decode())

    def set_threads(self, n: int) -> None:
        self.L.orc_set_threads(n)

    def gate_matrix(self, gate: int, phi: float = 0.0) -> np.ndarray:
        re, im = np.empty(4), np.empty(4)
        self._check(self.L.orc_gate_matrix(gate, phi, _ptr(re), _ptr(im)))
        return (re + 1j * im).reshape(2, 2)

    def controlled_unitary(self, u: np.ndarray, cpos: int, tpos: int, span: int) -> np.ndarray:
        ur = np.ascontiguousarray(u.real.reshape(4))
        ui = np.ascontiguousarray(u.imag.reshape(4))
        d = 1 << span
        re, im = np.empty((d, d)), np.empty((d, d))
        self._check(self.L.orc_controlled_unitary(_ptr(ur), _ptr(ui), cpos, tpos, span, _ptr(re), _ptr(im)))
        return re + 1j * im

    def matmul(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        ar, ai = np.ascontiguousarray(a.real), np.ascontiguousarray(a.imag)
        br, bi = np.ascontiguousarray(b.real), np.ascontiguousarray(b.imag)
        m, k = a.shape
        n = b.shape[1]
        cr, ci = np.empty((m, n)), np.empty((m, n))
        self._check(self.L.orc_matmul(_ptr(ar), _ptr(ai), _ptr(br), _ptr(bi), m, k, n, _ptr(cr), _ptr(ci)))
        return cr + 1j * ci

    def kronecker(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        ar, ai = np.ascontiguousarray(a.real), np.ascontiguousarray(a.imag)
        br, bi = np.ascontiguousarray(b.real), np.ascontiguousarray(b.imag)
        cr = np.empty((a.shape[0] * b.shape[0], a.shape[1] * b.shape[1]))
        ci = np.empty_like(cr)
        self._check(self.L.orc_kronecker(_ptr(ar), _ptr(ai), a.shape[0], a.shape[1], _ptr(br), _ptr(bi),
                                         b.shape[0], b.shape[1], _ptr(cr), _ptr(ci)))
        return cr + 1j * ci

    def step_layers(self, flat, step: int) -> Tuple[int, List[int]]:
        n_ops = int(flat.step_offsets[step + 1] - flat.step_offsets[step])
        lo = np.zeros(max(n_ops, 1), dtype=np.int32)
        nl = ctypes.c_int32()
        self._check(self.L.orc_step_layers(flat.ptr, step, ctypes.byref(nl), _ptr(lo)))
        return nl.value, lo[:n_ops].tolist()

    def _square(self, n_qubits: int):
        N = 1 << n_qubits
        return np.empty((N, N)), np.empty((N, N))

    def layer_operator(self, flat, step: int, layer: int) -> Tuple[np.ndarray, np.ndarray]:
        re, im = self._square(flat.n_qubits)
        self._check(self.L.orc_layer_operator(flat.ptr, step, layer, _ptr(re), _ptr(im)))
        return re, im

    def step_unitary(self, flat, step: int) -> Tuple[np.ndarray, np.ndarray]:
        re, im = self._square(flat.n_qubits)
        self._check(self.L.orc_step_unitary(flat.ptr, step, _ptr(re), _ptr(im)))
        return re, im

    def circuit_unitary(self, flat) -> Tuple[np.ndarray, np.ndarray]:
        re, im = self._square(flat.n_qubits)
        self._check(self.L.orc_circuit_unitary(flat.ptr, _ptr(re), _ptr(im)))
        return re, im

    def unitary_simulate(self, flat, guard: int = 0) -> Tuple[np.ndarray, np.ndarray]:
        N = 1 << flat.n_qubits
        re, im = np.empty(N), np.empty(N)
        self._check(self.L.orc_unitary_simulate(flat.ptr, guard, _ptr(re), _ptr(im)))
        return re, im

    def fsv(self, flat, re0: Optional[np.ndarray] = None, im0: Optional[np.ndarray] = None):
        N = 1 << flat.n_qubits
        re = np.zeros(N) if re0 is None else np.array(re0, dtype=np.float64)
        im = np.zeros(N) if im0 is None else np.array(im0, dtype=np.float64)
        if re0 is None:
            re[0] = 1.0
        self._check(self.L.orc_fsv_apply(flat.ptr, _ptr(re), _ptr(im)))
        return re, im

    def unitary_column(self, flat, col: int) -> Tuple[np.ndarray, np.ndarray]:
        """U[:, col] = fsv(e_col) — large-n oracle."""
        N = 1 << flat.n_qubits
        re, im = np.zeros(N), np.zeros(N)
        re[col] = 1.0
        return self.fsv(flat, re, im)

    def probabilities(self, re: np.ndarray, im: np.ndarray) -> np.ndarray:
        p = np.empty(len(re))
        self.L.orc_probabilities(_ptr(re), _ptr(im), len(re), _ptr(p))
        return p

    def norm_squared(self, re: np.ndarray, im: np.ndarray) -> float:
        return self.L.orc_norm_squared(_ptr(re), _ptr(im), len(re))

    def collapse(self, re: np.ndarray, im: np.ndarray, seed: int) -> int:
        return int(self.L.orc_collapse(_ptr(re), _ptr(im), len(re), seed))

    def splitmix64_unit(self, seed: int, draws: int = 1) -> float:
        st = ctypes.c_uint64(seed)
        u = 0.0
        for _ in range(draws):
            u = self.L.orc_splitmix64_unit(ctypes.byref(st))
        return u

    def memory_estimate(self, n: int, kind: int = 0) -> int:
        return int(self.L.orc_memory_estimate(n, kind))

    def engine_memory_estimate(self, n: int, kind: int = 0) -> int:
        return int(self.L.orc_engine_memory_estimate(n, kind))

    def format_bytes(self, b: int) -> str:
        buf = ctypes.create_string_buffer(64)
        self.L.orc_format_bytes(b, buf, 64)
        return buf.value.decode()

    def is_unitary(self, u: np.ndarray, tol: float) -> bool:
        re, im = np.ascontiguousarray(u.real), np.ascontiguousarray(u.imag)
        return bool(self.L.orc_is_unitary(_ptr(re), _ptr(im), u.shape[0], tol))


def reference_available() -> bool:
    return os.path.exists(REFSHIM_SO)


class RefProgram:
    def __init__(self, ref: "Reference", handle: int):
        if not handle:
            raise OracleError(8, ref.L.refsh_last_error().decode())
        self.ref, self.h = ref, handle

    def __del__(self):
        try:
            self.ref.L.refsh_free(self.h)
        except Exception:
            pass


class Reference:
    """The unmodified reference library (oracle/_ref), via ref_shim.cpp."""

    def __init__(self) -> None:
        if not reference_available():
            raise RuntimeError("oracle/_ref/libqsim_refshim.so is not built (needs /root/reference)")
        L = ctypes.CDLL(REFSHIM_SO)
        C = ctypes.c_char_p
        sig = {
            "refsh_last_error": (C, []),
            "refsh_free": (None, [P]),
            "refsh_named": (P, [C, ctypes.c_int, C]),
            "refsh_circuit_new": (P, [ctypes.c_int]),
            "refsh_add_gate": (ctypes.c_int, [P, I32, D, I32]),
            "refsh_add_control": (ctypes.c_int, [P, I32, D, I32, I32]),
            "refsh_add_instruction": (ctypes.c_int, [P, I32, I32]),
            "refsh_register_function": (ctypes.c_int, [P, C, I64, P, P]),
            "refsh_add_function": (ctypes.c_int, [P, C, I32, I32]),
            "refsh_rng_new": (P, [U64]),
            "refsh_rng_free": (None, [P]),
            "refsh_rng_uniform_size": (U64, [P, U64, U64]),
            "refsh_random_circuit": (P, [P, ctypes.c_int, ctypes.c_int]),
            "refsh_random_state": (ctypes.c_int, [P, ctypes.c_int, P, P]),
            "refsh_random_circuit_args": (P, [P, U64, U64, U64, U64]),
            "refsh_n_qubits": (ctypes.c_int, [P]),
            "refsh_n_steps": (ctypes.c_int, [P]),
            "refsh_n_ops": (ctypes.c_int, [P]),
            "refsh_n_functions": (ctypes.c_int, [P]),
            "refsh_serialize": (ctypes.c_int, [P, P, P]),
            "refsh_function_dim": (I64, [P, ctypes.c_int]),
            "refsh_function_matrix": (ctypes.c_int, [P, ctypes.c_int, P, P]),
            "refsh_step_unitary": (ctypes.c_int, [P, ctypes.c_int, P, P]),
            "refsh_step_operand_count": (ctypes.c_int, [P, ctypes.c_int, P]),
            "refsh_circuit_unitary": (ctypes.c_int, [P, ctypes.c_int, P, P]),
            "refsh_simulate": (ctypes.c_int, [P, C, ctypes.c_int, P, P]),
            "refsh_simulate_and_collapse": (ctypes.c_int, [P, C, U64, P]),
            "refsh_collapse": (ctypes.c_int, [ctypes.c_int, P, P, U64, P]),
            "refsh_probabilities": (ctypes.c_int, [ctypes.c_int, P, P, P, P]),
            "refsh_splitmix64_unit_bits": (U64, [U64, ctypes.c_int]),
            "refsh_memory_estimate": (U64, [ctypes.c_int, ctypes.c_int]),
            "refsh_engine_memory_estimate": (U64, [ctypes.c_int, ctypes.c_int]),
            "refsh_format_bytes": (ctypes.c_int, [U64, C, ctypes.c_int]),
            "refsh_set_worker_count": (None, [ctypes.c_int]),
            "refsh_worker_count": (ctypes.c_int, []),
            "refsh_time_step_unitary": (D, [P, ctypes.c_int]),
            "refsh_time_matmul": (D, [I64, I64, ctypes.c_int]),
            "refsh_time_simulate": (D, [P, C, ctypes.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self.L = L

    def _check(self, rc: int) -> None:
        if rc:
            raise OracleError(rc, self.L.refsh_last_error().decode())

    def named(self, name: str, qubits: int, oracle_spec: str = "") -> RefProgram:
        return RefProgram(self, self.L.refsh_named(name.encode(), qubits, oracle_spec.encode()))

    def serialize(self, prog: RefProgram):
        """-> (n_qubits, step_offsets int32, ops OP_DTYPE, [(fn_re, fn_im)])"""
        from paper_2305_14398_b200.native import OP_DTYPE

        n_steps = self.L.refsh_n_steps(prog.h)
        n_ops = self.L.refsh_n_ops(prog.h)
        offs = np.zeros(n_steps + 1, dtype=np.int32)
        ops = np.zeros(max(n_ops, 1), dtype=OP_DTYPE)
        self._check(self.L.refsh_serialize(prog.h, _ptr(offs), _ptr(ops)))
        fns = []
        for i in range(self.L.refsh_n_functions(prog.h)):
            d = self.L.refsh_function_dim(prog.h, i)
            re, im = np.empty((d, d)), np.empty((d, d))
            self._check(self.L.refsh_function_matrix(prog.h, i, _ptr(re), _ptr(im)))
            fns.append((re, im))
        return self.L.refsh_n_qubits(prog.h), offs, ops[:n_ops], fns

    def step_unitary(self, prog: RefProgram, step: int):
        N = 1 << self.L.refsh_n_qubits(prog.h)
        re, im = np.empty((N, N)), np.empty((N, N))
        self._check(self.L.refsh_step_unitary(prog.h, step, _ptr(re), _ptr(im)))
        return re, im

    def circuit_unitary(self, prog: RefProgram, parallel: bool = False):
        N = 1 << self.L.refsh_n_qubits(prog.h)
        re, im = np.empty((N, N)), np.empty((N, N))
        self._check(self.L.refsh_circuit_unitary(prog.h, 1 if parallel else 0, _ptr(re), _ptr(im)))
        return re, im

    def simulate(self, prog: RefProgram, backend: str = "unitary", guard: int = 0):
        N = 1 << self.L.refsh_n_qubits(prog.h)
        re, im = np.empty(N), np.empty(N)
        self._check(self.L.refsh_simulate(prog.h, backend.encode(), guard, _ptr(re), _ptr(im)))
        return re, im

    def collapse(self, re: np.ndarray, im: np.ndarray, seed: int) -> int:
        n = int(np.log2(len(re)))
        out = ctypes.c_uint64()
        self._check(self.L.refsh_collapse(n, _ptr(np.ascontiguousarray(re)), _ptr(np.ascontiguousarray(im)), seed,
                                          ctypes.byref(out)))
        return out.value
