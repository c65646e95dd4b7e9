"""ctypes binding of the C ABI (include/qsb.h) and the circuit flattener.

The product path is libqsb.so (hand-written sm_100a kernels + C++ runtime),
built in-tree by ``__graft_entry__.build()``. There is no fallback: if the
library is missing or no sm_100a device is present, calls raise loudly.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from .circuit import Circuit, ControlGate, FunctionOp, Gate, GateRegistry, Instruction, gate_matrix
from .errors import ArgumentError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqsb.so")

# qsb_op (include/qsb.h): 8 x int32, phi, u_re[4], u_im[4] -> 104 bytes.
OP_DTYPE = np.dtype([
    ("kind", "<i4"), ("gate", "<i4"), ("target", "<i4"), ("control", "<i4"),
    ("first", "<i4"), ("count", "<i4"), ("function", "<i4"), ("instruction", "<i4"),
    ("phi", "<f8"), ("u_re", "<f8", (4,)), ("u_im", "<f8", (4,)),
])
assert OP_DTYPE.itemsize == 104

OP_GATE, OP_CONTROL, OP_FUNCTION, OP_INSTRUCTION = 0, 1, 2, 3
GEMM_AUTO, GEMM_4M, GEMM_3M = 0, 1, 2
FLAG_NO_GRAPH, FLAG_MATERIALIZE, FLAG_COLUMN_BLOCKS, FLAG_NCCL_GATHER, FLAG_NO_PLAN_CACHE = 1, 2, 4, 8, 16
NCCL_ID_BYTES = 128
TILE_NAMES = {0: "zgemm_gen_kernel<128,64> (4M)", 1: "zgemm_gen_kernel<64,64> (4M)", 2: "zgemm_gen_kernel<32,32> (4M)",
              3: "zgemm_ws_kernel<4M>", 4: "zgemm_ws_kernel<3M>", 5: "zgemm_ws_kernel<3M, sum plane>",
              6: "zgemm_chain_kernel (K2c: the whole chain in one persistent launch)"}


class QsbFunction(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int64), ("re", ctypes.c_void_p), ("im", ctypes.c_void_p)]


class QsbCircuit(ctypes.Structure):
    _fields_ = [
        ("n_qubits", ctypes.c_int32), ("n_steps", ctypes.c_int32),
        ("step_offsets", ctypes.c_void_p), ("ops", ctypes.c_void_p),
        ("n_functions", ctypes.c_int32), ("functions", ctypes.c_void_p),
    ]


class QsbOptions(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("qubit_guard", ctypes.c_int32),
                ("gemm_mode", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("n_devices", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("devices", ctypes.c_void_p)]


class QsbPlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_qubits", ctypes.c_int32), ("n_steps", ctypes.c_int32), ("n_layers", ctypes.c_int32),
        ("n_gemms", ctypes.c_int32), ("n_identity_layers", ctypes.c_int32), ("n_launches", ctypes.c_int32),
        ("row_begin", ctypes.c_int64), ("row_count", ctypes.c_int64),
        ("gemm_flops", ctypes.c_double), ("expand_bytes", ctypes.c_double),
        ("gemm_tile", ctypes.c_int32), ("v_planes", ctypes.c_int32),
        ("gemm_splits", ctypes.c_int32), ("n_real_gemms", ctypes.c_int32), ("gemm_hw_flops", ctypes.c_double),
    ]


SV_STATE, SV_UNITARY = 0, 1


class QsbSvPlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_qubits", ctypes.c_int32), ("mode", ctypes.c_int32), ("n_ops", ctypes.c_int32),
        ("n_passes", ctypes.c_int32), ("n_function_passes", ctypes.c_int32), ("n_launches", ctypes.c_int32),
        ("slab_bits", ctypes.c_int32), ("max_batch_targets", ctypes.c_int32),
        ("col_begin", ctypes.c_int64), ("col_count", ctypes.c_int64), ("bytes_per_run", ctypes.c_double),
    ]


@dataclass
class FlatCircuit:
    """A circuit flattened into the ABI's arrays; keeps the numpy storage alive."""

    n_qubits: int
    step_offsets: np.ndarray
    ops: np.ndarray
    fn_planes: List[Tuple[np.ndarray, np.ndarray]]
    fn_structs: Optional[ctypes.Array]
    c: QsbCircuit

    @property
    def ptr(self):
        return ctypes.byref(self.c)

    def nbytes(self) -> int:
        return int(self.step_offsets.nbytes + self.ops.nbytes
                   + sum(r.nbytes + i.nbytes for r, i in self.fn_planes))


def _make_struct(n_qubits, step_offsets, ops, fn_planes) -> FlatCircuit:
    n_fn = len(fn_planes)
    fn_structs = None
    if n_fn:
        fn_structs = (QsbFunction * n_fn)()
        for i, (r, im) in enumerate(fn_planes):
            fn_structs[i].dim = r.shape[0]
            fn_structs[i].re = r.ctypes.data
            fn_structs[i].im = im.ctypes.data
    c = QsbCircuit(n_qubits, len(step_offsets) - 1, step_offsets.ctypes.data, ops.ctypes.data, n_fn,
                   ctypes.cast(fn_structs, ctypes.c_void_p).value if fn_structs is not None else None)
    return FlatCircuit(n_qubits, step_offsets, ops, fn_planes, fn_structs, c)


def flatten(circuit: Circuit, registry: Optional[GateRegistry] = None) -> FlatCircuit:
    """Flatten a Circuit (after its greedy last-step packing) into the ABI format;
    u = gate_matrix(g) (gates.cpp:40-77), registry matrices as re/im planes."""
    steps = circuit.steps()
    n_ops = sum(len(s.operations) for s in steps)
    ops = np.zeros(n_ops, dtype=OP_DTYPE)
    offsets = np.zeros(len(steps) + 1, dtype=np.int32)
    fn_index = {}
    fn_planes: List[Tuple[np.ndarray, np.ndarray]] = []
    k = 0
    for si, step in enumerate(steps):
        for op in step.operations:
            o = ops[k]
            if isinstance(op, (Gate, ControlGate)):
                o["kind"] = OP_GATE if isinstance(op, Gate) else OP_CONTROL
                o["gate"] = int(op.gate.tag)
                o["phi"] = op.gate.phi
                o["target"] = op.target
                if isinstance(op, ControlGate):
                    o["control"] = op.control
                m = gate_matrix(op.gate)
                o["u_re"] = m.real.reshape(4)
                o["u_im"] = m.imag.reshape(4)
            elif isinstance(op, FunctionOp):
                if registry is None:
                    raise ArgumentError(f"function '{op.name}' needs a registry")
                if op.name not in fn_index:
                    m = registry.lookup(op.name)
                    fn_index[op.name] = len(fn_planes)
                    fn_planes.append((np.ascontiguousarray(m.real), np.ascontiguousarray(m.imag)))
                o["kind"] = OP_FUNCTION
                o["first"] = op.first_qubit
                o["count"] = op.qubit_count
                o["function"] = fn_index[op.name]
            elif isinstance(op, Instruction):
                o["kind"] = OP_INSTRUCTION
                o["target"] = op.target
                o["instruction"] = int(op.kind)
            k += 1
        offsets[si + 1] = k
    return _make_struct(circuit.qubit_count(), offsets, ops, fn_planes)


def flat_from_arrays(n_qubits: int, step_offsets: np.ndarray, ops: np.ndarray,
                     fn_planes: List[Tuple[np.ndarray, np.ndarray]]) -> FlatCircuit:
    """Wrap arrays already in the ABI format (e.g. golden fixtures)."""
    return _make_struct(int(n_qubits), np.ascontiguousarray(step_offsets, dtype=np.int32),
                        np.ascontiguousarray(ops, dtype=OP_DTYPE),
                        [(np.ascontiguousarray(r, dtype=np.float64), np.ascontiguousarray(i, dtype=np.float64))
                         for r, i in fn_planes])


_lib = None


def _point_at_torch_nccl() -> None:
    """libqsb opens NCCL at first use. If it loaded the system libnccl.so.2 before torch
    is imported, torch's libtorch_cuda would bind to that copy (same soname) and fail on
    symbols of its own newer NCCL: point libqsb at the NCCL wheel torch uses, found on
    sys.path without importing torch (QSB_NCCL_LIB set by the caller wins)."""
    import sys

    if os.environ.get("QSB_NCCL_LIB"):
        return
    for base in sys.path:
        cand = os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so.2")
        if base and os.path.exists(cand):
            os.environ["QSB_NCCL_LIB"] = cand
            return


def lib() -> ctypes.CDLL:
    """Load libqsb.so (fails loudly: no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 path)")
    _point_at_torch_nccl()
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    sig = {
        "qsb_abi_version": (ctypes.c_int, []),
        "qsb_last_error": (ctypes.c_size_t, [ctypes.c_char_p, ctypes.c_size_t]),
        "qsb_create": (ctypes.c_int, [P, P]),
        "qsb_destroy": (ctypes.c_int, [P]),
        "qsb_qubit_guard": (ctypes.c_int, [P, P]),
        "qsb_simulate_full_state": (ctypes.c_int, [P, P, P, P]),
        "qsb_simulate_from_state": (ctypes.c_int, [P, P, P, P, P, P]),
        "qsb_build_unitary": (ctypes.c_int, [P, P, P, P]),
        "qsb_simulate_and_collapse": (ctypes.c_int, [P, P, U64, P]),
        "qsb_step_layer_count": (ctypes.c_int, [P, I32, P]),
        "qsb_layer_operator": (ctypes.c_int, [P, P, I32, I32, P, P]),
        "qsb_probabilities": (ctypes.c_int, [P, P, P, I64, P, P]),
        "qsb_plan_create": (ctypes.c_int, [P, P, I64, I64, P]),
        "qsb_plan_destroy": (ctypes.c_int, [P]),
        "qsb_plan_get_info": (ctypes.c_int, [P, P]),
        "qsb_plan_set_timing": (ctypes.c_int, [P, I32]),
        "qsb_plan_set_initial_state": (ctypes.c_int, [P, P, P, P]),
        "qsb_plan_execute": (ctypes.c_int, [P, P]),
        "qsb_plan_unitary_device": (ctypes.c_int, [P, P, P]),
        "qsb_plan_state_device": (ctypes.c_int, [P, P, P]),
        "qsb_plan_copy_state": (ctypes.c_int, [P, P, P, P]),
        "qsb_plan_last_timing": (ctypes.c_int, [P, P, P, P]),
        "qsb_plan_gemm_times": (ctypes.c_int, [P, P, P, I32, P]),
        "qsb_nccl_unique_id": (ctypes.c_int, [P]),
        "qsb_nccl_version": (ctypes.c_int, [P]),
        "qsb_comm_create": (ctypes.c_int, [P, P, I32, I32, P]),
        "qsb_comm_destroy": (ctypes.c_int, [P]),
        "qsb_simulate_full_state_sharded": (ctypes.c_int, [P, P, P, P, P]),
        "qsb_plan_allgather_state": (ctypes.c_int, [P, P, P, P, P]),
        "qsb_plan_allgather_unitary": (ctypes.c_int, [P, P, P, P, P]),
        "qsb_collapse": (ctypes.c_int, [P, P, P, I64, U64, P]),
        "qsb_is_unitary": (ctypes.c_int, [P, P, P, I64, D, P, P]),
        "qsb_fsv_qubit_guard": (ctypes.c_int, [P, P]),
        "qsb_fsv_simulate_full_state": (ctypes.c_int, [P, P, P, P]),
        "qsb_fsv_simulate_from_state": (ctypes.c_int, [P, P, P, P, P, P]),
        "qsb_structured_qubit_guard": (ctypes.c_int, [P, P]),
        "qsb_structured_build_unitary": (ctypes.c_int, [P, P, P, P]),
        "qsb_structured_simulate_full_state": (ctypes.c_int, [P, P, P, P]),
        "qsb_sv_plan_create": (ctypes.c_int, [P, P, I32, I64, I64, P]),
        "qsb_sv_plan_destroy": (ctypes.c_int, [P]),
        "qsb_sv_plan_get_info": (ctypes.c_int, [P, P]),
        "qsb_sv_plan_set_state": (ctypes.c_int, [P, P, P, P]),
        "qsb_sv_plan_execute": (ctypes.c_int, [P, P]),
        "qsb_sv_plan_result_device": (ctypes.c_int, [P, P, P]),
        "qsb_memory_estimate": (U64, [I32, I32]),
        "qsb_engine_memory_estimate": (U64, [I32, I32]),
        "qsb_hbm_footprint": (U64, [I32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols() -> List[str]:
    """Names declared in include/qsb.h (used by the symbol-export test)."""
    import re

    hdr = os.path.join(_HERE, "..", "include", "qsb.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"^(?:qsb_status|int|size_t|uint64_t)\s+(qsb_\w+)\(", text, re.M)))


def last_error() -> str:
    buf = ctypes.create_string_buffer(1024)
    lib().qsb_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def check(status: int) -> None:
    if status != 0:
        raise_for_status(status, last_error())


def dptr(a: np.ndarray) -> int:
    return a.ctypes.data
