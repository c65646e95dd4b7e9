"""Simulator plugin interface + the B200 backend, mirroring
core/include/qsim/simulator.hpp:32-68 and core/src/simulator.cpp:26-82.

``B200UnitarySimulator`` is registered as ``"unitary-b200"``. Every call goes
through libqsb.so's C ABI (include/qsb.h); nothing here computes amplitudes.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Tuple

import numpy as np

from . import native
from .circuit import Circuit, GateRegistry
from .errors import LookupError_, ShapeError

BACKEND_ID = "unitary-b200"
FSV_BACKEND_ID = "fsv-b200"
STRUCTURED_BACKEND_ID = "unitary-structured-b200"


@dataclass
class StateVector:
    """StateVector (state.hpp:46-51): amplitudes as re/im planes."""

    n_qubits: int
    re: np.ndarray
    im: np.ndarray

    def dimension(self) -> int:
        return len(self.re)

    @property
    def amplitudes(self) -> np.ndarray:
        return self.re + 1j * self.im


@dataclass
class CollapsedState:
    """CollapsedState (state.hpp:66-72)."""

    n_qubits: int
    basis_index: int

    def bitstring(self) -> str:
        return "".join("1" if (self.basis_index >> (self.n_qubits - 1 - q)) & 1 else "0"
                       for q in range(self.n_qubits))


@dataclass
class SimulatorOptions:
    """SimulatorOptions (simulator.hpp:53-56)."""

    qubit_guard: Optional[int] = None


class Simulator:
    """Simulator (simulator.hpp:32-51)."""

    def name(self) -> str:
        raise NotImplementedError

    def qubit_guard(self) -> int:
        raise NotImplementedError

    def simulate_full_state(self, circuit: Circuit, registry: Optional[GateRegistry] = None) -> StateVector:
        raise NotImplementedError

    def simulate_and_collapse(self, circuit: Circuit, registry: Optional[GateRegistry],
                              seed: int) -> CollapsedState:
        raise NotImplementedError


class Plan:
    """A device-resident compiled circuit for rows [row_begin, row_begin+row_count)
    of U (qsb_plan_*). Used by the benchmark and the multi-GPU row sharding."""

    def __init__(self, sim: "B200UnitarySimulator", flat: native.FlatCircuit, row_begin: int, row_count: int):
        self._flat = flat
        self._sim = sim
        self.columns = bool(sim.flags & native.FLAG_COLUMN_BLOCKS)
        self._p = ctypes.c_void_p()
        native.check(native.lib().qsb_plan_create(sim._h, flat.ptr, row_begin, row_count, ctypes.byref(self._p)))
        self.info = native.QsbPlanInfo()
        native.check(native.lib().qsb_plan_get_info(self._p, ctypes.byref(self.info)))

    def set_timing(self, enable) -> None:
        """False/0 off, True/1 phase events, 2 also an event pair around every K2 launch."""
        native.check(native.lib().qsb_plan_set_timing(self._p, int(enable)))

    def gemm_times(self) -> Tuple[List[float], List[int]]:
        """Per-K2-launch ms and kind bits (1 real, 2 materialised, 4 4M) of the last mode-2 execute."""
        count = ctypes.c_int32()
        native.check(native.lib().qsb_plan_gemm_times(self._p, None, None, 0, ctypes.byref(count)))
        ms = np.zeros(max(count.value, 1))
        kinds = np.zeros(max(count.value, 1), dtype=np.int32)
        native.check(native.lib().qsb_plan_gemm_times(self._p, native.dptr(ms), native.dptr(kinds), count.value,
                                                      ctypes.byref(count)))
        return ms[:count.value].tolist(), kinds[:count.value].tolist()

    def allgather_unitary(self, comm: "Comm", dst_re_ptr: int, dst_im_ptr: int, stream: int = 0) -> None:
        """ncclAllGather of every rank's rows of U into full N x N device planes (qsb_plan_allgather_unitary)."""
        native.check(native.lib().qsb_plan_allgather_unitary(self._p, comm._c, dst_re_ptr, dst_im_ptr,
                                                             stream or None))

    def allgather_state(self, comm: "Comm", dst_re_ptr: int, dst_im_ptr: int, stream: int = 0) -> None:
        """ncclAllGather of every rank's psi rows into full-length device planes (qsb_plan_allgather_state)."""
        native.check(native.lib().qsb_plan_allgather_state(self._p, comm._c, dst_re_ptr, dst_im_ptr, stream or None))

    def set_initial_state(self, re_ptr: int, im_ptr: int, stream: int = 0) -> None:
        native.check(native.lib().qsb_plan_set_initial_state(self._p, re_ptr, im_ptr, stream or None))

    def execute(self, stream: int = 0) -> None:
        native.check(native.lib().qsb_plan_execute(self._p, stream or None))

    def copy_state(self, dst_re_ptr: int, dst_im_ptr: int, stream: int = 0) -> None:
        native.check(native.lib().qsb_plan_copy_state(self._p, dst_re_ptr, dst_im_ptr, stream or None))

    def unitary_device(self) -> Tuple[int, int]:
        re, im = ctypes.c_void_p(), ctypes.c_void_p()
        native.check(native.lib().qsb_plan_unitary_device(self._p, ctypes.byref(re), ctypes.byref(im)))
        return re.value, im.value

    def state_device(self) -> Tuple[int, int]:
        re, im = ctypes.c_void_p(), ctypes.c_void_p()
        native.check(native.lib().qsb_plan_state_device(self._p, ctypes.byref(re), ctypes.byref(im)))
        return re.value, im.value

    def last_timing(self) -> Tuple[float, float, float]:
        t, g, m = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        native.check(native.lib().qsb_plan_last_timing(self._p, ctypes.byref(t), ctypes.byref(g), ctypes.byref(m)))
        return t.value, g.value, m.value

    def close(self) -> None:
        if self._p:
            native.lib().qsb_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _state_planes(re, im, dim: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """Contiguous float64 re/im planes of equal length (= dim when given). The C ABI
    carries no lengths, so a short plane would be a host out-of-bounds read: raise
    ShapeError like the reference's matvec (linalg.cpp:89-94) instead."""
    re = np.ascontiguousarray(re, dtype=np.float64).reshape(-1)
    im = np.ascontiguousarray(im, dtype=np.float64).reshape(-1)
    if len(re) != len(im):
        raise ShapeError(f"state planes differ in length: {len(re)} real vs {len(im)} imaginary")
    if dim is not None and len(re) != dim:
        raise ShapeError(f"matvec: {dim}x{dim} times vector of length {len(re)}")
    return re, im


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through libqsb (rank 0; broadcast the bytes to the other ranks)."""
    buf = ctypes.create_string_buffer(native.NCCL_ID_BYTES)
    native.check(native.lib().qsb_nccl_unique_id(buf))
    return buf.raw


def nccl_version() -> int:
    v = ctypes.c_int32()
    native.check(native.lib().qsb_nccl_version(ctypes.byref(v)))
    return v.value


class Comm:
    """An NCCL communicator of one process per GPU (qsb_comm_create on the handle's device)."""

    def __init__(self, sim: "B200UnitarySimulator", unique_id: bytes, n_ranks: int, rank: int) -> None:
        if len(unique_id) != native.NCCL_ID_BYTES:
            raise ValueError("an NCCL unique id has 128 bytes")
        self._id = ctypes.create_string_buffer(unique_id, native.NCCL_ID_BYTES)
        self._c = ctypes.c_void_p()
        native.check(native.lib().qsb_comm_create(sim._h, self._id, n_ranks, rank, ctypes.byref(self._c)))
        self.n_ranks, self.rank = n_ranks, rank

    def close(self) -> None:
        if self._c:
            native.check(native.lib().qsb_comm_destroy(self._c))
            self._c = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class B200UnitarySimulator(Simulator):
    """The drop-in backend: Algorithm 1 on B200 (unitary_backend.cpp:194-215)."""

    def __init__(self, qubit_guard: Optional[int] = None, device: int = 0,
                 gemm_mode: int = native.GEMM_AUTO, flags: int = 0, devices: Optional[List[int]] = None) -> None:
        L = native.lib()
        self._devices = None
        dev_ptr, n_dev = None, 0
        if devices:
            self._devices = (ctypes.c_int32 * len(devices))(*devices)
            dev_ptr, n_dev = ctypes.cast(self._devices, ctypes.c_void_p).value, len(devices)
        opts = native.QsbOptions(device, int(qubit_guard or 0), gemm_mode, flags, n_dev, 0, dev_ptr)
        self._h = ctypes.c_void_p()
        native.check(L.qsb_create(ctypes.byref(opts), ctypes.byref(self._h)))
        g = ctypes.c_int32()
        native.check(L.qsb_qubit_guard(self._h, ctypes.byref(g)))
        self._guard = g.value
        self.device = device
        self.flags = flags

    def name(self) -> str:
        return BACKEND_ID

    def qubit_guard(self) -> int:
        return self._guard

    @staticmethod
    def _flat(circuit, registry):
        return circuit if isinstance(circuit, native.FlatCircuit) else native.flatten(circuit, registry)

    def simulate_full_state(self, circuit, registry: Optional[GateRegistry] = None) -> StateVector:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        re = np.empty(N)
        im = np.empty(N)
        native.check(native.lib().qsb_simulate_full_state(self._h, flat.ptr, native.dptr(re), native.dptr(im)))
        return StateVector(flat.n_qubits, re, im)

    def simulate_full_state_sharded(self, circuit, registry, comm: "Comm") -> StateVector:
        """One process per GPU: this rank's row block of U, psi all-gathered over NCCL
        (qsb_simulate_full_state_sharded); every rank returns the whole psi."""
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        re = np.empty(N)
        im = np.empty(N)
        native.check(native.lib().qsb_simulate_full_state_sharded(self._h, comm._c, flat.ptr, native.dptr(re),
                                                                  native.dptr(im)))
        return StateVector(flat.n_qubits, re, im)

    def simulate_from_state(self, circuit, registry, psi0_re: np.ndarray, psi0_im: np.ndarray) -> StateVector:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        r0, i0 = _state_planes(psi0_re, psi0_im, N)
        re = np.empty(N)
        im = np.empty(N)
        native.check(native.lib().qsb_simulate_from_state(self._h, flat.ptr, native.dptr(r0), native.dptr(i0),
                                                          native.dptr(re), native.dptr(im)))
        return StateVector(flat.n_qubits, re, im)

    def simulate_and_collapse(self, circuit, registry: Optional[GateRegistry], seed: int) -> CollapsedState:
        flat = self._flat(circuit, registry)
        idx = ctypes.c_uint64()
        native.check(native.lib().qsb_simulate_and_collapse(self._h, flat.ptr, ctypes.c_uint64(seed),
                                                            ctypes.byref(idx)))
        return CollapsedState(flat.n_qubits, idx.value)

    def build_unitary(self, circuit, registry: Optional[GateRegistry] = None) -> Tuple[np.ndarray, np.ndarray]:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        re = np.empty((N, N))
        im = np.empty((N, N))
        native.check(native.lib().qsb_build_unitary(self._h, flat.ptr, native.dptr(re), native.dptr(im)))
        return re, im

    def layer_operator(self, circuit, registry, step: int, layer: int) -> Tuple[np.ndarray, np.ndarray]:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        re = np.empty((N, N))
        im = np.empty((N, N))
        native.check(native.lib().qsb_layer_operator(self._h, flat.ptr, step, layer, native.dptr(re),
                                                     native.dptr(im)))
        return re, im

    def probabilities(self, re: np.ndarray, im: np.ndarray) -> Tuple[np.ndarray, float]:
        re, im = _state_planes(re, im)
        p = np.empty(len(re))
        norm = ctypes.c_double()
        native.check(native.lib().qsb_probabilities(self._h, native.dptr(re), native.dptr(im), len(re),
                                                    native.dptr(p), ctypes.byref(norm)))
        return p, norm.value

    def plan(self, circuit, registry=None, row_begin: int = 0, row_count: Optional[int] = None) -> Plan:
        flat = self._flat(circuit, registry)
        if row_count is None:
            row_count = (1 << flat.n_qubits) - row_begin
        return Plan(self, flat, row_begin, row_count)

    def close(self) -> None:
        if getattr(self, "_h", None):
            native.lib().qsb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SvPlan:
    """A device-resident state-vector-engine plan (qsb_sv_plan_*): the fsv
    backend (mode SV_STATE) or columns [col_begin, col_begin+col_count) of the
    structured unitary (mode SV_UNITARY)."""

    def __init__(self, sim: "_HandleOwner", flat: native.FlatCircuit, mode: int, col_begin: int, col_count: int):
        self._flat = flat
        self._sim = sim
        self._p = ctypes.c_void_p()
        native.check(native.lib().qsb_sv_plan_create(sim._h, flat.ptr, mode, col_begin, col_count,
                                                     ctypes.byref(self._p)))
        self.info = native.QsbSvPlanInfo()
        native.check(native.lib().qsb_sv_plan_get_info(self._p, ctypes.byref(self.info)))

    def set_state(self, re_ptr: int, im_ptr: int, stream: int = 0) -> None:
        native.check(native.lib().qsb_sv_plan_set_state(self._p, re_ptr, im_ptr, stream or None))

    def execute(self, stream: int = 0) -> None:
        native.check(native.lib().qsb_sv_plan_execute(self._p, stream or None))

    def result_device(self) -> Tuple[int, int]:
        re, im = ctypes.c_void_p(), ctypes.c_void_p()
        native.check(native.lib().qsb_sv_plan_result_device(self._p, ctypes.byref(re), ctypes.byref(im)))
        return re.value, im.value

    def close(self) -> None:
        if self._p:
            native.lib().qsb_sv_plan_destroy(self._p)
            self._p = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _HandleOwner(Simulator):
    """Owns one qsb_handle (qsb_create / qsb_destroy)."""

    def __init__(self, qubit_guard: Optional[int] = None, device: int = 0,
                 gemm_mode: int = native.GEMM_AUTO, flags: int = 0, devices: Optional[List[int]] = None) -> None:
        L = native.lib()
        self._devices = None
        dev_ptr, n_dev = None, 0
        if devices:
            self._devices = (ctypes.c_int32 * len(devices))(*devices)
            dev_ptr, n_dev = ctypes.cast(self._devices, ctypes.c_void_p).value, len(devices)
        opts = native.QsbOptions(device, int(qubit_guard or 0), gemm_mode, flags, n_dev, 0, dev_ptr)
        self._h = ctypes.c_void_p()
        native.check(L.qsb_create(ctypes.byref(opts), ctypes.byref(self._h)))
        self.device = device

    @staticmethod
    def _flat(circuit, registry):
        return circuit if isinstance(circuit, native.FlatCircuit) else native.flatten(circuit, registry)

    def _guard_of(self, fn) -> int:
        g = ctypes.c_int32()
        native.check(fn(self._h, ctypes.byref(g)))
        return g.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            native.lib().qsb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class B200FsvSimulator(_HandleOwner):
    """FsvSimulator (fsv_backend.hpp:41-58, fsv_backend.cpp:135-158) on B200:
    every operation applied to the state in circuit order, batched into
    shared-memory passes. Bit-exact with the reference's fsv backend."""

    def name(self) -> str:
        return FSV_BACKEND_ID

    def qubit_guard(self) -> int:
        return self._guard_of(native.lib().qsb_fsv_qubit_guard)

    def simulate_full_state(self, circuit, registry: Optional[GateRegistry] = None) -> StateVector:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        re = np.empty(N)
        im = np.empty(N)
        native.check(native.lib().qsb_fsv_simulate_full_state(self._h, flat.ptr, native.dptr(re), native.dptr(im)))
        return StateVector(flat.n_qubits, re, im)

    def simulate_from_state(self, circuit, registry, psi0_re: np.ndarray, psi0_im: np.ndarray) -> StateVector:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        r0, i0 = _state_planes(psi0_re, psi0_im, N)
        re = np.empty(N)
        im = np.empty(N)
        native.check(native.lib().qsb_fsv_simulate_from_state(self._h, flat.ptr, native.dptr(r0), native.dptr(i0),
                                                              native.dptr(re), native.dptr(im)))
        return StateVector(flat.n_qubits, re, im)

    def simulate_and_collapse(self, circuit, registry: Optional[GateRegistry], seed: int) -> CollapsedState:
        # Simulator::simulate_and_collapse default (simulator.cpp:26-30): full state, then collapse
        st = self.simulate_full_state(circuit, registry)
        return CollapsedState(st.n_qubits, _collapse_on(self, st.re, st.im, seed))

    def plan(self, circuit, registry=None) -> SvPlan:
        return SvPlan(self, self._flat(circuit, registry), native.SV_STATE, 0, 1)


class B200StructuredUnitarySimulator(_HandleOwner):
    """Unitary simulation without dense GEMMs: U[:, c] = fsv(e_c) for every
    column c, all columns evolved at once by the state-vector engine (columns
    sharded over devices). A different algorithm from Algorithm 1's dense
    products — same U within rounding, reported separately."""

    def name(self) -> str:
        return STRUCTURED_BACKEND_ID

    def qubit_guard(self) -> int:
        return self._guard_of(native.lib().qsb_structured_qubit_guard)

    def simulate_full_state(self, circuit, registry: Optional[GateRegistry] = None) -> StateVector:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        re = np.empty(N)
        im = np.empty(N)
        native.check(native.lib().qsb_structured_simulate_full_state(self._h, flat.ptr, native.dptr(re),
                                                                     native.dptr(im)))
        return StateVector(flat.n_qubits, re, im)

    def simulate_and_collapse(self, circuit, registry: Optional[GateRegistry], seed: int) -> CollapsedState:
        st = self.simulate_full_state(circuit, registry)
        return CollapsedState(st.n_qubits, _collapse_on(self, st.re, st.im, seed))

    def build_unitary(self, circuit, registry: Optional[GateRegistry] = None) -> Tuple[np.ndarray, np.ndarray]:
        flat = self._flat(circuit, registry)
        N = 1 << flat.n_qubits
        re = np.empty((N, N))
        im = np.empty((N, N))
        native.check(native.lib().qsb_structured_build_unitary(self._h, flat.ptr, native.dptr(re), native.dptr(im)))
        return re, im

    def plan(self, circuit, registry=None, col_begin: int = 0, col_count: Optional[int] = None) -> SvPlan:
        flat = self._flat(circuit, registry)
        if col_count is None:
            col_count = (1 << flat.n_qubits) - col_begin
        return SvPlan(self, flat, native.SV_UNITARY, col_begin, col_count)


def _collapse_on(sim: "_HandleOwner", re: np.ndarray, im: np.ndarray, seed: int) -> int:
    """collapse (state.cpp:81-98) through qsb_collapse: K4 probabilities on the
    GPU, sequential inverse-CDF walk in the native runtime."""
    re, im = _state_planes(re, im)
    idx = ctypes.c_uint64()
    native.check(native.lib().qsb_collapse(sim._h, native.dptr(re), native.dptr(im), len(re), ctypes.c_uint64(seed),
                                           ctypes.byref(idx)))
    return idx.value


def is_unitary(sim, m: np.ndarray, tol: float) -> Tuple[bool, float]:
    """is_unitary (linalg.cpp:131-155) on the GPU through qsb_is_unitary:
    (verdict, max |(A^H A - I)_ij|). `sim` is any backend owning a handle."""
    m = np.asarray(m, dtype=np.complex128)
    re = np.ascontiguousarray(m.real)
    im = np.ascontiguousarray(m.imag)
    ok = ctypes.c_int32()
    dev = ctypes.c_double()
    native.check(native.lib().qsb_is_unitary(sim._h, native.dptr(re), native.dptr(im), m.shape[0], tol,
                                             ctypes.byref(ok), ctypes.byref(dev)))
    return bool(ok.value), dev.value


def gpu_unitarity_check(sim):
    """A GateRegistry unitarity check (circuit.set_unitarity_check) running on `sim`'s GPU."""
    return lambda m, tol: is_unitary(sim, m, tol)[0]


class _CudaArray:
    """Minimal __cuda_array_interface__ holder for a raw device pointer."""

    def __init__(self, ptr: int, shape, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def torch_view(ptr: int, shape, device: Optional[int] = None):
    """Zero-copy torch float64 view of device memory owned by a plan (valid until
    the plan is destroyed or re-executed)."""
    import torch

    return torch.as_tensor(_CudaArray(ptr, shape), device=f"cuda:{device or 0}")


def step_layer_count(circuit, registry, step: int) -> int:
    flat = circuit if isinstance(circuit, native.FlatCircuit) else native.flatten(circuit, registry)
    n = ctypes.c_int32()
    native.check(native.lib().qsb_step_layer_count(flat.ptr, step, ctypes.byref(n)))
    return n.value


# ---- backend registry (simulator.cpp:32-82) ----

SimulatorFactory = Callable[[SimulatorOptions], Simulator]
_lock = threading.Lock()
_factories: Dict[str, SimulatorFactory] = {
    BACKEND_ID: lambda o: B200UnitarySimulator(qubit_guard=o.qubit_guard),
    FSV_BACKEND_ID: lambda o: B200FsvSimulator(qubit_guard=o.qubit_guard),
    STRUCTURED_BACKEND_ID: lambda o: B200StructuredUnitarySimulator(qubit_guard=o.qubit_guard),
}


def make_simulator(backend_id: str, options: Optional[SimulatorOptions] = None) -> Simulator:
    with _lock:
        f = _factories.get(backend_id)
    if f is None:
        raise LookupError_(f"unknown backend '{backend_id}'")
    return f(options or SimulatorOptions())


def register_backend(backend_id: str, factory: SimulatorFactory) -> None:
    with _lock:
        _factories[backend_id] = factory


def backend_names() -> List[str]:
    with _lock:
        return sorted(_factories)


def memory_estimate(n_qubits: int, kind: int = 0) -> int:
    return int(native.lib().qsb_memory_estimate(n_qubits, kind))


def engine_memory_estimate(n_qubits: int, kind: int = 0) -> int:
    return int(native.lib().qsb_engine_memory_estimate(n_qubits, kind))
