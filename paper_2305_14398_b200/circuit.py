"""Host-side mirror of the reference circuit model and gate library.

Mirrors, name for name, the reference C++ types a caller builds circuits with
(paths relative to /root/reference/proj):

* ``GateTag`` / ``GateType``             core/include/qsim/circuit.hpp:28-47, core/src/circuit.cpp:26-46
* ``Gate``, ``ControlGate``, ``FunctionOp``, ``Instruction``, ``Operation``
                                          circuit.hpp:49-79
* ``touched_qubits``                     core/src/circuit.cpp:46-63
* ``Step``, ``Circuit`` (greedy last-step packing)
                                          circuit.hpp:83-133, circuit.cpp:65-156
* ``gate_matrix``, ``controlled_unitary``, ``GateRegistry``
                                          core/src/gates.cpp:27-137

Gate matrices are computed with the C library's ``cos``/``sin``/``sqrt`` (via
``math``), so they are bit-identical to the reference's ``gate_matrix``.
Matrices are numpy complex128 arrays here; the ABI flattener splits them into
re/im planes (the ComplexMatrix storage, linalg.hpp:39-70).
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import List, Union

import numpy as np

from .errors import ArgumentError, LookupError_, ValidationError

#: kDefaultQubitCap (circuit.hpp:90)
DEFAULT_QUBIT_CAP = 24
#: kRegistryUnitaryTol (gates.hpp:32)
REGISTRY_UNITARY_TOL = 1e-9


class GateTag(enum.IntEnum):
    """GateTag (circuit.hpp:31); values match the ABI's QSB_GATE_*."""

    H = 0
    X = 1
    Y = 2
    Z = 3
    S = 4
    T = 5
    R = 6


@dataclass(frozen=True)
class GateType:
    """GateType (circuit.hpp:33-47)."""

    tag: GateTag = GateTag.H
    phi: float = 0.0

    @staticmethod
    def h() -> "GateType":
        return GateType(GateTag.H)

    @staticmethod
    def x() -> "GateType":
        return GateType(GateTag.X)

    @staticmethod
    def y() -> "GateType":
        return GateType(GateTag.Y)

    @staticmethod
    def z() -> "GateType":
        return GateType(GateTag.Z)

    @staticmethod
    def s() -> "GateType":
        return GateType(GateTag.S)

    @staticmethod
    def t() -> "GateType":
        return GateType(GateTag.T)

    @staticmethod
    def r(phi: float) -> "GateType":
        """circuit.cpp:26-31: non-finite phi is an ArgumentError."""
        if not math.isfinite(phi):
            raise ArgumentError("phase gate: phi must be finite")
        return GateType(GateTag.R, float(phi))

    def name(self) -> str:
        return self.tag.name


class InstructionKind(enum.IntEnum):
    """InstructionKind (circuit.hpp:49); values match QSB_INSTR_*."""

    MEASURE = 0
    RESET = 1


@dataclass(frozen=True)
class Gate:
    gate: GateType
    target: int


@dataclass(frozen=True)
class ControlGate:
    gate: GateType
    control: int
    target: int


@dataclass(frozen=True)
class FunctionOp:
    name: str
    first_qubit: int
    qubit_count: int


@dataclass(frozen=True)
class Instruction:
    kind: InstructionKind
    target: int


Operation = Union[Gate, ControlGate, FunctionOp, Instruction]


def touched_qubits(op: Operation) -> List[int]:
    """circuit.cpp:46-63: sorted qubits an operation acts on (control gates
    touch only control and target, not the span between them)."""
    if isinstance(op, (Gate, Instruction)):
        return [op.target]
    if isinstance(op, ControlGate):
        return sorted([op.control, op.target])
    return list(range(op.first_qubit, op.first_qubit + op.qubit_count))


@dataclass
class Step:
    operations: List[Operation] = field(default_factory=list)


# ----------------------------------------------------------------- gates


def _phase_matrix(phi: float) -> np.ndarray:
    """gates.cpp:27-36."""
    if not math.isfinite(phi):
        raise ArgumentError("phase gate: phi must be finite")
    m = np.zeros((2, 2), dtype=np.complex128)
    m[0, 0] = 1.0
    m[1, 1] = complex(math.cos(phi), math.sin(phi))
    return m


def gate_matrix(g: GateType) -> np.ndarray:
    """gates.cpp:40-77."""
    m = np.zeros((2, 2), dtype=np.complex128)
    if g.tag == GateTag.H:
        s = math.sqrt(0.5)
        m[:] = [[s, s], [s, -s]]
        return m
    if g.tag == GateTag.X:
        m[0, 1] = 1.0
        m[1, 0] = 1.0
        return m
    if g.tag == GateTag.Y:
        m[0, 1] = complex(0.0, -1.0)
        m[1, 0] = complex(0.0, 1.0)
        return m
    if g.tag == GateTag.Z:
        m[0, 0] = 1.0
        m[1, 1] = -1.0
        return m
    if g.tag == GateTag.S:
        return _phase_matrix(math.pi / 2.0)
    if g.tag == GateTag.T:
        return _phase_matrix(math.pi / 4.0)
    if g.tag == GateTag.R:
        return _phase_matrix(g.phi)
    raise ArgumentError("unknown gate tag")


def controlled_unitary(u: np.ndarray, control_pos: int, target_pos: int, span: int) -> np.ndarray:
    """gates.cpp:79-110 (host reference only; the GPU generates these entries)."""
    if u.shape != (2, 2):
        from .errors import ShapeError

        raise ShapeError("controlled_unitary: u must be 2x2")
    if span < 2 or span > 30:
        raise ArgumentError("controlled_unitary: span must be in [2, 30]")
    if control_pos == target_pos or control_pos >= span or target_pos >= span:
        raise ArgumentError("controlled_unitary: invalid control/target positions")
    dim = 1 << span
    cmask = 1 << (span - 1 - control_pos)
    tmask = 1 << (span - 1 - target_pos)
    m = np.zeros((dim, dim), dtype=np.complex128)
    for col in range(dim):
        if (col & cmask) == 0:
            m[col, col] = 1.0
            continue
        tbit = 1 if (col & tmask) else 0
        m[col & ~tmask, col] = u[0, tbit]
        m[col | tmask, col] = u[1, tbit]
    return m


def _is_unitary(m: np.ndarray, tol: float) -> bool:
    """linalg.cpp:131-155: max |(A^dagger A - I)_ij| per re/im part <= tol."""
    prod = m.conj().T @ m
    prod -= np.eye(m.shape[0])
    return bool(np.all(np.abs(prod.real) <= tol) and np.all(np.abs(prod.imag) <= tol))


# The unitarity check GateRegistry.register_function runs (gates.cpp:121). The
# default is the host restatement above; set_unitarity_check() routes it to the
# GPU (simulator.gpu_unitarity_check: qsb_is_unitary, A^H A on the DMMA pipe).
_unitarity_check = _is_unitary


def set_unitarity_check(fn) -> None:
    """fn(m: complex ndarray, tol: float) -> bool, or None for the host default."""
    global _unitarity_check
    _unitarity_check = fn if fn is not None else _is_unitary


class GateRegistry:
    """GateRegistry (gates.hpp:45-60, gates.cpp:112-137)."""

    def __init__(self) -> None:
        self._entries: dict = {}

    def register_function(self, name: str, m: np.ndarray) -> None:
        m = np.asarray(m, dtype=np.complex128)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise ValidationError(f"registry: matrix for '{name}' is not square")
        n = m.shape[0]
        if n < 2 or (n & (n - 1)) != 0:
            raise ValidationError(
                f"registry: matrix dimension for '{name}' must be a power of two >= 2, got {n}")
        if not _unitarity_check(m, REGISTRY_UNITARY_TOL):
            raise ValidationError(f"registry: matrix for '{name}' is not unitary")
        self._entries[name] = np.ascontiguousarray(m)

    def lookup(self, name: str) -> np.ndarray:
        try:
            return self._entries[name]
        except KeyError:
            raise LookupError_(f"registry: no function named '{name}'") from None

    def contains(self, name: str) -> bool:
        return name in self._entries


# --------------------------------------------------------------- circuit


class Circuit:
    """Circuit (circuit.hpp:95-133): ordered steps over a fixed qubit count,
    built by greedy packing into the LAST step (circuit.cpp:81-103)."""

    def __init__(self, n_qubits: int, qubit_cap: int = DEFAULT_QUBIT_CAP) -> None:
        if n_qubits < 1 or n_qubits > qubit_cap:
            raise ArgumentError(f"circuit qubit count must be in [1, {qubit_cap}], got {n_qubits}")
        self._n = int(n_qubits)
        self._steps: List[Step] = []

    def qubit_count(self) -> int:
        return self._n

    def steps(self) -> List[Step]:
        return self._steps

    def _check_qubit(self, q: int) -> None:
        if q < 0 or q >= self._n:
            raise ArgumentError(f"qubit index {q} out of range for a {self._n}-qubit circuit")

    def _append(self, op: Operation) -> None:
        qubits = touched_qubits(op)
        if self._steps:
            free = True
            for existing in self._steps[-1].operations:
                used = touched_qubits(existing)
                if any(q in used for q in qubits):
                    free = False
                    break
            if free:
                self._steps[-1].operations.append(op)
                return
        self._steps.append(Step([op]))

    def add_gate(self, g: GateType, target: int) -> "Circuit":
        self._check_qubit(target)
        self._append(Gate(g, target))
        return self

    def add_control_gate(self, g: GateType, control: int, target: int) -> "Circuit":
        self._check_qubit(control)
        self._check_qubit(target)
        if control == target:
            raise ArgumentError("control gate: control and target must differ")
        self._append(ControlGate(g, control, target))
        return self

    def add_function(self, name: str, first_qubit: int, qubit_count: int,
                     registry: GateRegistry) -> "Circuit":
        if qubit_count < 1:
            raise ArgumentError("function must span at least one qubit")
        self._check_qubit(first_qubit)
        if first_qubit + qubit_count > self._n:
            raise ArgumentError(
                f"function range [{first_qubit}, {first_qubit + qubit_count}) exceeds circuit size")
        m = registry.lookup(name)
        want = 1 << qubit_count
        if m.shape[0] != want:
            raise ValidationError(
                f"function '{name}' is registered with dimension {m.shape[0]}, expected {want} "
                f"for {qubit_count} qubits")
        self._append(FunctionOp(name, first_qubit, qubit_count))
        return self

    def add_instruction(self, kind: InstructionKind, target: int) -> "Circuit":
        self._check_qubit(target)
        self._append(Instruction(InstructionKind(kind), target))
        return self

    def h(self, q: int) -> "Circuit":
        return self.add_gate(GateType.h(), q)

    def x(self, q: int) -> "Circuit":
        return self.add_gate(GateType.x(), q)

    def y(self, q: int) -> "Circuit":
        return self.add_gate(GateType.y(), q)

    def z(self, q: int) -> "Circuit":
        return self.add_gate(GateType.z(), q)

    def s(self, q: int) -> "Circuit":
        return self.add_gate(GateType.s(), q)

    def t(self, q: int) -> "Circuit":
        return self.add_gate(GateType.t(), q)

    def r(self, phi: float, q: int) -> "Circuit":
        return self.add_gate(GateType.r(phi), q)

    def cnot(self, c: int, t: int) -> "Circuit":
        return self.add_control_gate(GateType.x(), c, t)

    def cr(self, phi: float, c: int, t: int) -> "Circuit":
        return self.add_control_gate(GateType.r(phi), c, t)

    def measure(self, q: int) -> "Circuit":
        return self.add_instruction(InstructionKind.MEASURE, q)

    def reset(self, q: int) -> "Circuit":
        return self.add_instruction(InstructionKind.RESET, q)

    def flatten(self) -> List[Operation]:
        return [op for step in self._steps for op in step.operations]
