"""Workload generators mirroring core/src/circuit_library.cpp (the BASELINE
configs: QFT, Fully Entangled, Deutsch-Jozsa).

* ``bell``                      circuit_library.cpp:27-31
* ``fully_entangled``           :33-43
* ``oracle_matrix``             :45-58
* ``deutsch_jozsa``             :60-80
* ``all_zero_input_probability`` :82-89
* ``qft``                       :91-107
* ``parse_oracle_spec``         :109-150
* ``make_named_circuit``        :152-179 (DJ default oracle ``balanced-bit:0``)
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass
from typing import Callable, Tuple

import numpy as np

from .circuit import Circuit, GateRegistry
from .errors import ArgumentError, LookupError_, ValidationError

BoolFunction = Callable[[int], bool]


def bell() -> Circuit:
    c = Circuit(2)
    c.h(0).cnot(0, 1)
    return c


def fully_entangled(n_qubits: int) -> Circuit:
    if n_qubits < 2:
        raise ArgumentError("fully entangled circuit needs at least 2 qubits")
    c = Circuit(n_qubits)
    c.h(0)
    for target in range(n_qubits - 1, 0, -1):
        c.cnot(0, target)
    return c


def oracle_matrix(n_inputs: int, f: BoolFunction) -> np.ndarray:
    """|x, y> -> |x, y xor f(x)> over n_inputs + 1 qubits (ancilla = LSB)."""
    if n_inputs < 1:
        raise ArgumentError("oracle needs at least one input bit")
    dim = 1 << (n_inputs + 1)
    cols = np.arange(dim, dtype=np.int64)
    x = cols >> 1
    y = cols & 1
    fx = np.fromiter((1 if f(int(v)) else 0 for v in range(dim >> 1)), dtype=np.int64, count=dim >> 1)
    rows = (x << 1) | (y ^ fx[x])
    m = np.zeros((dim, dim), dtype=np.complex128)
    m[rows, cols] = 1.0
    return m


@dataclass
class DeutschJozsaProgram:
    circuit: Circuit
    registry: GateRegistry


def deutsch_jozsa(n_inputs: int, f: BoolFunction) -> DeutschJozsaProgram:
    n = n_inputs + 1
    ancilla = n_inputs
    registry = GateRegistry()
    registry.register_function("oracle", oracle_matrix(n_inputs, f))
    c = Circuit(n)
    c.x(ancilla)
    for q in range(n):
        c.h(q)
    c.add_function("oracle", 0, n, registry)
    for q in range(n_inputs):
        c.h(q)
    for q in range(n_inputs):
        c.measure(q)
    return DeutschJozsaProgram(c, registry)


def all_zero_input_probability(psi_re: np.ndarray, psi_im: np.ndarray, n_inputs: int) -> float:
    if (1 << (n_inputs + 1)) != len(psi_re):
        raise ArgumentError("state does not match the oracle's qubit count")
    p = psi_re * psi_re + psi_im * psi_im
    return float(p[0] + p[1])


def qft(n_qubits: int) -> Circuit:
    if n_qubits < 1:
        raise ArgumentError("qft needs at least one qubit")
    c = Circuit(n_qubits)
    for k in range(n_qubits):
        c.h(k)
        j = 1
        while j + k < n_qubits:
            c.cr(math.ldexp(math.pi, -j), k + j, k)
            j += 1
    for q in range(n_qubits // 2):
        p = n_qubits - 1 - q
        c.cnot(q, p).cnot(p, q).cnot(q, p)
    return c


@dataclass
class Oracle:
    name: str
    fn: BoolFunction


def parse_oracle_spec(spec: str, n_inputs: int) -> Oracle:
    if n_inputs < 1 or n_inputs > 63:
        raise ArgumentError("oracle input count must be in [1, 63]")
    if spec == "constant0":
        return Oracle("constant0", lambda x: False)
    if spec == "constant1":
        return Oracle("constant1", lambda x: True)
    if spec.startswith("balanced-bit:"):
        arg = spec[13:]
        if not re.fullmatch(r"[0-9]+", arg) or int(arg) >= n_inputs:
            raise ArgumentError(f"balanced-bit oracle: bit index must be below {n_inputs}")
        shift = n_inputs - 1 - int(arg)
        return Oracle(spec, lambda x, s=shift: ((x >> s) & 1) != 0)
    if spec.startswith("balanced-mask:"):
        arg = spec[14:]
        if not re.fullmatch(r"[0-9a-fA-F]+", arg):
            raise ArgumentError("balanced-mask oracle: expected a hex mask")
        mask = int(arg, 16)
        if mask == 0 or (n_inputs < 64 and mask >= (1 << n_inputs)):
            raise ArgumentError(f"balanced-mask oracle: mask must be nonzero and fit {n_inputs} bits")
        return Oracle(spec, lambda x, m=mask: (bin(x & m).count("1") & 1) != 0)
    raise ValidationError(
        f"unknown oracle spec '{spec}' (expected constant0, constant1, balanced-bit:<k> or "
        "balanced-mask:<hex>)")


def make_named_circuit(name: str, qubits: int, oracle_spec: str = "") -> Tuple[Circuit, GateRegistry]:
    """Returns (circuit, registry) like GeneratedCircuit."""
    if name == "bell":
        if qubits != 2:
            raise ArgumentError("bell is a 2-qubit circuit")
        return bell(), GateRegistry()
    if name == "entangle":
        return fully_entangled(qubits), GateRegistry()
    if name == "deutsch-jozsa":
        if qubits < 2:
            raise ArgumentError("deutsch-jozsa needs at least 2 qubits")
        oracle = parse_oracle_spec(oracle_spec or "balanced-bit:0", qubits - 1)
        prog = deutsch_jozsa(qubits - 1, oracle.fn)
        return prog.circuit, prog.registry
    if name == "qft":
        return qft(qubits), GateRegistry()
    raise LookupError_(f"unknown circuit '{name}' (expected bell, entangle, deutsch-jozsa or qft)")
