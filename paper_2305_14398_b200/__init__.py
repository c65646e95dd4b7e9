"""B200-native unitary-simulation hot path of TornadoQSim (arXiv 2305.14398).

The product is ``libqsb.so`` (C ABI in ``include/qsb.h``: sm_100a kernels + C++
runtime). This package mirrors the reference's host-side interface so callers
and tests read like the reference's own: the circuit model and gate library
(``circuit``, ``circuit_library``), the Simulator plugin registry
(``simulator``), and the error hierarchy (``errors``).
"""
from .circuit import (Circuit, ControlGate, FunctionOp, Gate, GateRegistry, GateTag, GateType, Instruction,
                      InstructionKind, Step, controlled_unitary, gate_matrix, touched_qubits)
from .circuit_library import (bell, deutsch_jozsa, fully_entangled, make_named_circuit, oracle_matrix,
                              parse_oracle_spec, qft)
from .errors import (ArgumentError, DeviceError, Error, LookupError_, ResourceError, ShapeError,
                     ValidationError)

__all__ = [
    "Circuit", "ControlGate", "FunctionOp", "Gate", "GateRegistry", "GateTag", "GateType", "Instruction",
    "InstructionKind", "Step", "controlled_unitary", "gate_matrix", "touched_qubits", "bell", "deutsch_jozsa",
    "fully_entangled", "make_named_circuit", "oracle_matrix", "parse_oracle_spec", "qft", "ArgumentError",
    "DeviceError", "Error", "LookupError_", "ResourceError", "ShapeError", "ValidationError",
]
