// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper over the UNMODIFIED reference library (qsim_core, built
// from /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/).
// It exposes the reference's own public API — circuit generators, the
// reference test support (tests/support/test_util.hpp: random_circuit,
// random_state, circuit_unitary), step_unitary, make_simulator(...)
// ->simulate_full_state, collapse, memory_estimate, matmul — so that
//   * tests/golden/make_golden.py can record golden vectors from the reference,
//   * bench.py --impl reference can time the reference CPU path on the host.
// Nothing here re-implements reference behaviour; it only marshals data.
#include <chrono>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "qsim/circuit.hpp"
#include "qsim/circuit_library.hpp"
#include "qsim/errors.hpp"
#include "qsim/fsv_backend.hpp"
#include "qsim/gates.hpp"
#include "qsim/linalg.hpp"
#include "qsim/parallel.hpp"
#include "qsim/simulator.hpp"
#include "qsim/state.hpp"
#include "qsim/unitary_backend.hpp"
#include "support/test_util.hpp"

#include "../include/qsb.h"

using namespace qsim;

namespace {

thread_local std::string g_err;

struct Program {
    Circuit circuit;
    GateRegistry registry;
};

int code_of(const std::exception& e) {
    if (dynamic_cast<const ResourceError*>(&e)) return 1;
    if (dynamic_cast<const ValidationError*>(&e)) return 2;
    if (dynamic_cast<const ShapeError*>(&e)) return 3;
    if (dynamic_cast<const ArgumentError*>(&e)) return 4;
    if (dynamic_cast<const LookupError*>(&e)) return 5;
    return 8;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

void copy_out(const ComplexMatrix& m, double* re, double* im) {
    std::memcpy(re, m.re_data(), sizeof(double) * m.rows() * m.cols());
    std::memcpy(im, m.im_data(), sizeof(double) * m.rows() * m.cols());
}

GateType gate_type(int32_t tag, double phi) {
    switch (tag) {
    case QSB_GATE_H: return GateType::h();
    case QSB_GATE_X: return GateType::x();
    case QSB_GATE_Y: return GateType::y();
    case QSB_GATE_Z: return GateType::z();
    case QSB_GATE_S: return GateType::s();
    case QSB_GATE_T: return GateType::t();
    default: return GateType::r(phi);
    }
}

// Function names in order of first appearance in the circuit.
std::vector<std::string> function_names(const Circuit& c) {
    std::vector<std::string> names;
    for (const Operation& op : c.flatten()) {
        if (const auto* fn = std::get_if<FunctionOp>(&op)) {
            bool seen = false;
            for (const auto& n : names) seen = seen || n == fn->name;
            if (!seen) names.push_back(fn->name);
        }
    }
    return names;
}

} // namespace

extern "C" {

const char* refsh_last_error() { return g_err.c_str(); }

void refsh_free(void* p) { delete static_cast<Program*>(p); }

// make_named_circuit (circuit_library.cpp:152-179)
void* refsh_named(const char* name, int qubits, const char* oracle_spec) {
    Program* out = nullptr;
    const int rc = guarded([&] {
        GeneratedCircuit g = make_named_circuit(name, static_cast<std::size_t>(qubits),
                                                oracle_spec ? oracle_spec : "");
        out = new Program{std::move(g.circuit), std::move(g.registry)};
    });
    return rc == 0 ? out : nullptr;
}

// Builder over Circuit (circuit.hpp:95-133); returns status codes.
void* refsh_circuit_new(int qubits) {
    Program* out = nullptr;
    guarded([&] { out = new Program{Circuit(static_cast<std::size_t>(qubits)), {}}; });
    return out;
}
int refsh_add_gate(void* p, int32_t tag, double phi, int32_t target) {
    return guarded([&] { static_cast<Program*>(p)->circuit.add_gate(gate_type(tag, phi), target); });
}
int refsh_add_control(void* p, int32_t tag, double phi, int32_t control, int32_t target) {
    return guarded([&] {
        static_cast<Program*>(p)->circuit.add_control_gate(gate_type(tag, phi), control, target);
    });
}
int refsh_add_instruction(void* p, int32_t kind, int32_t target) {
    return guarded([&] {
        static_cast<Program*>(p)->circuit.add_instruction(
            kind == QSB_INSTR_RESET ? InstructionKind::Reset : InstructionKind::Measure, target);
    });
}
int refsh_register_function(void* p, const char* name, int64_t dim, const double* re, const double* im) {
    return guarded([&] {
        ComplexMatrix m(static_cast<std::size_t>(dim), static_cast<std::size_t>(dim));
        std::memcpy(m.re_data(), re, sizeof(double) * dim * dim);
        std::memcpy(m.im_data(), im, sizeof(double) * dim * dim);
        static_cast<Program*>(p)->registry.register_function(name, std::move(m));
    });
}
int refsh_add_function(void* p, const char* name, int32_t first, int32_t count) {
    return guarded([&] {
        auto* prog = static_cast<Program*>(p);
        prog->circuit.add_function(name, first, count, prog->registry);
    });
}

// std::mt19937_64 + the reference test support generators (test_util.hpp:62-132)
void* refsh_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void refsh_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t refsh_rng_uniform_size(void* r, uint64_t lo, uint64_t hi) {
    std::uniform_int_distribution<std::size_t> d(lo, hi);
    return d(*static_cast<std::mt19937_64*>(r));
}
void* refsh_random_circuit(void* r, int qubits, int ops) {
    Program* out = nullptr;
    guarded([&] {
        out = new Program{test::random_circuit(*static_cast<std::mt19937_64*>(r),
                                               static_cast<std::size_t>(qubits),
                                               static_cast<std::size_t>(ops)),
                          {}};
    });
    return out;
}
// The literal expression of acceptance_main.cpp:277 / test bodies that draw the
// qubit and op counts as call arguments (argument evaluation order is the
// compiler's, so it is reproduced by compiling the same expression).
void* refsh_random_circuit_args(void* r, uint64_t qlo, uint64_t qhi, uint64_t olo, uint64_t ohi) {
    Program* out = nullptr;
    guarded([&] {
        auto& rng = *static_cast<std::mt19937_64*>(r);
        std::uniform_int_distribution<std::size_t> qubit_pick(qlo, qhi);
        std::uniform_int_distribution<std::size_t> op_pick(olo, ohi);
        out = new Program{test::random_circuit(rng, qubit_pick(rng), op_pick(rng)), {}};
    });
    return out;
}
int refsh_random_state(void* r, int qubits, double* re, double* im) {
    return guarded([&] {
        StateVector s = test::random_state(*static_cast<std::mt19937_64*>(r), qubits);
        std::memcpy(re, s.amplitudes.re.data(), sizeof(double) * s.dimension());
        std::memcpy(im, s.amplitudes.im.data(), sizeof(double) * s.dimension());
    });
}

int refsh_n_qubits(void* p) { return static_cast<int>(static_cast<Program*>(p)->circuit.qubit_count()); }
int refsh_n_steps(void* p) { return static_cast<int>(static_cast<Program*>(p)->circuit.steps().size()); }
int refsh_n_ops(void* p) { return static_cast<int>(static_cast<Program*>(p)->circuit.flatten().size()); }
int refsh_n_functions(void* p) { return static_cast<int>(function_names(static_cast<Program*>(p)->circuit).size()); }

// Flatten into the ABI format (include/qsb.h); u = gate_matrix(g) (gates.cpp:40-77).
int refsh_serialize(void* p, int32_t* step_offsets, qsb_op* ops) {
    return guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        const auto names = function_names(prog.circuit);
        int32_t k = 0;
        step_offsets[0] = 0;
        int32_t s = 0;
        for (const Step& step : prog.circuit.steps()) {
            for (const Operation& op : step.operations) {
                qsb_op& o = ops[k++];
                std::memset(&o, 0, sizeof o);
                auto put_gate = [&](const GateType& g) {
                    o.gate = static_cast<int32_t>(g.tag);
                    o.phi = g.phi;
                    const ComplexMatrix m = gate_matrix(g);
                    for (int e = 0; e < 4; ++e) {
                        o.u_re[e] = m.re(e / 2, e % 2);
                        o.u_im[e] = m.im(e / 2, e % 2);
                    }
                };
                if (const auto* g = std::get_if<Gate>(&op)) {
                    o.kind = QSB_OP_GATE;
                    o.target = static_cast<int32_t>(g->target);
                    put_gate(g->gate);
                } else if (const auto* cg = std::get_if<ControlGate>(&op)) {
                    o.kind = QSB_OP_CONTROL;
                    o.target = static_cast<int32_t>(cg->target);
                    o.control = static_cast<int32_t>(cg->control);
                    put_gate(cg->gate);
                } else if (const auto* fn = std::get_if<FunctionOp>(&op)) {
                    o.kind = QSB_OP_FUNCTION;
                    o.first = static_cast<int32_t>(fn->first_qubit);
                    o.count = static_cast<int32_t>(fn->qubit_count);
                    for (std::size_t i = 0; i < names.size(); ++i)
                        if (names[i] == fn->name) o.function = static_cast<int32_t>(i);
                } else {
                    const auto& in = std::get<Instruction>(op);
                    o.kind = QSB_OP_INSTRUCTION;
                    o.target = static_cast<int32_t>(in.target);
                    o.instruction = in.kind == InstructionKind::Reset ? QSB_INSTR_RESET : QSB_INSTR_MEASURE;
                }
            }
            step_offsets[++s] = k;
        }
    });
}

int64_t refsh_function_dim(void* p, int idx) {
    const Program& prog = *static_cast<Program*>(p);
    const auto names = function_names(prog.circuit);
    return static_cast<int64_t>(prog.registry.lookup(names.at(idx)).rows());
}
int refsh_function_matrix(void* p, int idx, double* re, double* im) {
    return guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        copy_out(prog.registry.lookup(function_names(prog.circuit).at(idx)), re, im);
    });
}

// step_unitary (unitary_backend.cpp:141-154)
int refsh_step_unitary(void* p, int step, double* re, double* im) {
    return guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        copy_out(step_unitary(prog.circuit.steps().at(step), prog.circuit.qubit_count(), prog.registry), re, im);
    });
}

// step_operand_list (unitary_backend.cpp:129-139): count, then each operand's dim + planes.
int refsh_step_operand_count(void* p, int step, int* count) {
    return guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        *count = static_cast<int>(
            step_operand_list(prog.circuit.steps().at(step), prog.circuit.qubit_count(), prog.registry).size());
    });
}

// test::circuit_unitary (test_util.hpp:135-142)
int refsh_circuit_unitary(void* p, int parallel, double* re, double* im) {
    return guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        copy_out(test::circuit_unitary(prog.circuit, prog.registry,
                                       parallel ? ExecMode::Parallel : ExecMode::Serial),
                 re, im);
    });
}

// make_simulator(backend, {guard})->simulate_full_state (simulator.cpp:59-68)
int refsh_simulate(void* p, const char* backend, int guard, double* re, double* im) {
    return guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        SimulatorOptions o;
        if (guard > 0) o.qubit_guard = static_cast<std::size_t>(guard);
        const StateVector s = make_simulator(backend, o)->simulate_full_state(prog.circuit, prog.registry);
        std::memcpy(re, s.amplitudes.re.data(), sizeof(double) * s.dimension());
        std::memcpy(im, s.amplitudes.im.data(), sizeof(double) * s.dimension());
    });
}

// Simulator::simulate_and_collapse (simulator.cpp:26-30)
int refsh_simulate_and_collapse(void* p, const char* backend, uint64_t seed, uint64_t* index) {
    return guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        *index = make_simulator(backend)->simulate_and_collapse(prog.circuit, prog.registry, seed).basis_index;
    });
}

// collapse / probabilities / norm_squared on a given state (state.cpp:49-98)
int refsh_collapse(int qubits, const double* re, const double* im, uint64_t seed, uint64_t* index) {
    return guarded([&] {
        StateVector s = zero_state(static_cast<std::size_t>(qubits));
        std::memcpy(s.amplitudes.re.data(), re, sizeof(double) * s.dimension());
        std::memcpy(s.amplitudes.im.data(), im, sizeof(double) * s.dimension());
        *index = collapse(s, seed).basis_index;
    });
}
int refsh_probabilities(int qubits, const double* re, const double* im, double* p, double* norm) {
    return guarded([&] {
        StateVector s = zero_state(static_cast<std::size_t>(qubits));
        std::memcpy(s.amplitudes.re.data(), re, sizeof(double) * s.dimension());
        std::memcpy(s.amplitudes.im.data(), im, sizeof(double) * s.dimension());
        const auto v = probabilities(s);
        std::memcpy(p, v.data(), sizeof(double) * v.size());
        *norm = norm_squared(s);
    });
}

uint64_t refsh_splitmix64_unit_bits(uint64_t seed, int draws) {
    SplitMix64 r(seed);
    double u = 0;
    for (int i = 0; i < draws; ++i) u = r.next_unit();
    uint64_t bits;
    std::memcpy(&bits, &u, 8);
    return bits;
}

uint64_t refsh_memory_estimate(int n, int kind) {
    uint64_t v = 0;
    guarded([&] { v = memory_estimate(n, kind == 0 ? BackendKind::Unitary : BackendKind::Fsv); });
    return v;
}
uint64_t refsh_engine_memory_estimate(int n, int kind) {
    uint64_t v = 0;
    guarded([&] { v = engine_memory_estimate(n, kind == 0 ? BackendKind::Unitary : BackendKind::Fsv); });
    return v;
}
int refsh_format_bytes(uint64_t bytes, char* buf, int len) {
    const std::string s = format_bytes(bytes);
    std::snprintf(buf, len, "%s", s.c_str());
    return 0;
}

void refsh_set_worker_count(int n) { set_worker_count(static_cast<std::size_t>(n)); }
int refsh_worker_count() { return static_cast<int>(worker_count()); }

// ---- CPU-baseline timing of the reference path (bench.py --impl reference) ----

// Wall time (s) of step_unitary for one step.
double refsh_time_step_unitary(void* p, int step) {
    double secs = -1;
    guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        const auto t0 = std::chrono::steady_clock::now();
        const ComplexMatrix a = step_unitary(prog.circuit.steps().at(step), prog.circuit.qubit_count(), prog.registry);
        const auto t1 = std::chrono::steady_clock::now();
        secs = std::chrono::duration<double>(t1 - t0).count();
        if (a.rows() == 0) secs = -1;
    });
    return secs;
}

// Wall time (s) of the reference's matmul(a, b, mode) with a = rows x N and
// b = N x N (the accumulate GEMM of unitary_backend.cpp:211 restricted to
// `rows` output rows; linalg.cpp:72-87 accepts rectangular shapes).
double refsh_time_matmul(int64_t rows, int64_t n, int parallel) {
    double secs = -1;
    guarded([&] {
        ComplexMatrix a(static_cast<std::size_t>(rows), static_cast<std::size_t>(n));
        ComplexMatrix b = ComplexMatrix::identity(static_cast<std::size_t>(n));
        for (std::size_t i = 0; i < a.rows(); ++i)
            for (std::size_t j = 0; j < a.cols(); ++j) {
                a.re(i, j) = 1.0 / (1.0 + static_cast<double>(i + j));
                a.im(i, j) = 0.5 / (1.0 + static_cast<double>(i + 2 * j));
            }
        const auto t0 = std::chrono::steady_clock::now();
        const ComplexMatrix c = matmul(a, b, parallel ? ExecMode::Parallel : ExecMode::Serial);
        const auto t1 = std::chrono::steady_clock::now();
        secs = std::chrono::duration<double>(t1 - t0).count();
        if (c.rows() == 0) secs = -1;
    });
    return secs;
}

// Wall time (s) of one full UnitarySimulator::simulate_full_state.
double refsh_time_simulate(void* p, const char* backend, int guard) {
    double secs = -1;
    guarded([&] {
        const Program& prog = *static_cast<Program*>(p);
        SimulatorOptions o;
        if (guard > 0) o.qubit_guard = static_cast<std::size_t>(guard);
        auto sim = make_simulator(backend, o);
        const auto t0 = std::chrono::steady_clock::now();
        const StateVector s = sim->simulate_full_state(prog.circuit, prog.registry);
        const auto t1 = std::chrono::steady_clock::now();
        secs = std::chrono::duration<double>(t1 - t0).count();
        if (s.dimension() == 0) secs = -1;
    });
    return secs;
}

} // extern "C"
