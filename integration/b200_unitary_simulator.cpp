// b200_unitary_simulator.cpp — flattens a qsim::Circuit into the C ABI and maps
// qsb_status back onto the qsim::Error hierarchy (errors.hpp:23-56).
#include "b200_unitary_simulator.hpp"

#include <cstdlib>
#include <map>
#include <memory>
#include <sstream>
#include <variant>
#include <vector>

#include "qsim/errors.hpp"
#include "qsim/gates.hpp"

namespace qsim {

namespace {

[[noreturn]] void throw_status(qsb_status st) {
    char buf[1024];
    qsb_last_error(buf, sizeof buf);
    const std::string msg(buf);
    switch (st) {
    case QSB_ERR_RESOURCE: throw ResourceError(msg);
    case QSB_ERR_VALIDATION: throw ValidationError(msg);
    case QSB_ERR_SHAPE: throw ShapeError(msg);
    case QSB_ERR_ARGUMENT: throw ArgumentError(msg);
    case QSB_ERR_LOOKUP: throw LookupError(msg);
    default: throw Error("unitary-b200: " + msg);
    }
}

void check(qsb_status st) {
    if (st != QSB_OK) throw_status(st);
}

// Owns the flattened arrays for the duration of one call (Circuit and
// GateRegistry are borrowed const& for the call only, as in the reference).
struct Flat {
    std::vector<int32_t> offsets{0};
    std::vector<qsb_op> ops;
    std::vector<qsb_function> functions;
    std::vector<std::vector<double>> planes;  // keeps registry copies alive only if needed
    qsb_circuit c{};
};

void put_gate(qsb_op& o, const GateType& g) {
    o.gate = static_cast<int32_t>(g.tag);
    o.phi = g.phi;
    const ComplexMatrix m = gate_matrix(g);  // the reference's gate library (gates.cpp:40-77)
    for (int e = 0; e < 4; ++e) {
        o.u_re[e] = m.re(e / 2, e % 2);
        o.u_im[e] = m.im(e / 2, e % 2);
    }
}

std::unique_ptr<Flat> flatten(const Circuit& circuit, const GateRegistry& registry) {
    auto f = std::make_unique<Flat>();
    std::map<std::string, int32_t> fn_index;
    for (const Step& step : circuit.steps()) {
        for (const Operation& op : step.operations) {
            qsb_op o{};
            if (const auto* g = std::get_if<Gate>(&op)) {
                o.kind = QSB_OP_GATE;
                o.target = static_cast<int32_t>(g->target);
                put_gate(o, g->gate);
            } else if (const auto* cg = std::get_if<ControlGate>(&op)) {
                o.kind = QSB_OP_CONTROL;
                o.target = static_cast<int32_t>(cg->target);
                o.control = static_cast<int32_t>(cg->control);
                put_gate(o, cg->gate);
            } else if (const auto* fn = std::get_if<FunctionOp>(&op)) {
                o.kind = QSB_OP_FUNCTION;
                o.first = static_cast<int32_t>(fn->first_qubit);
                o.count = static_cast<int32_t>(fn->qubit_count);
                auto it = fn_index.find(fn->name);
                if (it == fn_index.end()) {
                    const ComplexMatrix& m = registry.lookup(fn->name);  // LookupError as the reference
                    it = fn_index.emplace(fn->name, static_cast<int32_t>(f->functions.size())).first;
                    f->functions.push_back({static_cast<int64_t>(m.rows()), m.re_data(), m.im_data()});
                }
                o.function = it->second;
            } else {
                const auto& in = std::get<Instruction>(op);
                o.kind = QSB_OP_INSTRUCTION;
                o.target = static_cast<int32_t>(in.target);
                o.instruction = in.kind == InstructionKind::Reset ? QSB_INSTR_RESET : QSB_INSTR_MEASURE;
            }
            f->ops.push_back(o);
        }
        f->offsets.push_back(static_cast<int32_t>(f->ops.size()));
    }
    f->c.n_qubits = static_cast<int32_t>(circuit.qubit_count());
    f->c.n_steps = static_cast<int32_t>(circuit.steps().size());
    f->c.step_offsets = f->offsets.data();
    f->c.ops = f->ops.data();
    f->c.n_functions = static_cast<int32_t>(f->functions.size());
    f->c.functions = f->functions.data();
    return f;
}

}  // namespace

B200UnitarySimulator::B200UnitarySimulator(std::size_t qubit_guard, std::vector<int> devices) {
    std::vector<int32_t> ids(devices.begin(), devices.end());
    qsb_options o{ids.empty() ? 0 : ids[0], static_cast<int32_t>(qubit_guard), QSB_GEMM_AUTO, 0,
                  static_cast<int32_t>(ids.size()), 0, ids.data()};
    check(qsb_create(&o, &handle_));
    int32_t g = 0;
    check(qsb_qubit_guard(handle_, &g));
    guard_ = static_cast<std::size_t>(g);
}

B200UnitarySimulator::~B200UnitarySimulator() { qsb_destroy(handle_); }

StateVector B200UnitarySimulator::simulate_full_state(const Circuit& circuit, const GateRegistry& registry) const {
    const auto f = flatten(circuit, registry);
    StateVector s{circuit.qubit_count(), ComplexVector(std::size_t{1} << circuit.qubit_count())};
    check(qsb_simulate_full_state(handle_, &f->c, s.amplitudes.re.data(), s.amplitudes.im.data()));
    return s;
}

CollapsedState B200UnitarySimulator::simulate_and_collapse(const Circuit& circuit, const GateRegistry& registry,
                                                           std::uint64_t seed) const {
    const auto f = flatten(circuit, registry);
    uint64_t index = 0;
    check(qsb_simulate_and_collapse(handle_, &f->c, seed, &index));
    return {circuit.qubit_count(), index};
}

ComplexMatrix B200UnitarySimulator::circuit_unitary(const Circuit& circuit, const GateRegistry& registry) const {
    const auto f = flatten(circuit, registry);
    const std::size_t N = std::size_t{1} << circuit.qubit_count();
    ComplexMatrix u(N, N);
    check(qsb_build_unitary(handle_, &f->c, u.re_data(), u.im_data()));
    return u;
}

namespace {
std::vector<int> devices_from_env() {
    const char* env = std::getenv("QSB_DEVICES");
    std::vector<int> ids;
    if (!env || !*env) return {0};
    if (std::string(env) == "all") {
        // one row block per visible device, probed through the library
        for (int d = 0; d < 64; ++d) {
            qsb_options o{d, 0, QSB_GEMM_AUTO, 0, 0, 0, nullptr};
            qsb_handle* h = nullptr;
            if (qsb_create(&o, &h) != QSB_OK) break;
            qsb_destroy(h);
            ids.push_back(d);
        }
        return ids.empty() ? std::vector<int>{0} : ids;
    }
    std::stringstream ss(env);
    std::string tok;
    while (std::getline(ss, tok, ',')) ids.push_back(std::stoi(tok));
    return ids.empty() ? std::vector<int>{0} : ids;
}
}  // namespace

B200FsvSimulator::B200FsvSimulator(std::size_t qubit_guard, int device) {
    qsb_options o{device, static_cast<int32_t>(qubit_guard), QSB_GEMM_AUTO, 0, 0, 0, nullptr};
    check(qsb_create(&o, &handle_));
    int32_t g = 0;
    check(qsb_fsv_qubit_guard(handle_, &g));
    guard_ = static_cast<std::size_t>(g);
}

B200FsvSimulator::~B200FsvSimulator() { qsb_destroy(handle_); }

StateVector B200FsvSimulator::simulate_full_state(const Circuit& circuit, const GateRegistry& registry) const {
    const auto f = flatten(circuit, registry);
    StateVector s{circuit.qubit_count(), ComplexVector(std::size_t{1} << circuit.qubit_count())};
    check(qsb_fsv_simulate_full_state(handle_, &f->c, s.amplitudes.re.data(), s.amplitudes.im.data()));
    return s;
}

B200StructuredUnitarySimulator::B200StructuredUnitarySimulator(std::size_t qubit_guard, std::vector<int> devices) {
    std::vector<int32_t> ids(devices.begin(), devices.end());
    qsb_options o{ids.empty() ? 0 : ids[0], static_cast<int32_t>(qubit_guard), QSB_GEMM_AUTO, 0,
                  static_cast<int32_t>(ids.size()), 0, ids.data()};
    check(qsb_create(&o, &handle_));
    int32_t g = 0;
    check(qsb_structured_qubit_guard(handle_, &g));
    guard_ = static_cast<std::size_t>(g);
}

B200StructuredUnitarySimulator::~B200StructuredUnitarySimulator() { qsb_destroy(handle_); }

StateVector B200StructuredUnitarySimulator::simulate_full_state(const Circuit& circuit,
                                                                const GateRegistry& registry) const {
    const auto f = flatten(circuit, registry);
    StateVector s{circuit.qubit_count(), ComplexVector(std::size_t{1} << circuit.qubit_count())};
    check(qsb_structured_simulate_full_state(handle_, &f->c, s.amplitudes.re.data(), s.amplitudes.im.data()));
    return s;
}

ComplexMatrix B200StructuredUnitarySimulator::circuit_unitary(const Circuit& circuit,
                                                              const GateRegistry& registry) const {
    const auto f = flatten(circuit, registry);
    const std::size_t N = std::size_t{1} << circuit.qubit_count();
    ComplexMatrix u(N, N);
    check(qsb_structured_build_unitary(handle_, &f->c, u.re_data(), u.im_data()));
    return u;
}

bool b200_is_unitary(const ComplexMatrix& m, double tol) {
    if (m.rows() != m.cols())  // the reference's ShapeError (linalg.cpp:132-135)
        throw ShapeError("is_unitary: matrix is " + std::to_string(m.rows()) + "x" + std::to_string(m.cols()));
    static qsb_handle* handle = [] {
        qsb_options o{0, 0, QSB_GEMM_AUTO, 0, 0, 0, nullptr};
        qsb_handle* h = nullptr;
        check(qsb_create(&o, &h));
        return h;
    }();
    int32_t ok = 0;
    check(qsb_is_unitary(handle, m.re_data(), m.im_data(), static_cast<int64_t>(m.rows()), tol, &ok, nullptr));
    return ok != 0;
}

void register_b200_backend() {
    register_backend("unitary-b200", [](const SimulatorOptions& o) -> std::unique_ptr<Simulator> {
        return std::make_unique<B200UnitarySimulator>(o.qubit_guard.value_or(0), devices_from_env());
    });
    register_backend("fsv-b200", [](const SimulatorOptions& o) -> std::unique_ptr<Simulator> {
        return std::make_unique<B200FsvSimulator>(o.qubit_guard.value_or(0), devices_from_env().front());
    });
    register_backend("unitary-structured-b200", [](const SimulatorOptions& o) -> std::unique_ptr<Simulator> {
        return std::make_unique<B200StructuredUnitarySimulator>(o.qubit_guard.value_or(0), devices_from_env());
    });
}

}  // namespace qsim
