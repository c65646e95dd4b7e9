// b200_unitary_simulator.hpp — the reference-side binding a qsim maintainer adds
// to make the B200 path a drop-in backend.
//
// Implements the reference's plugin interface qsim::Simulator
// (proj/core/include/qsim/simulator.hpp:32-51) on top of the C ABI in
// include/qsb.h, and registers it under "unitary-b200" with
// qsim::register_backend (simulator.cpp:70-73) so run_bench, the CLI and any
// caller of make_simulator can select it. Circuit, GateRegistry, gate_matrix,
// StateVector and the error types are the reference's own, unchanged.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "qsb.h"
#include "qsim/simulator.hpp"

namespace qsim {

class B200UnitarySimulator final : public Simulator {
public:
    /// qubit_guard 0 = derived from HBM capacity (n <= 16 on one B200, 17 on 4-8).
    /// devices: more than one shards U by row blocks over them (no communication
    /// during the product chain; each device writes its psi rows to the result).
    explicit B200UnitarySimulator(std::size_t qubit_guard = 0, std::vector<int> devices = {0});
    ~B200UnitarySimulator() override;
    B200UnitarySimulator(const B200UnitarySimulator&) = delete;
    B200UnitarySimulator& operator=(const B200UnitarySimulator&) = delete;

    std::string name() const override { return "unitary-b200"; }
    std::size_t qubit_guard() const override { return guard_; }

    /// Algorithm 1 on the GPU: same contract as UnitarySimulator
    /// (unitary_backend.cpp:194-215), results within 1e-10 relative.
    StateVector simulate_full_state(const Circuit& circuit, const GateRegistry& registry) const override;

    /// Inverse-CDF collapse over the GPU-computed probabilities (state.cpp:81-98).
    CollapsedState simulate_and_collapse(const Circuit& circuit, const GateRegistry& registry,
                                         std::uint64_t seed) const override;

    /// The accumulated unitary (test::circuit_unitary, test_util.hpp:135-142).
    ComplexMatrix circuit_unitary(const Circuit& circuit, const GateRegistry& registry) const;

private:
    qsb_handle* handle_ = nullptr;
    std::size_t guard_ = 0;
};

/// FsvSimulator on the GPU (fsv_backend.cpp:135-158): every operation applied to
/// the state in circuit order; bit-exact with the reference's fsv backend.
class B200FsvSimulator final : public Simulator {
public:
    explicit B200FsvSimulator(std::size_t qubit_guard = 0, int device = 0);
    ~B200FsvSimulator() override;
    B200FsvSimulator(const B200FsvSimulator&) = delete;
    B200FsvSimulator& operator=(const B200FsvSimulator&) = delete;

    std::string name() const override { return "fsv-b200"; }
    std::size_t qubit_guard() const override { return guard_; }
    StateVector simulate_full_state(const Circuit& circuit, const GateRegistry& registry) const override;

private:
    qsb_handle* handle_ = nullptr;
    std::size_t guard_ = 0;
};

/// Unitary simulation without dense GEMMs: U[:, c] = fsv(e_c) for every column,
/// all columns evolved at once on the GPU (columns sharded over `devices`).
/// Same U as UnitarySimulator within rounding; psi = U e_0.
class B200StructuredUnitarySimulator final : public Simulator {
public:
    explicit B200StructuredUnitarySimulator(std::size_t qubit_guard = 0, std::vector<int> devices = {0});
    ~B200StructuredUnitarySimulator() override;
    B200StructuredUnitarySimulator(const B200StructuredUnitarySimulator&) = delete;
    B200StructuredUnitarySimulator& operator=(const B200StructuredUnitarySimulator&) = delete;

    std::string name() const override { return "unitary-structured-b200"; }
    std::size_t qubit_guard() const override { return guard_; }
    StateVector simulate_full_state(const Circuit& circuit, const GateRegistry& registry) const override;
    ComplexMatrix circuit_unitary(const Circuit& circuit, const GateRegistry& registry) const;

private:
    qsb_handle* handle_ = nullptr;
    std::size_t guard_ = 0;
};

/// is_unitary (linalg.cpp:131-155) on the GPU (qsb_is_unitary: A^H A on the
/// FP64 tensor cores), through a process-wide handle on device 0. The
/// replacement for the check in GateRegistry::register_function (gates.cpp:121).
bool b200_is_unitary(const ComplexMatrix& m, double tol);

/// register_backend("unitary-b200" | "fsv-b200" | "unitary-structured-b200", ...)
/// honouring SimulatorOptions::qubit_guard; the device list comes from
/// QSB_DEVICES ("0,1,2,3", or "all"; default "0").
void register_b200_backend();

}  // namespace qsim
