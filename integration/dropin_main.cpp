// dropin_main.cpp — drop-in proof: the UNMODIFIED reference library (oracle/_ref)
// with "unitary-b200" registered through its own plugin API, exercised by the
// reference's own harness and acceptance-style checks. Prints one PASS/FAIL line
// per check and exits non-zero on any failure. Test infrastructure (built by
// oracle/Makefile target `dropin`, run by tests/test_dropin_gpu.py).
#include <cmath>
#include <cstdio>
#include <functional>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "b200_unitary_simulator.hpp"
#include "qsim/bench.hpp"
#include "qsim/circuit_library.hpp"
#include "qsim/errors.hpp"
#include "qsim/fsv_backend.hpp"
#include "qsim/unitary_backend.hpp"
#include "support/test_util.hpp"

using namespace qsim;

namespace {

int failures = 0;

void report(const char* name, bool ok, const std::string& detail) {
    std::printf("%s  %s: %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
    if (!ok) ++failures;
}

std::string fmt(const char* f, double a, double b = 0) {
    char buf[256];
    std::snprintf(buf, sizeof buf, f, a, b);
    return buf;
}

// ComplexVector has no operator==; compare planes with vector == (so -0.0 == +0.0,
// as ComplexMatrix::operator==, linalg.hpp:63).
bool same(const ComplexVector& a, const ComplexVector& b) { return a.re == b.re && a.im == b.im; }

}  // namespace

int main(int argc, char** argv) {
    const bool with_bench = argc > 1 && std::string(argv[1]) == "--bench";
    register_b200_backend();
    const auto names = backend_names();
    bool listed = false;
    for (const auto& n : names) listed = listed || n == "unitary-b200";
    report("registry lists unitary-b200", listed, std::to_string(names.size()) + " backends");

    auto gpu = make_simulator("unitary-b200");

    {  // acceptance_main.cpp:60-76 — Bell ground truth at 1e-12
        const double s = std::sqrt(0.5);
        const auto out = gpu->simulate_full_state(bell(), {});
        double worst = std::max(std::abs(out.amplitudes.re[0] - s), std::abs(out.amplitudes.re[3] - s));
        worst = std::max(worst, std::hypot(out.amplitudes.re[1], out.amplitudes.im[1]));
        worst = std::max(worst, std::hypot(out.amplitudes.re[2], out.amplitudes.im[2]));
        report("Bell ground truth (1e-12)", worst <= 1e-12, fmt("worst %.3e", worst));
    }
    {  // acceptance_main.cpp:80-110 — 200 random circuits vs fsv at 1e-9, seed 20260810
        std::mt19937_64 rng(20260810);
        std::uniform_int_distribution<std::size_t> qubit_pick(2, 8);
        std::uniform_int_distribution<std::size_t> op_pick(1, 30);
        const FsvSimulator fsv;
        double worst = 0, worst_norm = 0;
        for (int i = 0; i < 200; ++i) {
            const std::size_t n = qubit_pick(rng);
            const Circuit c = test::random_circuit(rng, n, op_pick(rng));
            const auto a = gpu->simulate_full_state(c, {});
            const auto b = fsv.simulate_full_state(c, {});
            worst = std::max(worst, max_entry_diff(a.amplitudes, b.amplitudes));
            worst_norm = std::max(worst_norm, std::abs(norm_squared(a) - 1.0));
        }
        report("200 random circuits vs fsv (1e-9)", worst <= 1e-9 && worst_norm <= 1e-9,
               fmt("worst %.3e, norm %.3e", worst, worst_norm));
    }
    {  // fsv-b200: the reference's own FsvSimulator, bit for bit (same seed stream)
        std::mt19937_64 rng(20260810);
        std::uniform_int_distribution<std::size_t> qubit_pick(2, 14);
        std::uniform_int_distribution<std::size_t> op_pick(1, 60);
        const FsvSimulator fsv(24);
        auto gfsv = make_simulator("fsv-b200");
        bool same = true;
        for (int i = 0; i < 200; ++i) {
            const Circuit c = test::random_circuit(rng, qubit_pick(rng), op_pick(rng));
            same = same && ::same(gfsv->simulate_full_state(c, {}).amplitudes, fsv.simulate_full_state(c, {}).amplitudes);
        }
        for (std::size_t n : {13, 16})
            same = same && ::same(gfsv->simulate_full_state(qft(n), {}).amplitudes,
                                  fsv.simulate_full_state(qft(n), {}).amplitudes);
        const auto dj = make_named_circuit("deutsch-jozsa", 9);  // registration is_unitary is O(8^n) on the host
        same = same && ::same(gfsv->simulate_full_state(dj.circuit, dj.registry).amplitudes,
                              fsv.simulate_full_state(dj.circuit, dj.registry).amplitudes);
        report("fsv-b200 == reference FsvSimulator (200 random circuits, qft13/16, dj9; ==)", same, "");
    }
    {  // unitary-structured-b200: U within 1e-10 of the reference's U; U[:, c] == fsv(e_c)
        auto gst = make_simulator("unitary-structured-b200");
        const auto* st = dynamic_cast<const B200StructuredUnitarySimulator*>(gst.get());
        std::mt19937_64 rng(31415);
        std::uniform_int_distribution<std::size_t> qubit_pick(2, 6);
        std::uniform_int_distribution<std::size_t> op_pick(1, 25);
        double worst = 0;
        for (int i = 0; i < 40; ++i) {
            const Circuit c = test::random_circuit(rng, qubit_pick(rng), op_pick(rng));
            const ComplexMatrix a = st->circuit_unitary(c, {});
            const ComplexMatrix b = test::circuit_unitary(c, {});
            worst = std::max(worst, max_entry_diff(a, b));
        }
        const auto q8 = st->simulate_full_state(qft(8), {});
        const bool col0 = same(q8.amplitudes, FsvSimulator().simulate_full_state(qft(8), {}).amplitudes);
        report("unitary-structured-b200 U vs reference U (40 random, 1e-10); psi == fsv", worst <= 1e-10 && col0,
               fmt("worst %.3e", worst));
    }
    {  // registry validation on the GPU: same verdicts as the reference's is_unitary
        std::mt19937_64 rng(555);
        std::normal_distribution<double> nd;
        bool ok = true;
        for (std::size_t n : {1, 3, 6, 8}) {
            const std::size_t d = std::size_t{1} << n;
            ComplexMatrix perm(d, d), noisy(d, d);
            for (std::size_t i = 0; i < d; ++i) perm.re((i * 5 + 3) % d, i) = 1.0;  // a permutation
            for (std::size_t i = 0; i < d; ++i)
                for (std::size_t j = 0; j < d; ++j) {
                    noisy.re(i, j) = perm.re(i, j) + 1e-7 * nd(rng);
                    noisy.im(i, j) = 1e-7 * nd(rng);
                }
            ok = ok && b200_is_unitary(perm, kRegistryUnitaryTol) == is_unitary(perm, kRegistryUnitaryTol) &&
                 b200_is_unitary(noisy, kRegistryUnitaryTol) == is_unitary(noisy, kRegistryUnitaryTol) &&
                 b200_is_unitary(perm, kRegistryUnitaryTol) && !b200_is_unitary(noisy, kRegistryUnitaryTol);
        }
        report("b200_is_unitary verdicts == reference is_unitary (dims 2..256)", ok, "");
    }
    {  // acceptance_main.cpp:173-193 — QFT == DFT (n <= 6) and uniform QFT|0> (n <= 12)
        const auto* b200 = dynamic_cast<const B200UnitarySimulator*>(gpu.get());
        double worst = 0;
        for (std::size_t n = 1; n <= 6; ++n)
            worst = std::max(worst, max_entry_diff(b200->circuit_unitary(qft(n), {}), test::dft_matrix(n)));
        double worst_u = 0;
        for (std::size_t n = 1; n <= 12; ++n) {
            const auto out = gpu->simulate_full_state(qft(n), {});
            const double expect = 1.0 / std::sqrt(static_cast<double>(out.dimension()));
            for (std::size_t i = 0; i < out.dimension(); ++i)
                worst_u = std::max(worst_u, std::hypot(out.amplitudes.re[i] - expect, out.amplitudes.im[i]));
        }
        report("QFT == DFT (n<=6, 1e-9); QFT|0> uniform (n<=12, 1e-12)", worst <= 1e-9 && worst_u <= 1e-12,
               fmt("DFT %.3e, uniform %.3e", worst, worst_u));
    }
    {  // acceptance_main.cpp:197-242 — Deutsch-Jozsa classification
        bool ok = true;
        for (const bool value : {false, true}) {
            const auto p = deutsch_jozsa(2, [value](std::uint64_t) { return value; });
            ok = ok && std::abs(all_zero_input_probability(gpu->simulate_full_state(p.circuit, p.registry), 2) - 1.0) < 1e-9;
        }
        std::mt19937_64 rng(424242);
        std::uniform_int_distribution<std::uint64_t> mask_pick(1, 15);
        for (int i = 0; i < 20; ++i) {
            char spec[64];
            std::snprintf(spec, sizeof spec, "balanced-mask:%llx", static_cast<unsigned long long>(mask_pick(rng)));
            const auto p = deutsch_jozsa(4, parse_oracle_spec(spec, 4).fn);
            ok = ok && all_zero_input_probability(gpu->simulate_full_state(p.circuit, p.registry), 4) < 1e-9;
        }
        report("Deutsch-Jozsa constant/balanced classification", ok, "2 constant + 20 balanced masks");
    }
    {  // acceptance_main.cpp:246-266 analogue — guard refusal carries the byte estimate
        SimulatorOptions o;
        o.qubit_guard = 3;
        auto small = make_simulator("unitary-b200", o);
        bool ok = false;
        std::string what;
        try {
            small->simulate_full_state(Circuit(4), {});
        } catch (const ResourceError& e) {
            what = e.what();
            ok = what.find(std::to_string(memory_estimate(4, BackendKind::Unitary))) != std::string::npos;
        }
        // the reference backend's own refusal, word for word but for the backend name
        std::string ref_what;
        try {
            make_simulator("unitary", o)->simulate_full_state(Circuit(4), {});
        } catch (const ResourceError& e) {
            ref_what = e.what();
        }
        const std::string from = "unitary backend", to = "unitary-b200 backend";
        if (ref_what.rfind(from, 0) == 0) ref_what.replace(0, from.size(), to);
        ok = ok && !ref_what.empty() && what == ref_what;
        report("guard -> ResourceError with the reference's message", ok, what + " | reference: " + ref_what);
        bool reset_ok = false;
        try {
            Circuit bad(2);
            bad.reset(0).h(0);
            gpu->simulate_full_state(bad, {});
        } catch (const ValidationError&) {
            reset_ok = true;
        }
        report("mid-circuit reset -> ValidationError", reset_ok, "");
    }
    {  // acceptance_main.cpp:331-350 — collapse statistics over 10000 seeds
        std::size_t zeros = 0;
        bool support = true;
        for (std::uint64_t seed = 0; seed < 10000; ++seed) {
            const auto o = gpu->simulate_and_collapse(bell(), {}, seed);
            support = support && (o.basis_index == 0 || o.basis_index == 3);
            zeros += o.basis_index == 0;
        }
        const double freq = static_cast<double>(zeros) / 10000.0;
        report("collapse statistics (Bell, 10000 seeds)", support && freq >= 0.47 && freq <= 0.53,
               fmt("|00> frequency %.4f", freq));
        bool same = true;
        const UnitarySimulator cpu;
        for (std::uint64_t seed = 0; seed < 200; ++seed)
            same = same && cpu.simulate_and_collapse(qft(5), {}, seed).basis_index ==
                               gpu->simulate_and_collapse(qft(5), {}, seed).basis_index;
        report("collapse outcomes identical to the reference (qft5, 200 seeds)", same, "");
    }
    if (with_bench) {
        // bench.cpp:42-129: the reference harness cross-checks every backend at
        // 1e-9 before timing (throws on disagreement) and reports speedup vs the
        // first-listed backend.
        BenchConfig cfg;
        cfg.circuits = {"qft", "entangle", "deutsch-jozsa"};
        cfg.qubits_from = 4;
        cfg.qubits_to = 9;
        cfg.backends = {"unitary-parallel", "unitary-b200", "unitary-structured-b200", "fsv-b200"};
        cfg.warmup_iters = 3;
        cfg.sample_iters = 5;
        bool ok = true;
        std::string csv;
        try {
            csv = report(run_bench(cfg, &std::cerr), ReportFormat::Csv);
        } catch (const std::exception& e) {
            ok = false;
            csv = e.what();
        }
        std::printf("%s", csv.c_str());
        ::report("reference run_bench cross-check (1e-9) + timing", ok, "see CSV above");
    }
    std::printf("%d failure(s)\n", failures);
    return failures == 0 ? 0 : 1;
}
