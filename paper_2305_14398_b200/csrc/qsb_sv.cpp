// qsb_sv.cpp — host runtime of the state-vector engine behind the C ABI
// (include/qsb.h, "state-vector engine"): the fsv backend
// (FsvSimulator, fsv_backend.cpp:135-158) and the structured unitary
// (U[:, c] = fsv(e_c) for all columns at once).
//
// Responsibilities: validate exactly where the reference's fsv backend does
// (guard, reset placement, per-operation ranges and function dimensions:
// fsv_backend.cpp:25-31, 74-79, 86-97, 137-142), translate the circuit into
// flat-bit operations in application order (steps in order, operations in
// insertion order, instructions skipped: fsv_backend.cpp:143-156), group them
// into shared-memory batches, and run the passes on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "../../include/qsb.h"
#include "qsb_host.hpp"
#include "qsb_jit.hpp"
#include "qsb_sv.hpp"

using namespace qsbh;

struct qsb_sv_plan {
    qsb_handle* h = nullptr;
    DeviceCtx* dc = nullptr;
    int mode = QSB_SV_STATE;
    int n = 0, w = 0, m = 0;
    int64_t col_begin = 0, col_count = 1;
    struct FnPass {
        int k, s;
        qsb::SvTable tab;
    };
    enum PassKind { kReg = 0, kSlab = 1, kFn = 2 };
    struct Pass {
        int kind;
        std::shared_ptr<qsb::SvRegBatch> reg;  // kReg: gates / controlled gates, elements in registers
        void* jit = nullptr;                   // kReg: the batch compiled straight-line (qsb_jit.hpp), or null
        std::vector<double> coef;              // kReg + jit: the coefficients, in the kernel's parameter order
        int jit_smem = 0;                      // kReg + jit: dynamic shared memory (prefetch slots)
        qsb::SvBatch batch;   // kSlab: small apply_function blocks in shared memory
        FnPass f;             // kFn: apply_function blocks larger than a slab
    };
    std::vector<qsb::SvLocalOp> ops;  // local ops of every batch, contiguous per batch
    std::vector<Pass> passes;
    Buffers b;
    bool borrowed = false;
    int final_buf = 0;
    qsb_sv_plan_info info{};
};

namespace {

// One operation in flat-bit form.
struct FlatOp {
    int kind;        // qsb::SvOpKind
    int cls;         // qsb::SvPairClass
    int tbit;        // pair: target flat bit; function: flat bit of the block's lsb
    int cbit;        // pair: control flat bit or -1
    int k;           // function: qubit count
    int fn;          // function index
    double u_re[4], u_im[4];
};

int classify(const double* ur, const double* ui) {
    auto zero = [&](int e) { return ur[e] == 0.0 && ui[e] == 0.0; };
    auto one = [&](int e) { return ur[e] == 1.0 && ui[e] == 0.0; };
    if (zero(1) && zero(2)) return one(0) ? qsb::kPairDiag1 : qsb::kPairDiag;
    if (zero(0) && zero(3)) return (one(1) && one(2)) ? qsb::kPairSwap : qsb::kPairAnti;
    if (ui[0] == 0.0 && ui[1] == 0.0 && ui[2] == 0.0 && ui[3] == 0.0) return qsb::kPairReal;
    return qsb::kPairGeneral;
}

int popcount64(uint64_t x) { return __builtin_popcountll(x); }

int slab_bits_default() {
    const char* e = std::getenv("QSB_SV_SLAB_BITS");  // tuning / tests
    if (e && *e) {
        const int v = std::atoi(e);
        if (v >= 6 && v <= qsb::kSvMaxSlabBits) return v;
    }
    return qsb::kSvMaxSlabBits;
}

void sv_check_guard(const qsb_circuit* c, int guard, const char* backend) {
    if (c->n_qubits > guard) {
        raise(QSB_ERR_RESOURCE, "%s backend refuses %d qubits (guard %d)", backend, c->n_qubits, guard);
    }
    check_reset_placement(c);
}

std::vector<FlatOp> flatten_ops(const qsb_circuit* c, int w) {
    const int n = c->n_qubits;
    std::vector<FlatOp> out;
    for (int s = 0; s < c->n_steps; ++s) {
        if (c->step_offsets[s + 1] < c->step_offsets[s]) raise(QSB_ERR_ARGUMENT, "step offsets are not monotone");
        for (int i = c->step_offsets[s]; i < c->step_offsets[s + 1]; ++i) {
            const qsb_op& op = c->ops[i];
            if (op.kind == QSB_OP_FUNCTION && op.function >= 0 && op.function < c->n_functions && c->functions &&
                op.count >= 1 && op.count <= 30 && c->functions[op.function].dim != (int64_t{1} << op.count)) {
                // apply_function's own check (fsv_backend.cpp:90-95)
                raise(QSB_ERR_VALIDATION, "apply_function: matrix dimension %lld does not match 2^%d",
                      static_cast<long long>(c->functions[op.function].dim), op.count);
            }
            check_op(c, op);
            if (op.kind == QSB_OP_INSTRUCTION) continue;  // instructions do not change the state
            FlatOp f{};
            f.cbit = -1;
            if (op.kind == QSB_OP_FUNCTION) {
                f.kind = qsb::kSvFunction;
                f.k = op.count;
                f.tbit = w + (n - op.first - op.count);
                f.fn = op.function;
            } else {
                f.kind = qsb::kSvPair;
                f.tbit = w + (n - 1 - op.target);
                if (op.kind == QSB_OP_CONTROL) f.cbit = w + (n - 1 - op.control);
                std::memcpy(f.u_re, op.u_re, sizeof f.u_re);
                std::memcpy(f.u_im, op.u_im, sizeof f.u_im);
                f.cls = classify(f.u_re, f.u_im);
            }
            out.push_back(f);
        }
    }
    return out;
}

uint64_t target_bits(const FlatOp& f) {
    if (f.kind == qsb::kSvPair) return uint64_t{1} << f.tbit;
    return ((uint64_t{1} << f.k) - 1) << f.tbit;
}

// Targets per register batch: 5 when the batch is compiled straight-line (no
// merge points, 2^5 complex per thread fit in registers) and the array has
// column bits below the targets (structured unitary: coalesced, warp-uniform
// controls); 4 otherwise (measured: r35). QSB_SV_REG_K overrides (tests / tuning).
int reg_k_default(int w, int m) {
    const bool jit = qsbjit::available() && (m >= 18 || qsbjit::forced());
    const int cap = jit ? qsb::kSvRegMaxK : qsb::kSvRegDefaultK;
    const char* e = std::getenv("QSB_SV_REG_K");
    if (e && *e) {
        const int v = std::atoi(e);
        if (v >= 1 && v <= cap) return v;
    }
    return (jit && w >= 5) ? qsb::kSvRegMaxK : qsb::kSvRegDefaultK;
}

// A shared-memory slab batch over ops [i, j) whose target bits are T.
void push_slab_batch(qsb_sv_plan* p, const std::vector<FlatOp>& flat, size_t i, size_t j, uint64_t T, int L,
                     const std::vector<qsb::SvTable>& tabs) {
    const int m = p->m;
    // slab: low run [0, r) plus the targets at or above r, L bits in total
    int r = L;
    while (r > 1 && r + popcount64(T & ~((uint64_t{1} << r) - 1)) > L) --r;
    qsb::SvBatch bt{};
    bt.L = L;
    bt.r = r;
    bt.nhi = 0;
    int local_of[64];
    for (int q = 0; q < 64; ++q) local_of[q] = -1;
    for (int q = 0; q < r; ++q) local_of[q] = q;
    for (int q = r; q < m; ++q)
        if ((T >> q) & 1u) {
            if (bt.nhi >= qsb::kSvMaxHi) raise(QSB_ERR_INTERNAL, "sv batch: too many high slab bits");
            local_of[q] = r + bt.nhi;
            bt.hi[bt.nhi++] = q;
        }
    if (r + bt.nhi != L) raise(QSB_ERR_INTERNAL, "sv batch: slab of %d bits, expected %d", r + bt.nhi, L);
    const uint64_t all = (m >= 64) ? ~uint64_t{0} : ((uint64_t{1} << m) - 1);
    uint64_t slab_mask = (uint64_t{1} << r) - 1;
    for (int q = 0; q < bt.nhi; ++q) slab_mask |= uint64_t{1} << bt.hi[q];
    bt.outer_mask = all & ~slab_mask;
    bt.slabs = int64_t{1} << (m - L);
    bt.op_begin = static_cast<int>(p->ops.size());
    bt.op_count = static_cast<int>(j - i);
    for (size_t q = i; q < j; ++q) {
        const FlatOp& f = flat[q];
        qsb::SvLocalOp lo{};
        lo.kind = f.kind;
        lo.cls = f.cls;
        lo.lt = local_of[f.tbit];
        lo.k = f.k;
        lo.lc = -1;
        if (f.kind == qsb::kSvPair && f.cbit >= 0) {
            if (local_of[f.cbit] >= 0) {
                lo.lc = local_of[f.cbit];
                lo.lcmask = 1u << lo.lc;
            } else {
                lo.ocmask = uint64_t{1} << f.cbit;
            }
        }
        std::memcpy(lo.u_re, f.u_re, sizeof lo.u_re);
        std::memcpy(lo.u_im, f.u_im, sizeof lo.u_im);
        if (f.kind == qsb::kSvFunction) lo.tab = tabs[f.fn];
        if (lo.lt < 0) raise(QSB_ERR_INTERNAL, "sv batch: target outside its slab");
        p->ops.push_back(lo);
    }
    qsb_sv_plan::Pass ps{};
    ps.kind = qsb_sv_plan::kSlab;
    ps.batch = bt;
    p->passes.push_back(ps);
}

// A register batch over pair ops [i, j) whose target bits are T (|T| <= kSvRegMaxK,
// j - i <= kSvRegMaxOps); the ops travel in the launch's parameter space.
void push_reg_batch(qsb_sv_plan* p, const std::vector<FlatOp>& flat, size_t i, size_t j, uint64_t T) {
    auto rb = std::make_shared<qsb::SvRegBatch>();
    std::memset(rb.get(), 0, sizeof(qsb::SvRegBatch));
    int index_of[64];
    for (int q = 0; q < 64; ++q) index_of[q] = -1;
    for (int q = 0; q < p->m; ++q)
        if ((T >> q) & 1u) {
            index_of[q] = rb->K;
            rb->t[rb->K++] = q;
        }
    rb->groups = int64_t{1} << (p->m - rb->K);
    if (j - i > static_cast<size_t>(qsb::kSvRegMaxOps)) raise(QSB_ERR_INTERNAL, "sv register batch too long");
    rb->op_count = static_cast<int>(j - i);
    for (size_t q = i; q < j; ++q) {
        const FlatOp& f = flat[q];
        qsb::SvRegOp& o = rb->ops[q - i];
        o.tb = index_of[f.tbit];
        int cb = -1;
        if (f.cbit >= 0) {
            if (index_of[f.cbit] >= 0) {
                cb = index_of[f.cbit];
                o.emask = 1u << cb;
            } else {
                o.ocmask = 1u << f.cbit;
            }
        }
        o.code = qsb::sv_reg_code(f.cls, o.tb, cb);
        std::memcpy(o.u_re, f.u_re, sizeof o.u_re);
        std::memcpy(o.u_im, f.u_im, sizeof o.u_im);
        if (o.tb < 0) raise(QSB_ERR_INTERNAL, "sv register batch: target outside the batch");
    }
    qsb_sv_plan::Pass ps{};
    ps.kind = qsb_sv_plan::kReg;
    ps.reg = rb;
    p->passes.push_back(ps);
}

// ---- straight-line register batches (qsb_jit.hpp) ----------------------------

const char* kJitPrelude = R"(
#define QSB_MUL(a, b) __dmul_rn(a, b)
#define QSB_ADD(a, b) __dadd_rn(a, b)
#define QSB_SUB(a, b) __dsub_rn(a, b)
)";

// The kernel of one register batch: the same pair updates as pair_math
// (fsv_backend.cpp:52-55, classes qsb_sv.hpp), with every target, control and
// class a constant; X / CNOT pairs without an outer control are a renaming of
// the element variables. Coefficients are appended to *coef in parameter order.
std::string emit_reg_kernel(const std::string& name, const qsb::SvRegBatch& b, std::vector<double>* coef,
                            bool prefetch) {
    const int K = b.K, E = 1 << K;
    std::string o;
    char buf[512];
    auto put = [&](const char* fmt, auto... a) {
        std::snprintf(buf, sizeof buf, fmt, a...);
        o += buf;
    };
    std::vector<int> loc(E);
    for (int e = 0; e < E; ++e) loc[e] = e;
    std::string body;
    auto bput = [&](const char* fmt, auto... a) {
        std::snprintf(buf, sizeof buf, fmt, a...);
        body += buf;
    };
    auto cref = [&](double v) {
        coef->push_back(v);
        return static_cast<int>(coef->size()) - 1;
    };
    for (int k = 0; k < b.op_count; ++k) {
        const qsb::SvRegOp& op = b.ops[k];
        const int cat = op.code / qsb::kSvRegMaxK;
        const int cls = cat < 6 ? cat : (cat < 12 ? cat - 6 : (cat < 17 ? qsb::kPairDiag1 : qsb::kPairSwap));
        const int tb = op.tb;
        const int cb = op.emask ? __builtin_ctz(op.emask) : -1;
        const bool outer = op.ocmask != 0;
        if (outer) bput("    if (f & 0x%xu) {\n", op.ocmask);
        int u[8];
        if (cls == qsb::kPairDiag1) {
            u[0] = cref(op.u_re[3]);
            u[1] = cref(op.u_im[3]);
        } else if (cls == qsb::kPairDiag) {
            u[0] = cref(op.u_re[0]); u[1] = cref(op.u_im[0]); u[2] = cref(op.u_re[3]); u[3] = cref(op.u_im[3]);
        } else if (cls == qsb::kPairAnti) {
            u[0] = cref(op.u_re[1]); u[1] = cref(op.u_im[1]); u[2] = cref(op.u_re[2]); u[3] = cref(op.u_im[2]);
        } else if (cls == qsb::kPairReal) {
            for (int e = 0; e < 4; ++e) u[e] = cref(op.u_re[e]);
        } else if (cls == qsb::kPairGeneral) {
            for (int e = 0; e < 4; ++e) {
                u[2 * e] = cref(op.u_re[e]);
                u[2 * e + 1] = cref(op.u_im[e]);
            }
        }
        for (int e0 = 0; e0 < E; ++e0) {
            if (e0 & (1 << tb)) continue;
            if (cb >= 0 && !(e0 & (1 << cb))) continue;
            const int e1 = e0 | (1 << tb);
            const int A = loc[e0], B = loc[e1];
            switch (cls) {
            case qsb::kPairSwap:
                if (!outer)
                    std::swap(loc[e0], loc[e1]);
                else
                    bput("      { double t = r%d; r%d = r%d; r%d = t; t = i%d; i%d = i%d; i%d = t; }\n", A, A, B, B, A,
                         A, B, B);
                break;
            case qsb::kPairDiag1:
                bput("      { const double nr = QSB_SUB(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], i%d));"
                     " const double ni = QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], r%d)); r%d = nr; i%d = ni; }\n",
                     u[0], B, u[1], B, u[0], B, u[1], B, B, B);
                break;
            case qsb::kPairDiag:
                bput("      { const double n0r = QSB_SUB(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], i%d));"
                     " const double n0i = QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], r%d));\n",
                     u[0], A, u[1], A, u[0], A, u[1], A);
                bput("        const double n1r = QSB_SUB(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], i%d));"
                     " const double n1i = QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], r%d));"
                     " r%d = n0r; i%d = n0i; r%d = n1r; i%d = n1i; }\n",
                     u[2], B, u[3], B, u[2], B, u[3], B, A, A, B, B);
                break;
            case qsb::kPairAnti:
                bput("      { const double n0r = QSB_SUB(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], i%d));"
                     " const double n0i = QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], r%d));\n",
                     u[0], B, u[1], B, u[0], B, u[1], B);
                bput("        const double n1r = QSB_SUB(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], i%d));"
                     " const double n1i = QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], r%d));"
                     " r%d = n0r; i%d = n0i; r%d = n1r; i%d = n1i; }\n",
                     u[2], A, u[3], A, u[2], A, u[3], A, A, A, B, B);
                break;
            case qsb::kPairReal:
                bput("      { const double n0r = QSB_ADD(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], r%d));"
                     " const double n0i = QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], i%d));\n",
                     u[0], A, u[1], B, u[0], A, u[1], B);
                bput("        const double n1r = QSB_ADD(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], r%d));"
                     " const double n1i = QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], i%d));"
                     " r%d = n0r; i%d = n0i; r%d = n1r; i%d = n1i; }\n",
                     u[2], A, u[3], B, u[2], A, u[3], B, A, A, B, B);
                break;
            default: {
                // u00r*a0r - u00i*a0i + u01r*a1r - u01i*a1i, left to right (fsv_backend.cpp:52-55)
                bput("      { const double n0r = QSB_SUB(QSB_ADD(QSB_SUB(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], i%d)),"
                     " QSB_MUL(c.v[%d], r%d)), QSB_MUL(c.v[%d], i%d));\n",
                     u[0], A, u[1], A, u[2], B, u[3], B);
                bput("        const double n0i = QSB_ADD(QSB_ADD(QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], r%d)),"
                     " QSB_MUL(c.v[%d], i%d)), QSB_MUL(c.v[%d], r%d));\n",
                     u[0], A, u[1], A, u[2], B, u[3], B);
                bput("        const double n1r = QSB_SUB(QSB_ADD(QSB_SUB(QSB_MUL(c.v[%d], r%d), QSB_MUL(c.v[%d], i%d)),"
                     " QSB_MUL(c.v[%d], r%d)), QSB_MUL(c.v[%d], i%d));\n",
                     u[4], A, u[5], A, u[6], B, u[7], B);
                bput("        const double n1i = QSB_ADD(QSB_ADD(QSB_ADD(QSB_MUL(c.v[%d], i%d), QSB_MUL(c.v[%d], r%d)),"
                     " QSB_MUL(c.v[%d], i%d)), QSB_MUL(c.v[%d], r%d)); r%d = n0r; i%d = n0i; r%d = n1r; i%d = n1i; }\n",
                     u[4], A, u[5], A, u[6], B, u[7], B, A, A, B, B);
            }
            }
        }
        if (outer) body += "    }\n";
    }
    const int NC = std::max<int>(1, static_cast<int>(coef->size()));
    put("struct QsbCoef_%s { double v[%d]; };\n", name.c_str(), NC);
    put("extern \"C\" __global__ void __launch_bounds__(%d) %s(double* __restrict__ re, double* __restrict__ im,"
        " long long groups, const __grid_constant__ QsbCoef_%s c) {\n",
        qsb::kSvRegThreads, name.c_str(), name.c_str());
    auto pat = [&](int e) {
        unsigned p = 0;
        for (int i = 0; i < K; ++i)
            if (e & (1 << i)) p |= 1u << b.t[i];
        return p;
    };
    std::string base_fn;  // element 0 of group g: g with a zero inserted at every target bit
    for (int i = 0; i < K; ++i) {
        const unsigned low = (1u << b.t[i]) - 1u;
        std::snprintf(buf, sizeof buf, "    f = ((f & ~0x%xu) << 1) | (f & 0x%xu);\n", low, low);
        base_fn += buf;
    }
    // With flat bit 0 among the targets, elements e and e | 1 are adjacent words:
    // one 16-byte access for the pair (f has bit 0 clear, so it is aligned).
    const bool pairs = K > 0 && b.t[0] == 0;
    o += "  const long long stride = (long long)gridDim.x * blockDim.x;\n";
    if (prefetch) {
        // The next group streams into this thread's shared-memory slots (cp.async,
        // [element][plane][thread]) while the current one is updated and stored.
        auto issue = [&](const char* indent) {
            for (int e = 0; e < E; ++e)
                put("%sasm volatile(\"cp.async.ca.shared.global [%%0], [%%1], 8;\" :: \"r\"(slot + %uu), \"l\"(re + (f | 0x%xu)) : \"memory\");"
                    " asm volatile(\"cp.async.ca.shared.global [%%0], [%%1], 8;\" :: \"r\"(slot + %uu), \"l\"(im + (f | 0x%xu)) : \"memory\");\n",
                    indent, static_cast<unsigned>((2 * e) * qsb::kSvRegThreads * 8), pat(e),
                    static_cast<unsigned>((2 * e + 1) * qsb::kSvRegThreads * 8), pat(e));
            put("%sasm volatile(\"cp.async.commit_group;\" ::: \"memory\");\n", indent);
        };
        o += "  extern __shared__ double qsb_slots[];\n";
        o += "  const unsigned slot = (unsigned)__cvta_generic_to_shared(qsb_slots) + threadIdx.x * 8u;\n";
        o += "  long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;\n";
        o += "  if (g < groups) {\n    unsigned f = (unsigned)g;\n" + base_fn;
        issue("    ");
        o += "  }\n";
        o += "  for (; g < groups; g += stride) {\n    unsigned f = (unsigned)g;\n" + base_fn;
        o += "    asm volatile(\"cp.async.wait_all;\" ::: \"memory\");\n";
        for (int e = 0; e < E; ++e)
            put("    double r%d = qsb_slots[%d * %d + threadIdx.x]; double i%d = qsb_slots[%d * %d + threadIdx.x];\n", e,
                2 * e, qsb::kSvRegThreads, e, 2 * e + 1, qsb::kSvRegThreads);
        o += "    if (g + stride < groups) {\n      const unsigned f0 = f;\n      { unsigned f = (unsigned)(g + stride);\n";
        std::string indented;
        for (size_t q = 0; q < base_fn.size(); ++q) {
            if (q == 0 || base_fn[q - 1] == '\n') indented += "    ";
            indented += base_fn[q];
        }
        o += indented;
        issue("        ");
        o += "      }\n      (void)f0;\n    }\n";
    } else {
        o += "  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {\n";
        o += "    unsigned f = (unsigned)g;\n" + base_fn;
        if (pairs) {
            for (int e = 0; e < E; e += 2)
                put("    double r%d, r%d, i%d, i%d; { const double2 a = __ldcs(reinterpret_cast<const double2*>(re + (f | 0x%xu)));"
                    " const double2 b = __ldcs(reinterpret_cast<const double2*>(im + (f | 0x%xu)));"
                    " r%d = a.x; r%d = a.y; i%d = b.x; i%d = b.y; }\n",
                    e, e + 1, e, e + 1, pat(e), pat(e), e, e + 1, e, e + 1);
        } else {
            for (int e = 0; e < E; ++e)
                put("    double r%d = __ldcs(re + (f | 0x%xu)); double i%d = __ldcs(im + (f | 0x%xu));\n", e, pat(e), e,
                    pat(e));
        }
    }
    o += body;
    if (pairs) {
        for (int e = 0; e < E; e += 2)
            put("    __stcs(reinterpret_cast<double2*>(re + (f | 0x%xu)), make_double2(r%d, r%d));"
                " __stcs(reinterpret_cast<double2*>(im + (f | 0x%xu)), make_double2(i%d, i%d));\n",
                pat(e), loc[e], loc[e + 1], pat(e), loc[e], loc[e + 1]);
    } else {
        for (int e = 0; e < E; ++e)
            put("    __stcs(re + (f | 0x%xu), r%d); __stcs(im + (f | 0x%xu), i%d);\n", pat(e), loc[e], pat(e), loc[e]);
    }
    o += "  }\n}\n";
    return o;
}

// Compile every register batch of the plan into one module (cached by source).
void jit_register_batches(qsb_sv_plan* p) {
    if (!qsbjit::available()) return;
    if (p->m < 18 && !qsbjit::forced()) return;  // small arrays: the interpreted kernel, no compile latency
    std::string src = kJitPrelude;
    // cp.async prefetch of the next group (QSB_SV_JIT_PREFETCH=0: direct loads)
    const char* pe = std::getenv("QSB_SV_JIT_PREFETCH");
    const bool prefetch = !(pe && std::strcmp(pe, "0") == 0);
    std::vector<std::string> names;
    std::vector<size_t> idx;
    for (size_t i = 0; i < p->passes.size(); ++i) {
        qsb_sv_plan::Pass& ps = p->passes[i];
        if (ps.kind != qsb_sv_plan::kReg) continue;
        const std::string name = "qsb_sv_b" + std::to_string(i);
        ps.coef.clear();
        src += emit_reg_kernel(name, *ps.reg, &ps.coef, prefetch);
        names.push_back(name);
        idx.push_back(i);
    }
    if (names.empty()) return;
    if (const char* dump = std::getenv("QSB_SV_JIT_DUMP")) {  // debugging: the generated source
        if (FILE* fp = std::fopen(dump, "w")) {
            std::fputs(src.c_str(), fp);
            std::fclose(fp);
        }
    }
    const std::vector<void*> fns = qsbjit::kernels(src, names);
    for (size_t k = 0; k < idx.size(); ++k) {
        qsb_sv_plan::Pass& ps = p->passes[idx[k]];
        ps.jit = fns[k];
        ps.jit_smem = prefetch ? 2 * (1 << ps.reg->K) * qsb::kSvRegThreads * 8 : 0;
        if (ps.coef.empty()) ps.coef.push_back(0.0);
    }
}

// Group the ops into passes, in order: runs of gates / controlled gates on at
// most K distinct targets become register batches; apply_function blocks that
// fit a shared-memory slab become slab batches (consecutive ones merged); larger
// blocks get the out-of-place function kernel.
void build_passes(qsb_sv_plan* p, const std::vector<FlatOp>& flat, const std::vector<qsb::SvTable>& tabs) {
    const int m = p->m;
    const int L = std::min(slab_bits_default(), m);
    // blocks of up to 2^6 run inside a slab; larger ones get their own pass
    // (one thread per output: a 2^k-term sum per element is too long for one CTA)
    const int kmax = std::min((m <= L) ? m : L - 5, 6);
    const int KR = std::min(reg_k_default(p->w, m), m);
    size_t i = 0;
    int max_targets = 0;
    while (i < flat.size()) {
        const FlatOp& f0 = flat[i];
        if (f0.kind == qsb::kSvFunction && f0.k > kmax) {
            qsb_sv_plan::Pass ps{};
            ps.kind = qsb_sv_plan::kFn;
            ps.f = {f0.k, f0.tbit, tabs[f0.fn]};
            p->passes.push_back(ps);
            ++p->info.n_function_passes;
            ++i;
            continue;
        }
        // a state of at most one slab: every op in one shared-memory launch
        const bool fn_run = f0.kind == qsb::kSvFunction || m <= L;
        const int cap = m <= L ? m : (fn_run ? kmax : KR);
        uint64_t T = 0;
        size_t j = i;
        while (j < flat.size()) {
            const FlatOp& f = flat[j];
            if (m > L && (f.kind == qsb::kSvFunction) != fn_run) break;
            if (f.kind == qsb::kSvFunction && f.k > kmax) break;
            if (!fn_run && j - i >= static_cast<size_t>(qsb::kSvRegMaxOps)) break;
            const uint64_t need = T | target_bits(f);
            if (popcount64(need) > cap) break;
            T = need;
            ++j;
        }
        max_targets = std::max(max_targets, popcount64(T));
        if (fn_run)
            push_slab_batch(p, flat, i, j, T, L, tabs);
        else
            push_reg_batch(p, flat, i, j, T);
        i = j;
    }
    p->info.slab_bits = L;
    p->info.max_batch_targets = max_targets;
}

std::unique_ptr<qsb_sv_plan> make_sv_plan(qsb_handle* h, DeviceCtx* dc, const qsb_circuit* c, int mode,
                                          int64_t col_begin, int64_t col_count, bool borrow_cache) {
    validate_circuit_shape(c);
    if (mode == QSB_SV_STATE)
        sv_check_guard(c, h->fsv_guard, "fsv-b200");
    else if (mode == QSB_SV_UNITARY)
        sv_check_guard(c, h->structured_guard, "unitary-structured-b200");
    else
        raise(QSB_ERR_ARGUMENT, "unknown state-vector mode %d", mode);
    auto p = std::make_unique<qsb_sv_plan>();
    p->h = h;
    p->dc = dc;
    p->mode = mode;
    p->n = c->n_qubits;
    const int64_t N = int64_t{1} << p->n;
    if (mode == QSB_SV_UNITARY) {
        if (col_count < 1 || (col_count & (col_count - 1)) != 0 || col_count > N || col_begin < 0 ||
            col_begin % col_count != 0 || col_begin + col_count > N)
            raise(QSB_ERR_ARGUMENT, "column shard [%lld, +%lld) must be an aligned power-of-two block of [0, %lld)",
                  static_cast<long long>(col_begin), static_cast<long long>(col_count), static_cast<long long>(N));
        p->col_begin = col_begin;
        p->col_count = col_count;
        int w = 0;
        while ((int64_t{1} << w) < col_count) ++w;
        p->w = w;
    } else {
        p->col_begin = 0;
        p->col_count = 1;
        p->w = 0;
    }
    p->m = p->n + p->w;
    if (p->m > 32) raise(QSB_ERR_RESOURCE, "state-vector array of 2^%d elements exceeds the engine's 32-bit indexing", p->m);
    const std::vector<FlatOp> flat = flatten_ops(c, p->w);

    DeviceScope ds(dc->device);
    if (borrow_cache) {
        p->b = std::move(dc->cache);
        p->borrowed = true;
    }
    // registered matrices used by the circuit, uploaded once per plan as CSR
    // of their nonzeros (qsb_sv.hpp SvTable)
    std::vector<qsb::SvTable> tabs(static_cast<size_t>(std::max(c->n_functions, 0)));
    {
        std::vector<char> used(tabs.size(), 0);
        for (const FlatOp& f : flat)
            if (f.kind == qsb::kSvFunction) used[f.fn] = 1;
        struct Csr {
            std::vector<int32_t> rp, ci;
            std::vector<double> vr, vi;
        };
        std::vector<Csr> csr(tabs.size());
        size_t bytes = 0;
        for (size_t fi = 0; fi < used.size(); ++fi) {
            if (!used[fi]) continue;
            const qsb_function& fn = c->functions[fi];
            const int64_t d = fn.dim;
            Csr& cs = csr[fi];
            // two parallel sweeps over row chunks (count, then fill) on the host's cores
            const int64_t workers =
                d >= 512 ? std::min<int64_t>(16, std::max(1u, std::thread::hardware_concurrency())) : 1;
            auto run = [&](auto&& body) {
                if (workers <= 1) {
                    body(int64_t{0}, d);
                    return;
                }
                std::vector<std::thread> pool;
                for (int64_t w = 0; w < workers; ++w) pool.emplace_back(body, d * w / workers, d * (w + 1) / workers);
                for (auto& t : pool) t.join();
            };
            cs.rp.assign(d + 1, 0);
            run([&](int64_t r0, int64_t r1) {
                for (int64_t r = r0; r < r1; ++r) {
                    int32_t nz = 0;
                    for (int64_t k = 0; k < d; ++k) nz += (fn.re[r * d + k] != 0.0 || fn.im[r * d + k] != 0.0);
                    cs.rp[r + 1] = nz;
                }
            });
            for (int64_t r = 0; r < d; ++r) cs.rp[r + 1] += cs.rp[r];
            cs.ci.resize(cs.rp[d]);
            cs.vr.resize(cs.rp[d]);
            cs.vi.resize(cs.rp[d]);
            run([&](int64_t r0, int64_t r1) {
                for (int64_t r = r0; r < r1; ++r) {
                    int32_t z = cs.rp[r];
                    for (int64_t k = 0; k < d; ++k) {
                        const double a = fn.re[r * d + k], b = fn.im[r * d + k];
                        if (a == 0.0 && b == 0.0) continue;
                        cs.ci[z] = static_cast<int32_t>(k);
                        cs.vr[z] = a;
                        cs.vi[z] = b;
                        ++z;
                    }
                }
            });
            bytes += 16 * cs.vr.size() + 4 * (cs.rp.size() + cs.ci.size()) + 64;
        }
        if (bytes > 0) {
            p->b.tables.ensure(bytes);
            char* base = p->b.tables.as<char>();
            size_t off = 0;
            auto put = [&](const void* src, size_t nbytes) {
                char* dst = base + off;
                if (nbytes)  // on the plan stream: ordered before the passes that read the tables
                    cuda_check(cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyHostToDevice, dc->stream), "upload function");
                off += (nbytes + 15) & ~size_t{15};
                return dst;
            };
            for (size_t fi = 0; fi < used.size(); ++fi) {
                if (!used[fi]) continue;
                Csr& cs = csr[fi];
                tabs[fi].vr = reinterpret_cast<const double*>(put(cs.vr.data(), 8 * cs.vr.size()));
                tabs[fi].vi = reinterpret_cast<const double*>(put(cs.vi.data(), 8 * cs.vi.size()));
                tabs[fi].rp = reinterpret_cast<const int32_t*>(put(cs.rp.data(), 4 * cs.rp.size()));
                tabs[fi].ci = reinterpret_cast<const int32_t*>(put(cs.ci.data(), 4 * cs.ci.size()));
            }
        }
    }
    build_passes(p.get(), flat, tabs);
    jit_register_batches(p.get());
    const size_t elems = static_cast<size_t>(N) * static_cast<size_t>(p->col_count);
    p->b.v[0].ensure(2 * elems * sizeof(double));
    if (p->info.n_function_passes > 0) p->b.v[1].ensure(2 * elems * sizeof(double));
    if (mode == QSB_SV_STATE) {
        p->b.x.ensure(2 * elems * sizeof(double));
        double* x = p->b.x.as<double>();
        cuda_check(qsb::sv_launch_init_identity(x, x + elems, N, 1, 0, dc->stream), "sv_init_identity");
    }
    if (!p->ops.empty()) {
        const size_t bytes = p->ops.size() * sizeof(qsb::SvLocalOp);
        p->b.layers.ensure(bytes);
        void* st = dc->stage(bytes);
        std::memcpy(st, p->ops.data(), bytes);
        cuda_check(cudaMemcpyAsync(p->b.layers.p, st, bytes, cudaMemcpyHostToDevice, dc->stream), "upload ops");
    }
    // Plans executed on a caller's stream must see the uploads (host-API calls run on dc->stream).
    if (!borrow_cache) cuda_check(cudaStreamSynchronize(dc->stream), "cudaStreamSynchronize");
    qsb_sv_plan_info& in = p->info;
    in.n_qubits = p->n;
    in.mode = mode;
    in.n_ops = static_cast<int>(flat.size());
    in.n_passes = static_cast<int>(p->passes.size());
    in.n_launches = 1 + in.n_passes;
    in.col_begin = p->col_begin;
    in.col_count = p->col_count;
    double bytes = 0.0;
    for (const auto& ps : p->passes) {
        bytes += 2.0 * 16.0 * static_cast<double>(elems);  // read + write the whole array
        if (ps.kind == qsb_sv_plan::kFn) bytes += 0.0;  // the CSR table is small next to the array
    }
    in.bytes_per_run = bytes;
    return p;
}

void release_sv_plan(std::unique_ptr<qsb_sv_plan>& p) {
    if (!p) return;
    if (p->borrowed) {
        DeviceScope ds(p->dc->device);
        p->dc->cache = std::move(p->b);
    }
    p.reset();
}

void sv_execute(qsb_sv_plan* p, cudaStream_t s) {
    DeviceScope ds(p->dc->device);
    const int64_t R = int64_t{1} << p->n;
    const size_t elems = static_cast<size_t>(R) * static_cast<size_t>(p->col_count);
    double* v0 = p->b.v[0].as<double>();
    if (p->mode == QSB_SV_STATE) {
        cuda_check(cudaMemcpyAsync(v0, p->b.x.p, 2 * elems * sizeof(double), cudaMemcpyDeviceToDevice, s),
                   "copy psi0");
    } else {
        cuda_check(qsb::sv_launch_init_identity(v0, v0 + elems, R, p->col_count, p->col_begin, s),
                   "sv_init_identity");
    }
    int cur = 0;
    const qsb::SvLocalOp* ops = p->b.layers.as<qsb::SvLocalOp>();
    for (const auto& ps : p->passes) {
        double* v = p->b.v[cur].as<double>();
        if (ps.kind == qsb_sv_plan::kReg && ps.jit) {
            double* vre = v;
            double* vim = v + elems;
            long long groups = static_cast<long long>(ps.reg->groups);
            void* args[] = {&vre, &vim, &groups, const_cast<double*>(ps.coef.data())};
            const long long blocks = (groups + qsb::kSvRegThreads - 1) / qsb::kSvRegThreads;
            const unsigned grid = static_cast<unsigned>(std::min<long long>(blocks, 148LL * 8));
            cuda_check(qsbjit::launch(ps.jit, grid, qsb::kSvRegThreads, s, args, ps.jit_smem), "sv jit kernel");
        } else if (ps.kind == qsb_sv_plan::kReg) {
            cuda_check(qsb::sv_launch_reg(v, v + elems, *ps.reg, s), "sv_reg_kernel");
        } else if (ps.kind == qsb_sv_plan::kSlab) {
            cuda_check(qsb::sv_launch_batch(v, v + elems, ops, ps.batch, s), "sv_batch_kernel");
        } else {
            double* o = p->b.v[1 - cur].as<double>();
            cuda_check(qsb::sv_launch_function(v, v + elems, o, o + elems, ps.f.tab, ps.f.k, ps.f.s, p->m,
                                               s),
                       "sv_function_kernel");
            cur ^= 1;
        }
    }
    p->final_buf = cur;
}

const double* sv_result(const qsb_sv_plan* p) { return p->b.v[p->final_buf].as<double>(); }
size_t sv_elems(const qsb_sv_plan* p) { return (size_t{1} << p->n) * static_cast<size_t>(p->col_count); }

// Host-API structured unitary: columns sharded over the handle's devices.
void run_structured(qsb_handle* h, const qsb_circuit* c, double* u_re, double* u_im, double* psi_re,
                    double* psi_im) {
    std::lock_guard<std::mutex> lk(h->mu);
    h->drop_plan_cache();  // the dense path's kept V buffers would sit next to U
    validate_circuit_shape(c);
    const int64_t N = int64_t{1} << c->n_qubits;
    int G = static_cast<int>(h->devs.size());
    while (G > 1 && (N % G != 0 || (G & (G - 1)) != 0)) --G;
    const int64_t cols = N / G;
    std::vector<std::unique_ptr<qsb_sv_plan>> plans(G);
    auto release_all = [&] {
        for (auto& p : plans) release_sv_plan(p);
    };
    try {
        for (int g = 0; g < G; ++g)
            plans[g] = make_sv_plan(h, h->devs[g].get(), c, QSB_SV_UNITARY, g * cols, cols, true);
        for (int g = 0; g < G; ++g) {
            qsb_sv_plan* p = plans[g].get();
            DeviceScope ds(p->dc->device);
            cudaStream_t s = p->dc->stream;
            sv_execute(p, s);
            const double* v = sv_result(p);
            const size_t elems = sv_elems(p);
            if (u_re) {
                cuda_check(cudaMemcpy2DAsync(u_re + p->col_begin, N * 8, v, cols * 8, cols * 8, N,
                                             cudaMemcpyDeviceToHost, s),
                           "download U");
                cuda_check(cudaMemcpy2DAsync(u_im + p->col_begin, N * 8, v + elems, cols * 8, cols * 8, N,
                                             cudaMemcpyDeviceToHost, s),
                           "download U");
            }
            if (psi_re && p->col_begin == 0) {  // psi = U e_0 = column 0
                cuda_check(cudaMemcpy2DAsync(psi_re, 8, v, cols * 8, 8, N, cudaMemcpyDeviceToHost, s), "download psi");
                cuda_check(cudaMemcpy2DAsync(psi_im, 8, v + elems, cols * 8, 8, N, cudaMemcpyDeviceToHost, s),
                           "download psi");
            }
        }
        for (int g = 0; g < G; ++g) {
            DeviceScope ds(plans[g]->dc->device);
            cuda_check(cudaStreamSynchronize(plans[g]->dc->stream), "cudaStreamSynchronize");
        }
    } catch (...) {
        release_all();
        throw;
    }
    release_all();
}

void run_fsv(qsb_handle* h, const qsb_circuit* c, const double* psi0_re, const double* psi0_im, double* psi_re,
             double* psi_im) {
    std::lock_guard<std::mutex> lk(h->mu);
    h->drop_plan_cache();
    DeviceCtx& dc = h->dev0();
    std::unique_ptr<qsb_sv_plan> p = make_sv_plan(h, &dc, c, QSB_SV_STATE, 0, 1, true);
    try {
        DeviceScope ds(dc.device);
        const size_t N = size_t{1} << c->n_qubits;
        if (psi0_re) {
            double* x = p->b.x.as<double>();
            cuda_check(cudaMemcpyAsync(x, psi0_re, N * 8, cudaMemcpyHostToDevice, dc.stream), "upload psi0");
            cuda_check(cudaMemcpyAsync(x + N, psi0_im, N * 8, cudaMemcpyHostToDevice, dc.stream), "upload psi0");
        }
        sv_execute(p.get(), dc.stream);
        const double* v = sv_result(p.get());
        if (N <= 65536) {  // both planes in one copy through pinned staging
            double* st = static_cast<double*>(dc.stage_out(2 * N * 8));
            cuda_check(cudaMemcpyAsync(st, v, 2 * N * 8, cudaMemcpyDeviceToHost, dc.stream), "download psi");
            cuda_check(cudaStreamSynchronize(dc.stream), "cudaStreamSynchronize");
            std::memcpy(psi_re, st, N * 8);
            std::memcpy(psi_im, st + N, N * 8);
        } else {
            cuda_check(cudaMemcpyAsync(psi_re, v, N * 8, cudaMemcpyDeviceToHost, dc.stream), "download psi");
            cuda_check(cudaMemcpyAsync(psi_im, v + N, N * 8, cudaMemcpyDeviceToHost, dc.stream), "download psi");
            cuda_check(cudaStreamSynchronize(dc.stream), "cudaStreamSynchronize");
        }
    } catch (...) {
        release_sv_plan(p);
        throw;
    }
    release_sv_plan(p);
}

}  // namespace

extern "C" {

qsb_status qsb_fsv_qubit_guard(const qsb_handle* h, int32_t* guard) {
    return guarded([&] {
        if (!h || !guard) raise(QSB_ERR_ARGUMENT, "null argument");
        *guard = h->fsv_guard;
    });
}

qsb_status qsb_structured_qubit_guard(const qsb_handle* h, int32_t* guard) {
    return guarded([&] {
        if (!h || !guard) raise(QSB_ERR_ARGUMENT, "null argument");
        *guard = h->structured_guard;
    });
}

qsb_status qsb_fsv_simulate_full_state(qsb_handle* h, const qsb_circuit* c, double* psi_re, double* psi_im) {
    return guarded([&] {
        if (!h || !psi_re || !psi_im) raise(QSB_ERR_ARGUMENT, "null argument");
        run_fsv(h, c, nullptr, nullptr, psi_re, psi_im);
    });
}

qsb_status qsb_fsv_simulate_from_state(qsb_handle* h, const qsb_circuit* c, const double* psi0_re,
                                       const double* psi0_im, double* psi_re, double* psi_im) {
    return guarded([&] {
        if (!h || !psi0_re || !psi0_im || !psi_re || !psi_im) raise(QSB_ERR_ARGUMENT, "null argument");
        run_fsv(h, c, psi0_re, psi0_im, psi_re, psi_im);
    });
}

qsb_status qsb_structured_build_unitary(qsb_handle* h, const qsb_circuit* c, double* u_re, double* u_im) {
    return guarded([&] {
        if (!h || !u_re || !u_im) raise(QSB_ERR_ARGUMENT, "null argument");
        run_structured(h, c, u_re, u_im, nullptr, nullptr);
    });
}

qsb_status qsb_structured_simulate_full_state(qsb_handle* h, const qsb_circuit* c, double* psi_re,
                                              double* psi_im) {
    return guarded([&] {
        if (!h || !psi_re || !psi_im) raise(QSB_ERR_ARGUMENT, "null argument");
        run_structured(h, c, nullptr, nullptr, psi_re, psi_im);
    });
}

qsb_status qsb_sv_plan_create(qsb_handle* h, const qsb_circuit* c, int32_t mode, int64_t col_begin,
                              int64_t col_count, qsb_sv_plan** out) {
    return guarded([&] {
        if (!h || !out) raise(QSB_ERR_ARGUMENT, "null argument");
        *out = nullptr;
        std::lock_guard<std::mutex> lk(h->mu);  // make_sv_plan writes the device's pinned staging
        h->drop_plan_cache();
        std::unique_ptr<qsb_sv_plan> p = make_sv_plan(h, &h->dev0(), c, mode, col_begin, col_count, false);
        *out = p.release();
    });
}

qsb_status qsb_sv_plan_destroy(qsb_sv_plan* plan) {
    return guarded([&] {
        std::unique_ptr<qsb_sv_plan> p(plan);
        release_sv_plan(p);
    });
}

qsb_status qsb_sv_plan_get_info(const qsb_sv_plan* plan, qsb_sv_plan_info* info) {
    return guarded([&] {
        if (!plan || !info) raise(QSB_ERR_ARGUMENT, "null argument");
        *info = plan->info;
    });
}

qsb_status qsb_sv_plan_set_state(qsb_sv_plan* plan, const double* re, const double* im, void* stream) {
    return guarded([&] {
        if (!plan || !re || !im) raise(QSB_ERR_ARGUMENT, "null argument");
        if (plan->mode != QSB_SV_STATE) raise(QSB_ERR_ARGUMENT, "set_state needs a QSB_SV_STATE plan");
        DeviceScope ds(plan->dc->device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : plan->dc->stream;
        const size_t N = size_t{1} << plan->n;
        double* x = plan->b.x.as<double>();
        cuda_check(cudaMemcpyAsync(x, re, N * 8, cudaMemcpyDefault, s), "copy psi0");
        cuda_check(cudaMemcpyAsync(x + N, im, N * 8, cudaMemcpyDefault, s), "copy psi0");
    });
}

qsb_status qsb_sv_plan_execute(qsb_sv_plan* plan, void* stream) {
    return guarded([&] {
        if (!plan) raise(QSB_ERR_ARGUMENT, "null argument");
        sv_execute(plan, stream ? static_cast<cudaStream_t>(stream) : plan->dc->stream);
    });
}

qsb_status qsb_sv_plan_result_device(const qsb_sv_plan* plan, const double** re, const double** im) {
    return guarded([&] {
        if (!plan || !re || !im) raise(QSB_ERR_ARGUMENT, "null argument");
        *re = sv_result(plan);
        *im = sv_result(plan) + sv_elems(plan);
    });
}

}  // extern "C"
