// qsb_sv.hpp — descriptors of the state-vector engine shared by its host
// runtime (qsb_sv.cpp) and its sm_100a kernels (qsb_sv.cu).
//
// The engine evolves a [2][R][W] split-plane array (R = 2^n amplitudes of a
// state, W columns evolved together) by the reference's full-state-vector
// operations (fsv_backend.cpp:40-158), in circuit order:
//   * W = 1            : FsvSimulator — one state vector;
//   * W = 2^n columns  : the structured unitary — U[:, c] = fsv(e_c) for every
//                        column c at once, i.e. U built without a dense GEMM.
// The flat index of element (row, col) is row * W + col, an m = n + log2(W) bit
// number; qubit q acts on flat bit w + (n - 1 - q) (qubit 0 = MSB, gates.hpp:24-27).
//
// Consecutive operations are grouped into "batches" whose target bits (and the
// bits of small function blocks) number at most kmax. One launch applies a
// whole batch: each CTA stages a "slab" of 2^L elements in shared memory — the
// elements that vary in the batch's target bits plus the lowest flat bits (so
// global accesses are coalesced runs) — applies every operation of the batch to
// it in order, and writes it back. A slab is closed under every operation of
// its batch (each pair / block lies inside one slab; control bits outside the
// slab are constant over it), so the result is exactly the sequential
// operation-by-operation update of the reference.
#pragma once

#include <cstdint>

namespace qsb {

constexpr int kSvMaxHi = 8;        // high slab bits (targets above the low run)
constexpr int kSvMaxSlabBits = 12; // 2^12 elements x 16 B = 64 KB of shared memory
constexpr int kSvThreads = 256;

enum SvOpKind : int32_t { kSvPair = 0, kSvFunction = 1 };

// Pair-update classes (host-classified from the exact 2x2 entries). Every class
// computes the same values as the reference's general pair update
// (fsv_backend.cpp:52-55) — terms whose coefficient is an exact zero contribute
// a signed zero, which changes at most the sign of a zero result.
enum SvPairClass : int32_t {
    kPairGeneral = 0,  // full complex 2x2
    kPairReal = 1,     // all imaginary parts zero (H)
    kPairDiag = 2,     // u01 = u10 = 0
    kPairDiag1 = 3,    // diagonal with u00 = 1: only the |1> amplitude changes (Z, S, T, R, CR)
    kPairAnti = 4,     // u00 = u11 = 0 (Y)
    kPairSwap = 5      // u = X: exchange the pair
};

// A registered matrix as its nonzero entries, row by row with ascending
// columns (CSR). apply_function's sums run k = 0..2^k-1 in order
// (fsv_backend.cpp:119-126); a term whose matrix entry is an exact zero adds a
// signed zero, so summing only the nonzeros in the same order gives the same
// value (DJ oracles are permutations: one term per row instead of 2^k).
struct SvTable {
    const int32_t* rp;  // 2^k + 1 row pointers
    const int32_t* ci;  // column of each nonzero
    const double* vr;   // nonzero values
    const double* vi;
};

// One operation, translated into the local index space of its batch's slab.
struct SvLocalOp {
    int32_t kind;     // SvOpKind
    int32_t cls;      // SvPairClass (pairs)
    int32_t lt;       // pair: local target bit; function: local bit of the block's least significant qubit
    int32_t k;        // function: qubit count (block = 2^k)
    uint32_t lcmask;  // pair: control bits inside the slab (local positions)
    int32_t lc;       // pair: local control bit, or -1
    uint64_t ocmask;  // control bits outside the slab (flat positions): the op applies iff all are set
    double u_re[4];
    double u_im[4];
    SvTable tab;      // function: the registered matrix on the device
};

// One batch launch.
struct SvBatch {
    int32_t op_begin;
    int32_t op_count;
    int32_t L;            // slab bits
    int32_t r;            // low run: local bits [0, r) are flat bits [0, r)
    int32_t nhi;          // local bits [r, L) are flat bits hi[0..nhi)
    int32_t pad;
    int32_t hi[kSvMaxHi];
    uint64_t outer_mask;  // flat bits outside the slab (enumerate the slabs)
    int64_t slabs;
};

// A register batch: gate / controlled-gate operations on at most kSvRegMaxK
// distinct target bits. Each thread owns the 2^K elements of one "group" (the
// elements that differ only in the K target bits), loads them straight from
// HBM into registers, applies every operation of the batch, and stores them:
// one read + one write of the array per batch, no shared memory, no barriers.
// The operations travel in the kernel's parameter space (constant bank:
// uniform, no global-load latency per operation).
constexpr int kSvRegMaxK = 5;      // dispatch-code stride (sv_reg_code)
constexpr int kSvRegDefaultK = 4;  // largest K launched: 2^4 complex per thread, 160 registers, no spills
constexpr int kSvRegThreads = 128;
constexpr int kSvRegMaxOps = 192;  // 192 x 80 B: the launch stays under the 32 KB parameter limit

// Dispatch code of a register-batch op: category * kSvRegMaxK + target index.
// Categories 0-5: class (SvPairClass order) with no control inside the targets;
// 6-11: class with the control mask emask tested at run time; 12-16: diag-1
// (controlled phase) with the control at target index 0-4; 17-21: X (CNOT) likewise.
inline int32_t sv_reg_code(int32_t cls, int32_t tb, int32_t cb /* control index in t[], or -1 */) {
    static const int kCat[6] = {0, 1, 2, 3, 4, 5};  // SvPairClass -> category without control
    int cat;
    if (cb < 0)
        cat = kCat[cls];
    else if (cls == 3 /* kPairDiag1 */)
        cat = 12 + cb;
    else if (cls == 5 /* kPairSwap */)
        cat = 17 + cb;
    else
        cat = 6 + cls;
    return cat * 5 /* kSvRegMaxK */ + tb;
}

struct SvRegOp {
    int32_t code;     // sv_reg_code(cls, tb, control index)
    int32_t tb;       // index of the target within t[]
    uint32_t emask;   // control inside t[] (e-space bit), or 0
    uint32_t ocmask;  // control outside t[] (flat bit, tested on the group's element 0), or 0
    double u_re[4];
    double u_im[4];
};

struct SvRegBatch {
    int32_t op_count;
    int32_t K;
    int32_t t[kSvRegMaxK];  // flat target bits, ascending
    int32_t pad;
    int64_t groups;         // 2^(m - K)
    SvRegOp ops[kSvRegMaxOps];
};

// Launch wrappers (qsb_sv.cu); return cudaError_t as int.
int sv_launch_reg(double* re, double* im, const SvRegBatch& b, void* stream);
int sv_configure();
int sv_launch_batch(double* re, double* im, const SvLocalOp* ops, const SvBatch& b, void* stream);
// out[o][row][i] = sum_kk m[row][kk] * in[o][kk][i] for a 2^k block at flat bit s
// of an m-bit array (apply_function, fsv_backend.cpp:84-132, for blocks too
// large for one slab). Out of place.
int sv_launch_function(const double* in_re, const double* in_im, double* out_re, double* out_im,
                       const SvTable& tab, int k, int s, int m, void* stream);
// re[i * W + c] = (i == col_begin + c), im = 0: identity columns (W = 1, col_begin = 0: |0...0>).
int sv_launch_init_identity(double* re, double* im, int64_t R, int64_t W, int64_t col_begin, void* stream);

}  // namespace qsb
