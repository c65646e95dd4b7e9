// qsb_sv.cu — sm_100a kernels of the state-vector engine (qsb_sv.hpp):
//
//   sv_batch_kernel     one batch of gate / controlled-gate / small-function
//                       operations applied to shared-memory slabs of the
//                       [2][R][W] array (HBM-bound: one read + one write of the
//                       array per batch, however many operations it holds).
//   sv_function_kernel  apply_function for blocks too large for a slab
//                       (out of place, sequential k-order sums).
//   sv_init_identity    identity columns / |0...0>.
//
// Reference loops replaced (paths relative to /root/reference/proj):
//   update_pairs (apply_gate, apply_control_gate)  core/src/fsv_backend.cpp:40-82
//   apply_function                                 core/src/fsv_backend.cpp:84-132
//   FsvSimulator::simulate_full_state              core/src/fsv_backend.cpp:135-158
//   zero_state                                     core/src/state.cpp:37-47
// Every product and sum is rounded separately (__dmul_rn / __dadd_rn /
// __dsub_rn) in the reference's evaluation order (x86-64, no FMA contraction),
// so the state matches the reference's fsv backend bit for bit (up to the sign
// of zeros, which ComplexVector comparisons ignore).
#include <cuda_runtime.h>

#include <cstdint>

#include "qsb_sv.hpp"

namespace qsb {

namespace detail {

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// Local slab index j -> flat element index (without the slab's base).
__device__ __forceinline__ uint64_t local_to_flat(uint32_t j, const SvBatch& b) {
    const uint32_t lo = j & ((1u << b.r) - 1u);
    uint32_t hi = j >> b.r;
    uint64_t f = lo;
#pragma unroll
    for (int i = 0; i < kSvMaxHi; ++i) {
        if (i < b.nhi && ((hi >> i) & 1u)) f |= uint64_t{1} << b.hi[i];
    }
    return f;
}

// Insert bit value v at position p of x.
__device__ __forceinline__ uint32_t insert_bit(uint32_t x, int p, uint32_t v) {
    const uint32_t low = x & ((1u << p) - 1u);
    return ((x >> p) << (p + 1)) | (v << p) | low;
}

// The pair update of fsv_backend.cpp:52-55 for one class, on values:
// (a0, a1) -> (a0', a1') with i0 = target bit clear, i1 = target bit set.
template <int CLS, typename Op>
__device__ __forceinline__ void pair_math(const Op& op, double& a0r, double& a0i, double& a1r, double& a1i) {
    if (CLS == kPairSwap) {
        const double tr = a0r, ti = a0i;
        a0r = a1r; a0i = a1i;
        a1r = tr; a1i = ti;
    } else if (CLS == kPairDiag1) {
        const double ur = op.u_re[3], ui = op.u_im[3];
        const double r = ds(dm(ur, a1r), dm(ui, a1i));
        const double i = da(dm(ur, a1i), dm(ui, a1r));
        a1r = r; a1i = i;
    } else if (CLS == kPairDiag) {
        const double u0r = op.u_re[0], u0i = op.u_im[0], u3r = op.u_re[3], u3i = op.u_im[3];
        const double r0 = ds(dm(u0r, a0r), dm(u0i, a0i));
        const double i0 = da(dm(u0r, a0i), dm(u0i, a0r));
        const double r1 = ds(dm(u3r, a1r), dm(u3i, a1i));
        const double i1 = da(dm(u3r, a1i), dm(u3i, a1r));
        a0r = r0; a0i = i0; a1r = r1; a1i = i1;
    } else if (CLS == kPairAnti) {
        const double u1r = op.u_re[1], u1i = op.u_im[1], u2r = op.u_re[2], u2i = op.u_im[2];
        const double r0 = ds(dm(u1r, a1r), dm(u1i, a1i));
        const double i0 = da(dm(u1r, a1i), dm(u1i, a1r));
        const double r1 = ds(dm(u2r, a0r), dm(u2i, a0i));
        const double i1 = da(dm(u2r, a0i), dm(u2i, a0r));
        a0r = r0; a0i = i0; a1r = r1; a1i = i1;
    } else if (CLS == kPairReal) {
        const double u0 = op.u_re[0], u1 = op.u_re[1], u2 = op.u_re[2], u3 = op.u_re[3];
        const double r0 = da(dm(u0, a0r), dm(u1, a1r));
        const double i0 = da(dm(u0, a0i), dm(u1, a1i));
        const double r1 = da(dm(u2, a0r), dm(u3, a1r));
        const double i1 = da(dm(u2, a0i), dm(u3, a1i));
        a0r = r0; a0i = i0; a1r = r1; a1i = i1;
    } else {
        const double u00r = op.u_re[0], u00i = op.u_im[0], u01r = op.u_re[1], u01i = op.u_im[1];
        const double u10r = op.u_re[2], u10i = op.u_im[2], u11r = op.u_re[3], u11i = op.u_im[3];
        // u00r * a0r - u00i * a0i + u01r * a1r - u01i * a1i, left to right
        const double r0 = ds(da(ds(dm(u00r, a0r), dm(u00i, a0i)), dm(u01r, a1r)), dm(u01i, a1i));
        const double i0 = da(da(da(dm(u00r, a0i), dm(u00i, a0r)), dm(u01r, a1i)), dm(u01i, a1r));
        const double r1 = ds(da(ds(dm(u10r, a0r), dm(u10i, a0i)), dm(u11r, a1r)), dm(u11i, a1i));
        const double i1 = da(da(da(dm(u10r, a0i), dm(u10i, a0r)), dm(u11r, a1i)), dm(u11i, a1r));
        a0r = r0; a0i = i0; a1r = r1; a1i = i1;
    }
}

// The same update on shared-memory elements i0, i1.
template <int CLS>
__device__ __forceinline__ void pair_update(const SvLocalOp& op, double* __restrict__ sre, double* __restrict__ sim,
                                            uint32_t i0, uint32_t i1) {
    double a0r = sre[i0], a0i = sim[i0], a1r = sre[i1], a1i = sim[i1];
    pair_math<CLS>(op, a0r, a0i, a1r, a1i);
    if (CLS != kPairDiag1) {
        sre[i0] = a0r;
        sim[i0] = a0i;
    }
    sre[i1] = a1r;
    sim[i1] = a1i;
}

// Visit exactly the pairs the reference updates: target bit clear, every local
// control bit set (single control: both bits inserted, lower position first).
template <int CLS>
__device__ __forceinline__ void apply_pair(const SvLocalOp& op, double* sre, double* sim, int S) {
    const int lt = op.lt;
    if (op.lc < 0) {
        const int pairs = S >> 1;
        for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
            const uint32_t i0 = insert_bit(static_cast<uint32_t>(i), lt, 0u);
            pair_update<CLS>(op, sre, sim, i0, i0 | (1u << lt));
        }
    } else {
        const int lc = op.lc;
        const int plo = lt < lc ? lt : lc, phi = lt < lc ? lc : lt;
        const uint32_t vlo = lt < lc ? 0u : 1u, vhi = lt < lc ? 1u : 0u;
        const int quads = S >> 2;
        for (int i = threadIdx.x; i < quads; i += blockDim.x) {
            const uint32_t i0 = insert_bit(insert_bit(static_cast<uint32_t>(i), plo, vlo), phi, vhi);
            pair_update<CLS>(op, sre, sim, i0, i0 | (1u << lt));
        }
    }
}

constexpr int kSvMaxPer = (1 << kSvMaxSlabBits) / kSvThreads;

// apply_function on a block inside the slab (fsv_backend.cpp:109-129): for every
// setting of the other local bits, out[row] = sum_k m[row][k] * in[k], k ascending.
__device__ __forceinline__ void apply_function_local(const SvLocalOp& op, double* sre, double* sim, int S) {
    const int blk = 1 << op.k;
    const int ls = op.lt;
    const uint32_t bmask = static_cast<uint32_t>(blk - 1) << ls;
    double outr[kSvMaxPer], outi[kSvMaxPer];
#pragma unroll
    for (int q = 0; q < kSvMaxPer; ++q) {
        const int j = threadIdx.x + q * kSvThreads;
        if (j < S) {
            const int row = (j >> ls) & (blk - 1);
            const uint32_t g = static_cast<uint32_t>(j) & ~bmask;
            double sr = 0.0, si = 0.0;
            for (int z = __ldg(op.tab.rp + row), ze = __ldg(op.tab.rp + row + 1); z < ze; ++z) {
                const uint32_t idx = g | (static_cast<uint32_t>(__ldg(op.tab.ci + z)) << ls);
                const double xr = sre[idx], xi = sim[idx];
                const double m_r = __ldg(op.tab.vr + z), m_i = __ldg(op.tab.vi + z);
                sr = da(sr, ds(dm(m_r, xr), dm(m_i, xi)));
                si = da(si, da(dm(m_r, xi), dm(m_i, xr)));
            }
            outr[q] = sr;
            outi[q] = si;
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kSvMaxPer; ++q) {
        const int j = threadIdx.x + q * kSvThreads;
        if (j < S) {
            sre[j] = outr[q];
            sim[j] = outi[q];
        }
    }
}

__global__ void __launch_bounds__(kSvThreads) sv_batch_kernel(double* __restrict__ re, double* __restrict__ im,
                                                            const SvLocalOp* __restrict__ ops,
                                                            const __grid_constant__ SvBatch b) {
    extern __shared__ double sv_smem[];
    const int S = 1 << b.L;
    double* sre = sv_smem;
    double* sim = sv_smem + S;
    for (int64_t slab = blockIdx.x; slab < b.slabs; slab += gridDim.x) {
        // base: the slab number deposited into the outer bits
        uint64_t base = 0, om = b.outer_mask;
        for (uint64_t sb = static_cast<uint64_t>(slab); om != 0; sb >>= 1) {
            const uint64_t low = om & (~om + 1);
            if (sb & 1u) base |= low;
            om ^= low;
        }
        // stage: consecutive local pairs are consecutive flat pairs (r >= 1)
        for (int j = 2 * threadIdx.x; j < S; j += 2 * blockDim.x) {
            const uint64_t f = base | local_to_flat(static_cast<uint32_t>(j), b);
            const double2 vr = *reinterpret_cast<const double2*>(re + f);
            const double2 vi = *reinterpret_cast<const double2*>(im + f);
            *reinterpret_cast<double2*>(sre + j) = vr;
            *reinterpret_cast<double2*>(sim + j) = vi;
        }
        __syncthreads();
        for (int o = 0; o < b.op_count; ++o) {
            const SvLocalOp& op = ops[b.op_begin + o];
            if ((base & op.ocmask) != op.ocmask) continue;  // a control outside the slab is clear
            if (op.kind == kSvFunction) {
                apply_function_local(op, sre, sim, S);
            } else {
                switch (op.cls) {
                case kPairSwap: apply_pair<kPairSwap>(op, sre, sim, S); break;
                case kPairDiag1: apply_pair<kPairDiag1>(op, sre, sim, S); break;
                case kPairDiag: apply_pair<kPairDiag>(op, sre, sim, S); break;
                case kPairAnti: apply_pair<kPairAnti>(op, sre, sim, S); break;
                case kPairReal: apply_pair<kPairReal>(op, sre, sim, S); break;
                default: apply_pair<kPairGeneral>(op, sre, sim, S); break;
                }
            }
            __syncthreads();
        }
        for (int j = 2 * threadIdx.x; j < S; j += 2 * blockDim.x) {
            const uint64_t f = base | local_to_flat(static_cast<uint32_t>(j), b);
            *reinterpret_cast<double2*>(re + f) = *reinterpret_cast<const double2*>(sre + j);
            *reinterpret_cast<double2*>(im + f) = *reinterpret_cast<const double2*>(sim + j);
        }
        __syncthreads();
    }
}

// ---- register batches ----------------------------------------------------
// Pair (e, e | 1 << TB) of a group held in registers; a control inside the
// batch's targets is the e-space mask emask (e is a compile-time index, so the
// predicate never forces a register array into local memory).
// CB >= 0: the control is target bit CB of the batch (pairs with that bit clear
// are skipped at compile time); CB == -1: no control inside the targets;
// CB == -2: control mask op.emask tested at run time (e is a compile-time index,
// so no predicate ever forces a register array into local memory).
template <int K, int CLS, int CB, int TB>
__device__ __forceinline__ void reg_apply(const SvRegOp& op, double (&vr)[1 << K], double (&vi)[1 << K]) {
    if constexpr (TB < K && CB < K && CB != TB) {
#pragma unroll
        for (int e = 0; e < (1 << K); ++e) {
            if (e & (1 << TB)) continue;
            if constexpr (CB >= 0) {
                if (!(e & (1 << CB))) continue;
            }
            if constexpr (CB == -2) {
                if ((static_cast<uint32_t>(e) & op.emask) != op.emask) continue;
            }
            pair_math<CLS>(op, vr[e], vi[e], vr[e | (1 << TB)], vi[e | (1 << TB)]);
        }
    }
}

#define QSB_REG_CASES(CAT, CLS, CB)                                      \
    case (CAT) * kSvRegMaxK + 0: reg_apply<K, CLS, CB, 0>(op, vr, vi); break; \
    case (CAT) * kSvRegMaxK + 1: reg_apply<K, CLS, CB, 1>(op, vr, vi); break; \
    case (CAT) * kSvRegMaxK + 2: reg_apply<K, CLS, CB, 2>(op, vr, vi); break; \
    case (CAT) * kSvRegMaxK + 3: reg_apply<K, CLS, CB, 3>(op, vr, vi); break; \
    case (CAT) * kSvRegMaxK + 4: reg_apply<K, CLS, CB, 4>(op, vr, vi); break;

// One indirect branch per operation: op.code = category * kSvRegMaxK + target
// index (categories: sv_reg_code in qsb_sv.hpp).
template <int K>
__device__ __forceinline__ void reg_dispatch(const SvRegOp& op, double (&vr)[1 << K], double (&vi)[1 << K]) {
    switch (op.code) {
        QSB_REG_CASES(0, kPairGeneral, -1)
        QSB_REG_CASES(1, kPairReal, -1)
        QSB_REG_CASES(2, kPairDiag, -1)
        QSB_REG_CASES(3, kPairDiag1, -1)
        QSB_REG_CASES(4, kPairAnti, -1)
        QSB_REG_CASES(5, kPairSwap, -1)
        QSB_REG_CASES(6, kPairGeneral, -2)
        QSB_REG_CASES(7, kPairReal, -2)
        QSB_REG_CASES(8, kPairDiag, -2)
        QSB_REG_CASES(9, kPairDiag1, -2)
        QSB_REG_CASES(10, kPairAnti, -2)
        QSB_REG_CASES(11, kPairSwap, -2)
        QSB_REG_CASES(12, kPairDiag1, 0)
        QSB_REG_CASES(13, kPairDiag1, 1)
        QSB_REG_CASES(14, kPairDiag1, 2)
        QSB_REG_CASES(15, kPairDiag1, 3)
        QSB_REG_CASES(16, kPairDiag1, 4)
        QSB_REG_CASES(17, kPairSwap, 0)
        QSB_REG_CASES(18, kPairSwap, 1)
        QSB_REG_CASES(19, kPairSwap, 2)
        QSB_REG_CASES(20, kPairSwap, 3)
        QSB_REG_CASES(21, kPairSwap, 4)
    default: break;
    }
}
#undef QSB_REG_CASES

__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

// Each thread owns one group per iteration: the 2^K elements differing only in
// the batch's K target bits. The next group is prefetched into this thread's
// shared-memory slots with cp.async while the current one is updated in
// registers and stored, so HBM traffic overlaps the FP64 work; slots are
// [element][plane][thread] (consecutive threads, consecutive 8-byte words).
template <int K>
__global__ void __launch_bounds__(kSvRegThreads, 3) sv_reg_kernel(double* __restrict__ re, double* __restrict__ im,
                                                             const __grid_constant__ SvRegBatch b) {
    constexpr int E = 1 << K;
    extern __shared__ double sv_pref[];
    // flat indices fit 32 bits: m <= 32 (host-checked)
    uint32_t tb[K];
#pragma unroll
    for (int i = 0; i < K; ++i) tb[i] = 1u << b.t[i];
    // element 0 of group g: g with a zero inserted at every target bit
    // (ascending positions, so each insert is in final coordinates)
    auto base_of = [&](int64_t g) {
        uint32_t f = static_cast<uint32_t>(g);
#pragma unroll
        for (int i = 0; i < K; ++i) f = ((f & ~(tb[i] - 1u)) << 1) | (f & (tb[i] - 1u));
        return f;
    };
    auto offset = [&](uint32_t f, int e) {
        uint32_t off = f;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (e & (1 << i)) off |= tb[i];
        return off;
    };
    const uint32_t slot = static_cast<uint32_t>(__cvta_generic_to_shared(sv_pref)) + threadIdx.x * 8;
    constexpr uint32_t SLOT_STRIDE = kSvRegThreads * 8;
    auto prefetch = [&](uint32_t f) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t off = offset(f, e);
            cp_async8(slot + (2 * e) * SLOT_STRIDE, re + off);
            cp_async8(slot + (2 * e + 1) * SLOT_STRIDE, im + off);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (g < b.groups) prefetch(base_of(g));
    for (; g < b.groups; g += stride) {
        const uint32_t f = base_of(g);
        double vr[E], vi[E];
        asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
        for (int e = 0; e < E; ++e) {
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(vr[e]) : "r"(slot + (2 * e) * SLOT_STRIDE) : "memory");
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(vi[e]) : "r"(slot + (2 * e + 1) * SLOT_STRIDE) : "memory");
        }
        if (g + stride < b.groups) prefetch(base_of(g + stride));
#pragma unroll 1
        for (int o = 0; o < b.op_count; ++o) {
            const SvRegOp& op = b.ops[o];
            const uint32_t oc = op.ocmask;
            if ((f & oc) != oc) continue;  // a control outside the targets is clear
            reg_dispatch<K>(op, vr, vi);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const uint32_t off = offset(f, e);
            __stcs(re + off, vr[e]);
            __stcs(im + off, vi[e]);
        }
    }
}

// out[o][row][i] = sum_kk m[row][kk] * in[o][kk][i] over the nonzeros of row
// `row` in ascending kk (bit-exact with the dense sequential sum); one thread
// per output, consecutive threads on consecutive inner indices i (coalesced).
__global__ void __launch_bounds__(kSvThreads) sv_function_kernel(const double* __restrict__ in_re,
                                                               const double* __restrict__ in_im,
                                                               double* __restrict__ out_re,
                                                               double* __restrict__ out_im, const SvTable tab,
                                                               int k, int s, int m) {
    const int64_t inner = int64_t{1} << s;
    const int64_t blk = int64_t{1} << k;
    const int64_t total = int64_t{1} << m;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e & (inner - 1);
        const int64_t row = (e >> s) & (blk - 1);
        const int64_t base = e - (row << s);  // element with the block bits cleared
        double sr = 0.0, si = 0.0;
        for (int z = __ldg(tab.rp + row), ze = __ldg(tab.rp + row + 1); z < ze; ++z) {
            const int64_t x = base + (static_cast<int64_t>(__ldg(tab.ci + z)) << s);
            const double xr = in_re[x], xi = in_im[x];
            const double m_r = __ldg(tab.vr + z), m_i = __ldg(tab.vi + z);
            sr = da(sr, ds(dm(m_r, xr), dm(m_i, xi)));
            si = da(si, da(dm(m_r, xi), dm(m_i, xr)));
        }
        out_re[e] = sr;
        out_im[e] = si;
        (void)i;
    }
}

__global__ void __launch_bounds__(kSvThreads) sv_init_identity_kernel(double* __restrict__ re,
                                                                    double* __restrict__ im, int64_t R,
                                                                    int64_t W, int64_t col_begin) {
    const int64_t pairs = R * W / 2;
    for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < pairs;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e0 = 2 * p, e1 = e0 + 1;
        const double v0 = (e0 / W == col_begin + e0 % W) ? 1.0 : 0.0;
        const double v1 = (e1 / W == col_begin + e1 % W) ? 1.0 : 0.0;
        reinterpret_cast<double2*>(re)[p] = make_double2(v0, v1);
        reinterpret_cast<double2*>(im)[p] = make_double2(0.0, 0.0);
    }
}

int grid_for(int64_t work, int per_sm) {
    const int64_t cap = static_cast<int64_t>(148) * per_sm;
    return static_cast<int>(work < 1 ? 1 : (work < cap ? work : cap));
}

}  // namespace detail

using namespace detail;

int sv_configure() {
    int e = static_cast<int>(cudaFuncSetAttribute(sv_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  2 * (1 << kSvMaxSlabBits) * static_cast<int>(sizeof(double))));
    return e;
}

int sv_launch_batch(double* re, double* im, const SvLocalOp* ops, const SvBatch& b, void* stream) {
    const int smem = 2 * (1 << b.L) * static_cast<int>(sizeof(double));
    int per_sm = (200 * 1024) / (smem < 4096 ? 4096 : smem);
    if (per_sm > 8) per_sm = 8;
    sv_batch_kernel<<<grid_for(b.slabs, per_sm), kSvThreads, smem, static_cast<cudaStream_t>(stream)>>>(re, im, ops,
                                                                                                     b);
    return static_cast<int>(cudaGetLastError());
}

template <int K>
static int launch_reg_t(double* re, double* im, const SvRegBatch& b, cudaStream_t st) {
    const int64_t blocks = (b.groups + kSvRegThreads - 1) / kSvRegThreads;
    const int smem = 2 * (1 << K) * kSvRegThreads * static_cast<int>(sizeof(double));
    sv_reg_kernel<K><<<grid_for(blocks, 3), kSvRegThreads, smem, st>>>(re, im, b);
    return static_cast<int>(cudaGetLastError());
}

int sv_launch_reg(double* re, double* im, const SvRegBatch& b, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (b.K) {
    case 1: return launch_reg_t<1>(re, im, b, st);
    case 2: return launch_reg_t<2>(re, im, b, st);
    case 3: return launch_reg_t<3>(re, im, b, st);
    default: return launch_reg_t<4>(re, im, b, st);  // K <= kSvRegDefaultK (host-capped)
    }
}

int sv_launch_function(const double* in_re, const double* in_im, double* out_re, double* out_im,
                       const SvTable& tab, int k, int s, int m, void* stream) {
    const int64_t total = int64_t{1} << m;
    sv_function_kernel<<<grid_for((total + kSvThreads - 1) / kSvThreads, 8), kSvThreads, 0,
                         static_cast<cudaStream_t>(stream)>>>(in_re, in_im, out_re, out_im, tab, k, s, m);
    return static_cast<int>(cudaGetLastError());
}

int sv_launch_init_identity(double* re, double* im, int64_t R, int64_t W, int64_t col_begin, void* stream) {
    const int64_t pairs = R * W / 2;
    sv_init_identity_kernel<<<grid_for((pairs + kSvThreads - 1) / kSvThreads, 16), kSvThreads, 0,
                              static_cast<cudaStream_t>(stream)>>>(re, im, R, W, col_begin);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace qsb
