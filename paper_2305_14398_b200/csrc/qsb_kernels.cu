// qsb_kernels.cu — sm_100a kernels of the unitary-simulation hot path.
//
//   K1 expand_kernel        materialises rows of one layer operator (HBM-bound
//                           coalesced 16-byte stores); used for the first
//                           operator of the chain (V = L_last[rows, :]).
//   K2 zgemm_gen_kernel     V' = V * L: complex FP64 GEMM on the DMMA tensor pipe
//                           (mma.sync m8n8k4 f64), A = V staged by TMA
//                           (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier
//                           pipeline), B = L generated straight into shared
//                           memory from the layer descriptor — the operator is
//                           never read from HBM.
//   K2s small_circuit_kernel whole circuit in one CTA for 2^n <= 32.
//   K3 matvec_kernel        psi = V * psi0, one warp per row, shuffle reduce.
//   K4 probs_kernel         p_i = re^2 + im^2 (separately rounded, bit-exact with
//                           state.cpp:58-65) + deterministic two-pass norm.
//
// Reference loops replaced (paths relative to /root/reference/proj):
//   kronecker_fold / kronecker      core/src/unitary_backend.cpp:119-125, core/src/linalg.cpp:109-129
//   controlled_unitary              core/src/gates.cpp:79-110
//   matmul_rows (accumulate GEMM)   core/src/linalg.cpp:46-87, unitary_backend.cpp:211
//   matvec                          core/src/linalg.cpp:89-107, unitary_backend.cpp:213-214
//   probabilities / norm_squared    core/src/state.cpp:49-65
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "qsb_internal.hpp"

namespace qsb {

// ----------------------------------------------------------------------------
// Operator-entry generator (shared by K1, K2, K2s)
// ----------------------------------------------------------------------------

// Complex product with every multiply and add rounded separately, as the
// reference's `ar * br - ai * bi`, `ar * bi + ai * br` (linalg.cpp:122-123)
// on x86-64 without FMA contraction.
__device__ __forceinline__ void cmul_rn(double ar, double ai, double br, double bi, double& cr,
                                        double& ci) {
    cr = __dsub_rn(__dmul_rn(ar, br), __dmul_rn(ai, bi));
    ci = __dadd_rn(__dmul_rn(ar, bi), __dmul_rn(ai, br));
}

// Entry (rb, cb) of one non-identity block, rb/cb = the block's bits of r/c.
__device__ __forceinline__ void block_entry(const BlockDesc& b, uint32_t r, uint32_t c, double& er,
                                            double& ei) {
    const uint32_t rb = (r >> b.shift) & b.mask;
    const uint32_t cb = (c >> b.shift) & b.mask;
    if (b.kind == kBlockGate) {
        const int e = static_cast<int>(rb * 2 + cb);
        er = b.u_re[e];
        ei = b.u_im[e];
    } else if (b.kind == kBlockControlled) {
        // controlled_unitary (gates.cpp:94-107): a column whose control bit is
        // clear is the identity column; otherwise u acts on the target bit.
        if ((cb & b.cmask) == 0) {
            er = (rb == cb) ? 1.0 : 0.0;
            ei = 0.0;
        } else if (((rb ^ cb) & ~b.tmask) != 0) {
            er = 0.0;
            ei = 0.0;
        } else {
            const int e = ((rb & b.tmask) ? 2 : 0) + ((cb & b.tmask) ? 1 : 0);
            er = b.u_re[e];
            ei = b.u_im[e];
        }
    } else if (b.kind == kBlockMonomial) {
        const bool hit = __ldg(b.t_col + rb) == static_cast<int32_t>(cb);
        er = hit ? __ldg(b.t_re + rb) : 0.0;
        ei = hit ? __ldg(b.t_im + rb) : 0.0;
    } else {
        const size_t e = (static_cast<size_t>(rb) << b.span) + cb;
        er = __ldg(b.t_re + e);
        ei = __ldg(b.t_im + e);
    }
}

// Entry (r, c) of the layer operator.
template <class Desc>  // LayerDesc, or the small path's SmallLayerDesc
__device__ __forceinline__ void layer_entry(const Desc& d, uint32_t r, uint32_t c, double& vr,
                                            double& vi) {
    // zmask = identity bits + controlled blocks' non-target bits: the entry is an exact
    // zero unless r and c agree there (the fold would give a signed zero; == ignores the sign)
    if ((r ^ c) & d.zmask) {
        vr = 0.0;
        vi = 0.0;
        return;
    }
    if (d.nblocks == 0) {
        vr = 1.0;
        vi = 0.0;
        return;
    }
    double ar, ai;
    block_entry(d.blocks[0], r, c, ar, ai);
    for (int b = 1; b < d.nblocks; ++b) {
        if (ar == 0.0 && ai == 0.0) break;  // the fold stays (signed) zero
        double er, ei, tr, ti;
        block_entry(d.blocks[b], r, c, er, ei);
        cmul_rn(ar, ai, er, ei, tr, ti);
        ar = tr;
        ai = ti;
    }
    vr = ar;
    vi = ai;
}

// Column of the single nonzero of row r of a monomial layer (or -1 if the row
// is zero): each block maps the row's bits to the column's bits.
__device__ __forceinline__ int64_t mono_col(const LayerDesc& d, uint32_t r) {
    uint32_t c = r;
    for (int b = 0; b < d.nblocks; ++b) {
        const BlockDesc& B = d.blocks[b];
        const uint32_t rb = (r >> B.shift) & B.mask;
        uint32_t cb = rb;
        if (B.mono == 1) {
            if (B.kind == kBlockGate)
                cb = rb ^ 1u;
            else if (rb & B.cmask)
                cb = rb ^ B.tmask;  // controlled_unitary (gates.cpp:94-107) with an anti-diagonal u
        } else if (B.mono == 2) {
            const int32_t t = __ldg(B.t_col + rb);
            if (t < 0) return -1;
            cb = static_cast<uint32_t>(t);
        }
        c = (c & ~(B.mask << B.shift)) | (cb << B.shift);
    }
    return static_cast<int64_t>(c);
}

// Continue the left fold from block `b` with the running value (ar, ai).
// Real layers multiply real parts only: (a, 0) * (e, 0) = (a*e - 0*0, a*0 + 0*e)
// = (a*e, +-0), so the real product is bit-identical to the complex one.
__device__ __forceinline__ void fold_from(const LayerDesc& d, int b, uint32_t r, uint32_t c, double& ar,
                                          double& ai) {
    if (d.real) {
        for (; b < d.nblocks; ++b) {
            if (ar == 0.0) break;
            double er, ei;
            block_entry(d.blocks[b], r, c, er, ei);
            ar = __dmul_rn(ar, er);
        }
        ai = 0.0;
        return;
    }
    for (; b < d.nblocks; ++b) {
        if (ar == 0.0 && ai == 0.0) break;
        double er, ei, tr, ti;
        block_entry(d.blocks[b], r, c, er, ei);
        cmul_rn(ar, ai, er, ei, tr, ti);
        ar = tr;
        ai = ti;
    }
}

// Tile-level view of one layer for a BK x BN operator tile whose row and column
// indices vary only in their low LOWBITS bits: blocks entirely above LOWBITS are
// constant over the tile and — being the most significant — form a prefix of
// the fold, so their product P is computed once per tile; identity bits above
// LOWBITS decide whether the whole tile is zero. Per element only the
// remaining (low) blocks are folded, continuing from P: the same sequence of
// roundings as the full fold, hence still bit-exact.
struct TilePrefix {
    double pr, pi;  // prefix product (valid if nconst > 0)
    int nconst;     // blocks in the prefix
    bool zero;      // whole tile is zero
};

template <int LOWBITS>
__device__ __forceinline__ TilePrefix tile_prefix(const LayerDesc& d, uint32_t r0, uint32_t c0) {
    constexpr uint32_t LOW = (1u << LOWBITS) - 1u;
    TilePrefix tp{1.0, 0.0, 0, ((r0 ^ c0) & d.zmask & ~LOW) != 0};
    if (tp.zero) return tp;
    int b = 0;
    while (b < d.nblocks && d.blocks[b].shift >= LOWBITS) ++b;
    tp.nconst = b;
    if (b > 0) {
        block_entry(d.blocks[0], r0, c0, tp.pr, tp.pi);
        double pr = tp.pr, pi = tp.pi;
        // fold the rest of the prefix
        for (int k = 1; k < b; ++k) {
            if (pr == 0.0 && pi == 0.0) break;
            double er, ei, tr, ti;
            block_entry(d.blocks[k], r0, c0, er, ei);
            if (d.real) {
                pr = __dmul_rn(pr, er);
                pi = 0.0;
            } else {
                cmul_rn(pr, pi, er, ei, tr, ti);
                pr = tr;
                pi = ti;
            }
        }
        tp.pr = pr;
        tp.pi = pi;
        tp.zero = (pr == 0.0 && pi == 0.0);
    }
    return tp;
}

template <int LOWBITS>
__device__ __forceinline__ void tile_entry(const LayerDesc& d, const TilePrefix& tp, uint32_t r, uint32_t c,
                                           double& vr, double& vi) {
    constexpr uint32_t LOW = (1u << LOWBITS) - 1u;
    if ((r ^ c) & d.idmask & LOW) {
        vr = 0.0;
        vi = 0.0;
        return;
    }
    if (tp.nconst > 0) {
        vr = tp.pr;
        vi = tp.pi;
        fold_from(d, tp.nconst, r, c, vr, vi);
    } else if (d.nblocks == 0) {
        vr = 1.0;
        vi = 0.0;
    } else {
        block_entry(d.blocks[0], r, c, vr, vi);
        fold_from(d, 1, r, c, vr, vi);
    }
}

// Producer-side batch generator: EB elements per thread, blocks outermost so
// each block's parameters are loaded once (uniformly) per batch and entries
// are selected in registers — no divergent constant-bank loads. The running
// value starts at the tile prefix P (or 1 + 0i when no block is constant:
// 1*e = e exactly, up to the sign of zero), then multiplies every low block in
// fold order with separately rounded products: bit-exact with kronecker_fold.
__device__ __forceinline__ double sel4(int e, double a0, double a1, double a2, double a3) {
    const double lo = (e & 1) ? a1 : a0;
    const double hi = (e & 1) ? a3 : a2;
    return (e & 2) ? hi : lo;
}

template <int EB, int LOWBITS>
__device__ __forceinline__ void gen_batch(const LayerDesc& d, const TilePrefix& tp, const uint32_t (&r)[EB],
                                          const uint32_t (&c)[EB], double (&vr)[EB], double (&vi)[EB]) {
    constexpr uint32_t LOW = (1u << LOWBITS) - 1u;
    const bool real = d.real != 0;
#pragma unroll
    for (int k = 0; k < EB; ++k) {
        const bool nz = ((r[k] ^ c[k]) & d.zmask & LOW) == 0;
        vr[k] = nz ? (tp.nconst > 0 ? tp.pr : 1.0) : 0.0;
        vi[k] = nz ? (tp.nconst > 0 ? tp.pi : 0.0) : 0.0;
    }
    for (int b = tp.nconst; b < d.nblocks; ++b) {
        const BlockDesc& B = d.blocks[b];
        const int kind = B.kind, shift = B.shift;
        const uint32_t mask = B.mask;
        if (kind == kBlockTable || kind == kBlockMonomial) {
#pragma unroll
            for (int k = 0; k < EB; ++k) {
                const uint32_t rb = (r[k] >> shift) & mask, cb = (c[k] >> shift) & mask;
                double er, ei;
                if (kind == kBlockMonomial) {
                    const bool hit = __ldg(B.t_col + rb) == static_cast<int32_t>(cb);
                    er = hit ? __ldg(B.t_re + rb) : 0.0;
                    ei = hit ? __ldg(B.t_im + rb) : 0.0;
                } else {
                    const size_t e = (static_cast<size_t>(rb) << B.span) + cb;
                    er = __ldg(B.t_re + e);
                    ei = __ldg(B.t_im + e);
                }
                double tr, ti;
                if (real) {
                    vr[k] = __dmul_rn(vr[k], er);
                } else {
                    cmul_rn(vr[k], vi[k], er, ei, tr, ti);
                    vr[k] = tr;
                    vi[k] = ti;
                }
            }
            continue;
        }
        const double u0 = B.u_re[0], u1 = B.u_re[1], u2 = B.u_re[2], u3 = B.u_re[3];
        const double w0 = B.u_im[0], w1 = B.u_im[1], w2 = B.u_im[2], w3 = B.u_im[3];
        const uint32_t cm = B.cmask, tm = B.tmask;
        const bool controlled = kind == kBlockControlled;
#pragma unroll
        for (int k = 0; k < EB; ++k) {
            const uint32_t rb = (r[k] >> shift) & mask, cb = (c[k] >> shift) & mask;
            double er, ei;
            if (controlled) {
                // controlled_unitary (gates.cpp:94-107)
                const bool active = (cb & cm) != 0;
                const bool hit = ((rb ^ cb) & ~tm) == 0;
                const int e = ((rb & tm) ? 2 : 0) + ((cb & tm) ? 1 : 0);
                er = active ? (hit ? sel4(e, u0, u1, u2, u3) : 0.0) : (rb == cb ? 1.0 : 0.0);
                ei = active ? (hit ? sel4(e, w0, w1, w2, w3) : 0.0) : 0.0;
            } else {
                const int e = static_cast<int>(rb * 2 + cb);
                er = sel4(e, u0, u1, u2, u3);
                ei = sel4(e, w0, w1, w2, w3);
            }
            if (real) {
                vr[k] = __dmul_rn(vr[k], er);
            } else {
                double tr, ti;
                cmul_rn(vr[k], vi[k], er, ei, tr, ti);
                vr[k] = tr;
                vi[k] = ti;
            }
        }
    }
    if (real) {
#pragma unroll
        for (int k = 0; k < EB; ++k) vi[k] = 0.0;
    }
}

// ----------------------------------------------------------------------------
// K1: expansion
// ----------------------------------------------------------------------------

// TRANSPOSE: rows [row_begin, row_begin + M) of L^T, i.e. out[i][j] = L(j, row_begin + i)
// (column blocks: V starts as the first layer's columns).
template <bool TRANSPOSE>
__global__ void __launch_bounds__(256) expand_kernel(const __grid_constant__ LayerDesc d,
                                                     uint32_t row_begin, int M, int N,
                                                     double* __restrict__ out, int planes) {
    const size_t plane = static_cast<size_t>(M) * N;
    const size_t pairs = plane / 2;
    const uint32_t half_n = static_cast<uint32_t>(N) / 2;
    for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < pairs;
         p += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t row = static_cast<uint32_t>(p / half_n);
        const uint32_t col = static_cast<uint32_t>(p % half_n) * 2;
        double r0, i0, r1, i1;
        if (TRANSPOSE) {
            layer_entry(d, col, row_begin + row, r0, i0);
            layer_entry(d, col + 1, row_begin + row, r1, i1);
        } else {
            layer_entry(d, row_begin + row, col, r0, i0);
            layer_entry(d, row_begin + row, col + 1, r1, i1);
        }
        reinterpret_cast<double2*>(out)[p] = make_double2(r0, r1);
        reinterpret_cast<double2*>(out + plane)[p] = make_double2(i0, i1);
        if (planes == 3)
            reinterpret_cast<double2*>(out + 2 * plane)[p] = make_double2(__dadd_rn(r0, i0), __dadd_rn(r1, i1));
    }
}

int launch_expand(const LayerDesc& layer, uint32_t row_begin, int M, int N, double* out, int planes,
                  void* stream) {
    const size_t pairs = static_cast<size_t>(M) * N / 2;
    int blocks = static_cast<int>((pairs + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    expand_kernel<false><<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(layer, row_begin, M, N, out, planes);
    return static_cast<int>(cudaGetLastError());
}

int launch_expand_cols(const LayerDesc& layer, uint32_t col_begin, int M, int N, double* out, int planes,
                       void* stream) {
    const size_t pairs = static_cast<size_t>(M) * N / 2;
    int blocks = static_cast<int>((pairs + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    expand_kernel<true><<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(layer, col_begin, M, N, out, planes);
    return static_cast<int>(cudaGetLastError());
}

// ----------------------------------------------------------------------------
// K2: generated-operand complex GEMM on DMMA
// ----------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

__device__ __forceinline__ double2 lds128(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts128(uint32_t addr, double x, double y) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(x), "d"(y) : "memory");
}

// D = A(8x4) * B(4x8) + C on the FP64 tensor pipe (SASS DMMA.8x8x4).
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ double neg(double x) {
    return __longlong_as_double(__double_as_longlong(x) ^ static_cast<long long>(0x8000000000000000ULL));
}

template <int BM, int BN>
struct GemmCfg {
    static constexpr int BK = 16;  // one 128-byte swizzle line of doubles
    static constexpr int WM = BM / 32;
    static constexpr int WN = BN / 32;
    static constexpr int THREADS = 32 * WM * WN;
    static constexpr int STAGES = 4;
    static constexpr int A_STAGE = 2 * BM * BK * 8;  // re + im planes
    static constexpr int B_BUF = 2 * BN * BK * 8;
    static constexpr int PAIRS = 8 * BN / THREADS;  // generated (k, k+1) pairs per thread
    static constexpr int SMEM = 1024 + STAGES * A_STAGE + 2 * B_BUF + 64;
};

// Shared-memory tiles are [plane][rows][16 doubles] with the 128-byte TMA
// swizzle: the 16-byte chunk c of line l sits at chunk c ^ (l & 7). Lane (g, t)
// of an m8n8k4 fragment reads the chunks 2t and 2t+1 of line g, i.e. k indices
// {4t, 4t+1} and {4t+2, 4t+3}; the four k-steps of a tile therefore use the
// k-permutation k(t, s) = 4t + s, identically for A and B, which keeps every
// 128-bit fragment load bank-conflict-free.
template <int BM, int BN>
__global__ void __launch_bounds__(GemmCfg<BM, BN>::THREADS, 1)
    zgemm_gen_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ LayerDesc layer,
                     double* __restrict__ out, int M, int N) {
    using C = GemmCfg<BM, BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sA = smem_u32(smem);
    const uint32_t sB = sA + C::STAGES * C::A_STAGE;
    const uint32_t sBar = sB + 2 * C::B_BUF;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int g = lane >> 2;
    const int t = lane & 3;
    const int wm = warp / C::WN;
    const int wn = warp % C::WN;
    const int m0 = blockIdx.y * BM;
    const int n0 = blockIdx.x * BN;
    const int KT = N / C::BK;

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) mbar_init(sBar + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    auto issue_a = [&](int kt) {
        const int s = kt % C::STAGES;
        mbar_expect_tx(sBar + 8 * s, C::A_STAGE);
        tma_load_3d(sA + s * C::A_STAGE, &tmA, sBar + 8 * s, kt * C::BK, m0, 0);
    };

    // Generate the BK x BN tile of L for k-tile kt into B buffer `buf`.
    auto generate_b = [&](int kt, int buf) {
        const uint32_t base = sB + buf * C::B_BUF;
#pragma unroll
        for (int q = 0; q < C::PAIRS; ++q) {
            const int idx = tid + q * C::THREADS;
            const int n = idx % BN;
            const int p = idx / BN;  // chunk: k = 2p, 2p + 1
            const uint32_t r0 = static_cast<uint32_t>(kt * C::BK + 2 * p);
            const uint32_t col = static_cast<uint32_t>(n0 + n);
            double a_r, a_i, b_r, b_i;
            layer_entry(layer, r0, col, a_r, a_i);
            layer_entry(layer, r0 + 1, col, b_r, b_i);
            const uint32_t off = n * 128 + ((p ^ (n & 7)) << 4);
            sts128(base + off, a_r, b_r);
            sts128(base + BN * 128 + off, a_i, b_i);
        }
    };

    // Warp tile 32x32 = 4 x 4 m8n8 tiles; real and imaginary accumulators.
    double cr[4][4][2], ci[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            cr[i][j][0] = cr[i][j][1] = 0.0;
            ci[i][j][0] = ci[i][j][1] = 0.0;
        }

    if (tid == 0) {
        for (int kt = 0; kt < C::STAGES - 1 && kt < KT; ++kt) issue_a(kt);
    }
    generate_b(0, 0);
    __syncthreads();

    for (int kt = 0; kt < KT; ++kt) {
        if (tid == 0 && kt + C::STAGES - 1 < KT) issue_a(kt + C::STAGES - 1);
        if (kt + 1 < KT) generate_b(kt + 1, (kt + 1) & 1);
        const int s = kt % C::STAGES;
        mbar_wait(sBar + 8 * s, (kt / C::STAGES) & 1);

        const uint32_t aRe = sA + s * C::A_STAGE;
        const uint32_t aIm = aRe + BM * 128;
        const uint32_t bRe = sB + (kt & 1) * C::B_BUF;
        const uint32_t bIm = bRe + BN * 128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t choff = static_cast<uint32_t>(((2 * t + h) ^ g) << 4);
            double2 ar[4], ai[4], br[4], bi[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t line = static_cast<uint32_t>(wm * 32 + i * 8 + g) * 128 + choff;
                ar[i] = lds128(aRe + line);
                ai[i] = lds128(aIm + line);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t line = static_cast<uint32_t>(wn * 32 + j * 8 + g) * 128 + choff;
                br[j] = lds128(bRe + line);
                bi[j] = lds128(bIm + line);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double a_r = e ? ar[i].y : ar[i].x;
                    const double a_i = e ? ai[i].y : ai[i].x;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double b_r = e ? br[j].y : br[j].x;
                        const double b_i = e ? bi[j].y : bi[j].x;
                        dmma(cr[i][j], a_r, b_r);
                        dmma(cr[i][j], a_i, neg(b_i));
                        dmma(ci[i][j], a_r, b_i);
                        dmma(ci[i][j], a_i, b_r);
                    }
                }
            }
        }
        __syncthreads();
    }

    // Epilogue: C fragment (g, 2t..2t+1) of every m8n8 tile, 16-byte stores.
    const size_t plane = static_cast<size_t>(M) * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + wm * 32 + i * 8 + g;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = n0 + wn * 32 + j * 8 + 2 * t;
            const size_t o = static_cast<size_t>(row) * N + col;
            *reinterpret_cast<double2*>(out + o) = make_double2(cr[i][j][0], cr[i][j][1]);
            *reinterpret_cast<double2*>(out + plane + o) = make_double2(ci[i][j][0], ci[i][j][1]);
        }
    }
}

// ----------------------------------------------------------------------------
// K2 v2: warp-specialised generated-operand complex GEMM (4M or 3M on DMMA)
// ----------------------------------------------------------------------------
//
// 12 warps: warpgroups 0-1 are consumers (8 warps of DMMA), warpgroup 2 is the
// producer (its first lane issues the TMA of the A tile, all 128 threads
// generate the B tile of the same stage). Stages are handed over with
// mbarriers (full: 1 TMA arrival + transaction bytes + 4 producer-warp
// arrivals; empty: 8 consumer-warp arrivals), so operator generation overlaps
// the DMMA work instead of stalling it at a block barrier. setmaxnreg moves
// registers from the producer warpgroup to the consumers.
//
// 4M: Cr += Ar*Br + Ai*(-Bi), Ci += Ar*Bi + Ai*Br (warp tile 32x32, CTA 128x64).
// 3M: T1 += Ar*Br, T2 += Ai*Bi, T3 += (Ar+Ai)*(Br+Bi); Cr = T1 - T2,
//     Ci = T3 - T1 - T2 (warp tile 32x16, CTA 64x64; the producer writes the
//     Br+Bi plane, consumers form Ar+Ai in registers).

// REAL: the layer operator has an exactly-zero imaginary plane (H, X, CNOT, SWAP,
// DJ oracles): V' = V L is two real GEMMs, Vr' = Vr Lr and Vi' = Vi Lr — the
// products with Li are exact zeros in every arithmetic — so B is one plane and
// the consumers issue 2 instead of 3 (3M) DMMAs per fragment pair. Same tile
// shape as 3M, so plans mix both variants freely.
template <bool THREE_M, bool SUMPLANE = false, bool REAL = false>
struct WsCfg {
    static constexpr int BK = 16;
    static constexpr int CONSUMER_WARPS = 8;
    static constexpr int PRODUCER_WARPS = 4;
    static constexpr int THREADS = 32 * (CONSUMER_WARPS + PRODUCER_WARPS);
    static constexpr int WT_N = THREE_M ? 16 : 32;   // warp tile columns
    static constexpr int NT = WT_N / 8;              // m8n8 tiles per warp row
    static constexpr int CWM = THREE_M ? 2 : 4;      // consumer warps along M
    static constexpr int CWN = CONSUMER_WARPS / CWM; // consumer warps along N
    static constexpr int BM = CWM * 32;
    static constexpr int BN = CWN * WT_N;
    static constexpr int B_PLANES = REAL ? 1 : (THREE_M ? 3 : 2);
    // SUMPLANE: V carries a third plane Vr+Vi written by the previous GEMM's
    // epilogue (or K1), so 3M consumers load it instead of adding in registers.
    static constexpr int A_PLANES = (THREE_M && SUMPLANE && !REAL) ? 3 : 2;
    static constexpr int A_TMA_BYTES = A_PLANES * BM * BK * 8;
    static constexpr int A_BYTES = A_TMA_BYTES;
    static constexpr int B_BYTES = B_PLANES * BN * BK * 8;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = (200 * 1024) / STAGE;
    static constexpr int SMEM = 1024 + STAGES * STAGE + 3 * STAGES * 8;
    static constexpr int PAIRS = 8 * BN / (32 * PRODUCER_WARPS);
    static constexpr int LOWBITS = 6;  // log2(BN) >= log2(BK): tile indices vary below this bit
    static_assert((1 << LOWBITS) == BN, "BN must be 2^LOWBITS");
    static constexpr int CONSUMER_REGS = 216;
    static constexpr int PRODUCER_REGS = 72;
};

// All threads of the thread-block cluster: release our shared-memory writes,
// acquire everyone else's.
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::
                     : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Producer side of the warp-specialised K2: operator tile B (rows ktg*BK.., columns
// n0..n0+BN) of `layer` generated into the stage at bBase by the 128 producer
// threads (ptid), in the consumers' swizzled layout. Zero tiles are cleared;
// monomial layers write zeros plus the hits; others fold block entries per element.
// `zero_stages` (per producer thread, bit s = stage s's B region still holds the zeros
// this thread wrote there): a zero tile in a stage that already holds zeros needs no
// stores — the clearing costs producer issue slots next to the DMMAs.
template <bool THREE_M, bool SUMPLANE, bool REAL>
__device__ __forceinline__ void ws_produce_b(const LayerDesc& layer, uint32_t bBase, int ptid, int ktg, int n0,
                                             int stage, uint32_t& zero_stages) {
    using C = WsCfg<THREE_M, SUMPLANE, REAL>;
    constexpr int BN = C::BN;
    const TilePrefix tp = tile_prefix<C::LOWBITS>(layer, static_cast<uint32_t>(ktg * C::BK),
                                                  static_cast<uint32_t>(n0));
    if (tp.zero) {
        // whole operator tile is zero: clear the B planes of this stage (unless they are)
        if (!((zero_stages >> stage) & 1u))
            for (int o = ptid * 16; o < C::B_BYTES; o += 16 * 32 * C::PRODUCER_WARPS) sts128(bBase + o, 0.0, 0.0);
        zero_stages |= 1u << stage;
        return;
    }
    zero_stages &= ~(1u << stage);
    if (layer.monomial) {
        // one nonzero per operator row: thread = (line n, half of the 8 k-chunks);
        // an entry is nonzero only where the row's column is this line's
        static_assert(32 * C::PRODUCER_WARPS == 2 * BN, "two producer threads per tile line");
        const int n = ptid & (BN - 1);
        const int half = ptid / BN;
        const uint32_t col = static_cast<uint32_t>(n0 + n);
        // FP64 arithmetic only for the (at most BK) hits: the FP64 pipe is the DMMA pipe.
        // Columns of this thread's 8 rows first (single-block layers — CNOT, CR, X,
        // DJ oracle — with independent loads), then the entries of the hits.
        int64_t cols[8];
        const uint32_t rbase = static_cast<uint32_t>(ktg * C::BK + 8 * half);
        if (layer.nblocks == 1) {
            const BlockDesc& B = layer.blocks[0];
            const uint32_t keep = ~(B.mask << B.shift);
            int32_t cb[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t rb = ((rbase + q) >> B.shift) & B.mask;
                cb[q] = static_cast<int32_t>(rb);
                if (B.mono == 2) {
                    cb[q] = __ldg(B.t_col + rb);
                } else if (B.mono == 1) {
                    if (B.kind == kBlockGate)
                        cb[q] = static_cast<int32_t>(rb ^ 1u);
                    else if (rb & B.cmask)
                        cb[q] = static_cast<int32_t>(rb ^ B.tmask);
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                cols[q] = cb[q] < 0 ? -1
                                    : static_cast<int64_t>(((rbase + q) & keep) |
                                                           (static_cast<uint32_t>(cb[q]) << B.shift));
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) cols[q] = mono_col(layer, rbase + q);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int pch = half * 4 + q;  // k = 2 pch, 2 pch + 1
            const uint32_t r0 = rbase + 2 * q;
            double v0r = 0.0, v0i = 0.0, v1r = 0.0, v1i = 0.0, s0 = 0.0, s1 = 0.0;
            if (cols[2 * q] == static_cast<int64_t>(col)) {
                layer_entry(layer, r0, col, v0r, v0i);
                if (THREE_M && !REAL) s0 = __dadd_rn(v0r, v0i);
            }
            if (cols[2 * q + 1] == static_cast<int64_t>(col)) {
                layer_entry(layer, r0 + 1, col, v1r, v1i);
                if (THREE_M && !REAL) s1 = __dadd_rn(v1r, v1i);
            }
            const uint32_t off = n * 128 + ((pch ^ (n & 7)) << 4);
            sts128(bBase + off, v0r, v1r);
            if (!REAL) sts128(bBase + BN * 128 + off, v0i, v1i);
            if (THREE_M && !REAL) sts128(bBase + 2 * BN * 128 + off, s0, s1);
        }
    } else {
        constexpr int EB = 4;  // elements per batch = 2 (k, k+1) pairs
#pragma unroll
        for (int q0 = 0; q0 < C::PAIRS; q0 += EB / 2) {
            uint32_t rr[EB], cc[EB];
            int nn[EB / 2], pp[EB / 2];
#pragma unroll
            for (int h = 0; h < EB / 2; ++h) {
                const int idx = ptid + (q0 + h) * 32 * C::PRODUCER_WARPS;
                nn[h] = idx % BN;
                pp[h] = idx / BN;
                rr[2 * h] = static_cast<uint32_t>(ktg * C::BK + 2 * pp[h]);
                rr[2 * h + 1] = rr[2 * h] + 1;
                cc[2 * h] = cc[2 * h + 1] = static_cast<uint32_t>(n0 + nn[h]);
            }
            double vr[EB], vi[EB];
            gen_batch<EB, C::LOWBITS>(layer, tp, rr, cc, vr, vi);
#pragma unroll
            for (int h = 0; h < EB / 2; ++h) {
                const uint32_t off = nn[h] * 128 + ((pp[h] ^ (nn[h] & 7)) << 4);
                sts128(bBase + off, vr[2 * h], vr[2 * h + 1]);
                if (REAL) continue;
                sts128(bBase + BN * 128 + off, vi[2 * h], vi[2 * h + 1]);
                if (THREE_M) {
                    // real layers: Br + Bi = Br (adding an exact zero; no FP64 op)
                    if (layer.real)
                        sts128(bBase + 2 * BN * 128 + off, vr[2 * h], vr[2 * h + 1]);
                    else
                        sts128(bBase + 2 * BN * 128 + off, __dadd_rn(vr[2 * h], vi[2 * h]),
                               __dadd_rn(vr[2 * h + 1], vi[2 * h + 1]));
                }
            }
        }
    }
}

// Consumer side of the warp-specialised K2: the DMMAs of one stage (BK = 16, two
// k-halves of the lane's 128-bit fragments) into this warp's accumulators. The
// plane addresses are passed in, so stage layouts of different sizes share it.
template <bool THREE_M, bool SUMPLANE, bool REAL, int NACC, int NT>
__device__ __forceinline__ void ws_consume_stage(uint32_t aRe, uint32_t aIm, uint32_t aSm, uint32_t bRe, uint32_t bIm,
                                                 uint32_t bSm, int wm, int wn, int g, int t,
                                                 double (&acc)[NACC][4][NT][2]) {
    using C = WsCfg<THREE_M, SUMPLANE, REAL>;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t choff = static_cast<uint32_t>(((2 * t + h) ^ g) << 4);
        double2 ar[4], ai[4], as2[4], br[NT], bi[NT], bs[NT];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t line = static_cast<uint32_t>(wm * 32 + i * 8 + g) * 128 + choff;
            ar[i] = lds128(aRe + line);
            ai[i] = lds128(aIm + line);
            if (SUMPLANE && !REAL) as2[i] = lds128(aSm + line);
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const uint32_t line = static_cast<uint32_t>(wn * C::WT_N + j * 8 + g) * 128 + choff;
            br[j] = lds128(bRe + line);
            if (!REAL) bi[j] = lds128(bIm + line);
            if (THREE_M && !REAL) bs[j] = lds128(bSm + line);
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            double xr[4], xi[4], yr[NT], yi[NT];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                xr[i] = e ? ar[i].y : ar[i].x;
                xi[i] = e ? ai[i].y : ai[i].x;
            }
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                yr[j] = e ? br[j].y : br[j].x;
                if (!REAL) yi[j] = e ? bi[j].y : bi[j].x;
            }
            if (REAL) {
                // Cr += Ar Br, Ci += Ai Br (Bi = 0 exactly)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[0][i][j], xr[i], yr[j]);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[1][i][j], xi[i], yr[j]);
            } else if (THREE_M) {
                double xs[4], ys[NT];
#pragma unroll
                for (int i = 0; i < 4; ++i) xs[i] = SUMPLANE ? (e ? as2[i].y : as2[i].x) : __dadd_rn(xr[i], xi[i]);
#pragma unroll
                for (int j = 0; j < NT; ++j) ys[j] = e ? bs[j].y : bs[j].x;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[0][i][j], xr[i], yr[j]);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[1][i][j], xi[i], yi[j]);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[2][i][j], xs[i], ys[j]);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[0][i][j], xr[i], yr[j]);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[1][i][j], xr[i], yi[j]);
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[0][i][j], xi[i], neg(yi[j]));
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(acc[1][i][j], xi[i], yr[j]);
            }
        }
    }
}

// Output tile of linear tile index t. group_m = 0: row-major. group_m = G > 0: tiles
// are numbered group by group, a group being G row blocks x all column blocks walked
// column by column (G row blocks per column), so the tiles of one data-parallel wave
// (P consecutive indices) cover G row blocks x ~P/G column blocks instead of ~2 row
// blocks x every column block: each wave re-reads ~P/G B column blocks instead of all
// of them, and the group's G A row blocks stay in L2 across its waves.
__device__ __forceinline__ void sk_tile_coords(int t, int tiles_n, int group_m, int tiles_m, int& tm, int& tn) {
    if (group_m <= 1) {
        tm = t / tiles_n;
        tn = t % tiles_n;
        return;
    }
    const int per_group = group_m * tiles_n;
    const int g = t / per_group;
    const int first = g * group_m;
    const int rows = min(group_m, tiles_m - first);  // the last group may be shorter
    const int r = t - g * per_group;
    tm = first + r % rows;
    tn = r / rows;
}

// MAT_B: the operator was materialised (transposed, [planes][N][N], by
// expand_t_kernel) and B tiles arrive by TMA like A — no FP64 generation work
// in the producer, whose FP64 instructions would otherwise queue behind DMMA on
// the shared FP64 pipe (used for dense, non-monomial layers such as H on every qubit).
template <bool THREE_M, bool SUMPLANE, bool MAT_B, bool REAL = false>
__global__ void __launch_bounds__(WsCfg<THREE_M, SUMPLANE, REAL>::THREADS, 1)
    zgemm_ws_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ LayerDesc layer, double* __restrict__ out, int M, int N,
                    const __grid_constant__ SkArgs sk) {
    using C = WsCfg<THREE_M, SUMPLANE, REAL>;
    constexpr int BM = C::BM, BN = C::BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sBase = smem_u32(smem);
    const uint32_t sFull = sBase + C::STAGES * C::STAGE;
    const uint32_t sEmpty = sFull + 8 * C::STAGES;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    // split-K over the cluster (gridDim.z = cluster size): rank r owns k-tiles [kt0, kt1)
    const int splits = gridDim.z;
    const int rank = blockIdx.z;
    const int KTall = N / C::BK;
    const int kt0 = (KTall * rank) / splits;
    const int KT = (KTall * (rank + 1)) / splits - kt0;
    // Work as segments: classic grids own one segment (their tile, their split-K
    // range). Stream-K grids (P = gridDim.x persistent CTAs) first run sk.dp_waves
    // data-parallel waves — CTA c takes whole tile w P + c in wave w, so the CTAs
    // running together share A row blocks in L2 — then own [I c / P, I (c + 1) / P)
    // of the I = (T - W P) KTall iterations of the remaining tiles (stream-K).
    const int tiles_n = N / BN;
    const int W = sk.enabled ? sk.dp_waves : 0;
    const int tile_base = W * static_cast<int>(gridDim.x);
    const long long I = static_cast<long long>(sk.tiles - tile_base) * KTall;
    const long long it_begin =
        sk.enabled ? I * blockIdx.x / gridDim.x
                   : static_cast<long long>(blockIdx.y * tiles_n + blockIdx.x) * KTall + kt0;
    const long long it_end = sk.enabled ? I * (blockIdx.x + 1) / gridDim.x : it_begin + KT;
    // Next segment of this CTA: data-parallel waves, then the (stream-K) range.
    auto next_segment = [&](int& seg, long long& it, int& tile, int& k0, int& k1) -> bool {
        if (seg < W) {
            tile = seg * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x);
            k0 = 0;
            k1 = KTall;
            ++seg;
            return true;
        }
        if (it >= it_end) return false;
        tile = tile_base + static_cast<int>(it / KTall);
        k0 = static_cast<int>(it % KTall);
        k1 = static_cast<int>(min(static_cast<long long>(KTall), k0 + (it_end - it)));
        it += k1 - k0;
        return true;
    };
    // CTA whose stream-K share holds iteration x
    auto cta_of = [&](long long x) {
        long long c = x * gridDim.x / I;
        while (c + 1 < gridDim.x && I * (c + 1) / gridDim.x <= x) ++c;
        while (c > 0 && I * c / gridDim.x > x) --c;
        return static_cast<int>(c);
    };
    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(sFull + 8 * s, 1 + C::PRODUCER_WARPS);
            mbar_init(sEmpty + 8 * s, C::CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        if (MAT_B) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    __syncthreads();  // barriers initialised (synccheck's report at this barrier)
    // Programmatic dependent launch: everything above overlapped the previous
    // GEMM's tail; from here on we read its output (A) and overwrite its input
    // (out), so every thread waits for its completion. Then let the next GEMM start launching.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp >= C::CONSUMER_WARPS) {
        // ------------------------------ producer warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::PRODUCER_REGS));
        const int ptid = tid - 32 * C::CONSUMER_WARPS;
        int kc = 0;  // stage counter across segments
        uint32_t zero_stages = 0;  // stages whose B region this thread left zero
        int seg = 0, tile, seg_k0, seg_k1;
        long long it = it_begin;
        while (next_segment(seg, it, tile, seg_k0, seg_k1)) {
        int tm, tn;
        sk_tile_coords(tile, tiles_n, sk.enabled ? sk.group_m : 0, M / BM, tm, tn);
        const int m0 = tm * BM;
        const int n0 = tn * BN;
        for (int ktg = seg_k0; ktg < seg_k1; ++ktg, ++kc) {
            const int s = kc % C::STAGES;
            if (kc >= C::STAGES) mbar_wait(sEmpty + 8 * s, ((kc / C::STAGES) & 1) ^ 1);
            const uint32_t stage = sBase + s * C::STAGE;
            const uint32_t tma_bar = sFull + 8 * s;
            const uint32_t bBase = stage + C::A_BYTES;
            if (MAT_B) {
                // operator tiles the layer's structure makes exactly zero (row and column
                // disagree on an identity / control bit above the tile: most tiles of a
                // controlled-phase or permutation layer) are cleared in shared memory
                // instead of streamed from the materialised operator — same DMMAs, no bytes
                constexpr uint32_t LOW = (1u << C::LOWBITS) - 1u;
                const bool zero = sk.zero_skip &&
                                  ((static_cast<uint32_t>(ktg * C::BK) ^ static_cast<uint32_t>(n0)) & layer.zmask &
                                   ~LOW) != 0;
                if (ptid == 0) {
                    mbar_expect_tx(tma_bar, C::A_TMA_BYTES + (zero ? 0 : C::B_BYTES));
                    tma_load_3d(stage, &tmA, tma_bar, ktg * C::BK, m0, 0);
                    if (!zero) tma_load_3d(bBase, &tmB, tma_bar, ktg * C::BK, n0, 0);
                }
                if (zero && !((zero_stages >> s) & 1u))
                    for (int o = ptid * 16; o < C::B_BYTES; o += 16 * 32 * C::PRODUCER_WARPS) sts128(bBase + o, 0.0, 0.0);
                zero_stages = zero ? (zero_stages | (1u << s)) : (zero_stages & ~(1u << s));
                __syncwarp();
                if (lane == 0) mbar_arrive(sFull + 8 * s);
                continue;
            }
            if (ptid == 0) {
                mbar_expect_tx(tma_bar, C::A_TMA_BYTES);
                tma_load_3d(stage, &tmA, tma_bar, ktg * C::BK, m0, 0);
            }
            ws_produce_b<THREE_M, SUMPLANE, REAL>(layer, bBase, ptid, ktg, n0, s, zero_stages);
            __syncwarp();
            if (lane == 0) mbar_arrive(sFull + 8 * s);
        }
        }
        if (splits > 1) {  // every thread of the cluster takes part in both cluster barriers
            cluster_sync();
            cluster_sync();
        }
        return;
    }

    // ------------------------------ consumer warpgroups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CONSUMER_REGS));
    const int g = lane >> 2;
    const int t = lane & 3;
    const int wm = warp / C::CWN;
    const int wn = warp % C::CWN;
    constexpr int NT = C::NT;
    constexpr int NACC = (THREE_M && !REAL) ? 3 : 2;
    int kc = 0;  // stage counter across segments (mirrors the producer's)
    // A stage is released (arrive on sEmpty) only after a block boundary that follows all of
    // its DMMAs: at the top of the next k-tile iteration, or after the k-loop. Releasing at the
    // end of the k-tile is not enough: ptxas schedules that arrive right after the stage's last
    // LDS, before its data has returned (the DMMAs consuming it come later), and the producer's
    // TMA refill can then overwrite the stage under the load — seen as one wrong k-tile in the
    // last fragment of whichever warp arrives last. Issued DMMAs have read their operands.
    int pending = -1;
    int seg = 0, tile, seg_k0, seg_k1;
    long long it = it_begin;
    while (next_segment(seg, it, tile, seg_k0, seg_k1)) {
    int tm, tn;
    sk_tile_coords(tile, tiles_n, sk.enabled ? sk.group_m : 0, M / BM, tm, tn);
    const int m0 = tm * BM;
    const int n0 = tn * BN;
    double acc[NACC][4][NT][2];
#pragma unroll
    for (int a = 0; a < NACC; ++a)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[a][i][j][0] = acc[a][i][j][1] = 0.0;

    for (int ktg = seg_k0; ktg < seg_k1; ++ktg, ++kc) {
        if (pending >= 0) {  // the previous stage (its DMMAs are issued: its loads have returned)
            __syncwarp();
            if (lane == 0) mbar_arrive(sEmpty + 8 * pending);
        }
        const int s = kc % C::STAGES;
        mbar_wait(sFull + 8 * s, (kc / C::STAGES) & 1);
        pending = s;
        const uint32_t aRe = sBase + s * C::STAGE;
        const uint32_t aIm = aRe + BM * 128;
        const uint32_t aSm = aIm + BM * 128;
        const uint32_t bRe = aRe + C::A_BYTES;
        const uint32_t bIm = bRe + BN * 128;
        const uint32_t bSm = bIm + BN * 128;
        ws_consume_stage<THREE_M, SUMPLANE, REAL>(aRe, aIm, aSm, bRe, bIm, bSm, wm, wn, g, t, acc);
    }
    if (pending >= 0) {  // the segment's last stage, before the epilogue
        __syncwarp();
        if (lane == 0) mbar_arrive(sEmpty + 8 * pending);
        pending = -1;
    }

    // Output fragment (i, j) of this warp: combine the accumulators (3M: Cr = T1 - T2,
    // Ci = T3 - T1 - T2) and store re, im (and re + im for the next 3M GEMM).
    const size_t plane = static_cast<size_t>(M) * N;
    auto store = [&](int i, int j, const double (&f)[NACC][2]) {
        const int row = m0 + wm * 32 + i * 8 + g;
        const int col = n0 + wn * C::WT_N + j * 8 + 2 * t;
        const size_t o = static_cast<size_t>(row) * N + col;
        double r0, r1, i0, i1;
        if (THREE_M && !REAL) {
            r0 = f[0][0] - f[1][0];
            r1 = f[0][1] - f[1][1];
            i0 = f[2][0] - f[0][0] - f[1][0];
            i1 = f[2][1] - f[0][1] - f[1][1];
        } else {
            r0 = f[0][0];
            r1 = f[0][1];
            i0 = f[1][0];
            i1 = f[1][1];
        }
        *reinterpret_cast<double2*>(out + o) = make_double2(r0, r1);
        *reinterpret_cast<double2*>(out + plane + o) = make_double2(i0, i1);
        if (SUMPLANE)
            *reinterpret_cast<double2*>(out + 2 * plane + o) = make_double2(__dadd_rn(r0, i0), __dadd_rn(r1, i1));
    };

    if (splits > 1) {
        // Deterministic split-K: every rank parks its partial accumulators in its own
        // shared memory ([value][consumer thread]); rank r then finishes the m8 row
        // blocks i with i * splits / 4 == r, summing the partials of ranks 0..s-1 in
        // that fixed order through distributed shared memory, and stores them.
        constexpr int CT = 32 * C::CONSUMER_WARPS;
        constexpr int NV = NACC * 4 * NT * 2;
        static_assert(NV * CT * 8 <= C::STAGES * C::STAGE, "partials must fit the pipeline buffers");
        asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");  // all consumers are past the last stage
        const uint32_t part = sBase + static_cast<uint32_t>(tid) * 8;
        auto vidx = [](int a, int i, int j, int e) { return ((a * 4 + i) * NT + j) * 2 + e; };
#pragma unroll
        for (int a = 0; a < NACC; ++a)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        asm volatile("st.shared.f64 [%0], %1;" ::"r"(part + vidx(a, i, j, e) * CT * 8),
                                     "d"(acc[a][i][j][e])
                                     : "memory");
        cluster_sync();
        // Rank r's share: the row blocks i with i * splits / 4 == r (none when splits = 8 and r is
        // odd). All remote loads of a fragment are issued before any add, so their DSMEM latencies
        // overlap instead of chaining; the sum then runs over ranks 0..s-1 in order (deterministic).
        uint32_t src[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < splits) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(src[q]) : "r"(part), "r"(q));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if ((i * splits) / 4 != rank) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                double x[8][NACC][2];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q >= splits) break;
#pragma unroll
                    for (int a = 0; a < NACC; ++a)
#pragma unroll
                        for (int e = 0; e < 2; ++e)
                            asm volatile("ld.shared::cluster.f64 %0, [%1];"
                                         : "=d"(x[q][a][e])
                                         : "r"(src[q] + vidx(a, i, j, e) * CT * 8));
                }
                double f[NACC][2];
#pragma unroll
                for (int a = 0; a < NACC; ++a)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        f[a][e] = x[0][a][e];
#pragma unroll
                        for (int q = 1; q < 8; ++q)
                            if (q < splits) f[a][e] = f[a][e] + x[q][a][e];
                    }
                store(i, j, f);
            }
        }
        cluster_sync();  // every rank keeps its shared memory alive until all have read it
        return;
    }

    if (sk.enabled && !(seg_k0 == 0 && seg_k1 == KTall)) {
        // Stream-K tile shared with other CTAs: the CTA holding k-tiles [0, k1) owns it.
        constexpr int CT = 32 * C::CONSUMER_WARPS;
        constexpr int NV = NACC * 4 * NT * 2;
        auto vidx = [](int a, int i, int j, int e) { return ((a * 4 + i) * NT + j) * 2 + e; };
        // A split tile is its owner's LAST segment, so the owner CTA indexes the partial
        // slots and the flag: the workspace is [P][maxc] slots, not one per tile.
        const long long tile_first = static_cast<long long>(tile - tile_base) * KTall;  // stream-K space
        const int owner = seg_k0 > 0 ? cta_of(tile_first) : static_cast<int>(blockIdx.x);
        double* tile_ws = sk.ws + static_cast<size_t>(owner) * sk.maxc * NV * CT + tid;
        int* flag = sk.flags + owner;
        if (seg_k0 > 0) {
            // contributor: publish the partial, then count it in
            double* dst = tile_ws + static_cast<size_t>(static_cast<int>(blockIdx.x) - owner - 1) * NV * CT;
#pragma unroll
            for (int a = 0; a < NACC; ++a)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) __stcg(dst + vidx(a, i, j, e) * CT, acc[a][i][j][e]);
            // release: every consumer fences its own stores, the CTA barrier orders them before
            // thread 0's fence + flag increment, which the owner's threads acquire
            __threadfence();
            asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
            if (tid == 0) {
                __threadfence();
                const int old = atomicAdd(flag, 1);
                if (sk.dbg) {
                    const int slot = static_cast<int>(blockIdx.x) - owner - 1;
                    const int nc = cta_of(tile_first + KTall - 1) - owner;
                    atomicAdd(sk.dbg + 3, 1);
                    if (slot < 0 || slot >= sk.maxc) atomicAdd(sk.dbg + 1, 1);
                    if (old >= nc) atomicAdd(sk.dbg + 5, 1);
                }
            }
            continue;
        }
        // owner: wait for the contributors, add their partials in k order, store. Every
        // consumer thread acquires the flag itself (no reliance on barrier cumulativity).
        const int ncontrib = cta_of(tile_first + KTall - 1) - static_cast<int>(blockIdx.x);
        {
            int v = 0;
            do {
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            } while (v < ncontrib);
            if (sk.dbg && tid == 0) {
                atomicAdd(sk.dbg + 2, 1);
                atomicAdd(sk.dbg + 4, ncontrib);
                if (v != ncontrib) atomicAdd(sk.dbg + 0, 1);
            }
        }
        __syncwarp();
        for (int q = 0; q < ncontrib; ++q) {
            const double* src = tile_ws + static_cast<size_t>(q) * NV * CT;
#pragma unroll
            for (int a = 0; a < NACC; ++a)
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j)
#pragma unroll
                        for (int e = 0; e < 2; ++e) acc[a][i][j][e] += __ldcg(src + vidx(a, i, j, e) * CT);
        }
        // the owner is this flag's only reader in this launch: re-arm it for the next
        // GEMM (which starts after this grid completes: griddepcontrol.wait)
        asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
        if (tid == 0) *flag = 0;
    }

#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            double f[NACC][2];
#pragma unroll
            for (int a = 0; a < NACC; ++a) {
                f[a][0] = acc[a][i][j][0];
                f[a][1] = acc[a][i][j][1];
            }
            store(i, j, f);
        }
    }  // segments
}

template <bool THREE_M, bool SUMPLANE, bool REAL>
static int configure_ws_one() {
    int e = static_cast<int>(cudaFuncSetAttribute(zgemm_ws_kernel<THREE_M, SUMPLANE, false, REAL>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  WsCfg<THREE_M, SUMPLANE, REAL>::SMEM));
    if (e) return e;
    return static_cast<int>(cudaFuncSetAttribute(zgemm_ws_kernel<THREE_M, SUMPLANE, true, REAL>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 WsCfg<THREE_M, SUMPLANE, REAL>::SMEM));
}

template <bool THREE_M, bool SUMPLANE>
static int configure_ws_t() {
    int e = configure_ws_one<THREE_M, SUMPLANE, false>();
    if (e || !THREE_M) return e;
    return configure_ws_one<THREE_M, SUMPLANE, true>();
}

template <bool THREE_M, bool SUMPLANE, bool MAT_B, bool REAL>
static int launch_ws_t(const GemmArgs& a, void* stream) {
    using C = WsCfg<THREE_M, SUMPLANE, REAL>;
    const int splits = a.splits > 1 ? a.splits : 1;
    // REAL reads two planes of V (and one of a materialised operator): their own tensor maps
    const CUtensorMap& tmA = *static_cast<const CUtensorMap*>(REAL && a.tmap_real ? a.tmap_real : a.tmap);
    const CUtensorMap& tmB =
        MAT_B ? *static_cast<const CUtensorMap*>(REAL && a.tmap_b_real ? a.tmap_b_real : a.tmap_b) : tmA;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = a.sk.enabled ? dim3(static_cast<unsigned>(ws_max_active_clusters(1)), 1, 1)
                               : dim3(a.N / C::BN, a.M / C::BM, splits);
    cfg.blockDim = dim3(C::THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[2];
    int na = 0;
    // chained GEMMs overlap launch and prologue with the previous one's tail (griddepcontrol)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = std::getenv("QSB_NO_PDL") ? 0 : 1;
    ++na;
    if (splits > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = splits;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, zgemm_ws_kernel<THREE_M, SUMPLANE, MAT_B, REAL>, tmA, tmB,
                                               *a.layer, a.out, a.M, a.N, a.sk));
}

template <bool THREE_M, bool SUMPLANE>
static int launch_ws_any(const GemmArgs& a, void* stream) {
    if (THREE_M && a.real) {
        return a.tmap_b ? launch_ws_t<THREE_M, SUMPLANE, true, true>(a, stream)
                        : launch_ws_t<THREE_M, SUMPLANE, false, true>(a, stream);
    }
    return a.tmap_b ? launch_ws_t<THREE_M, SUMPLANE, true, false>(a, stream)
                    : launch_ws_t<THREE_M, SUMPLANE, false, false>(a, stream);
}

// K1t: the layer operator transposed, Lt[p][n][k] = L[k][n] for planes re, im
// (and re + im when planes == 3): the TMA source of a materialised B operand.
// Entries are layer_entry's (bit-exact); consecutive threads write consecutive k.
// skip_zero: entries inside K2 operator tiles that K2 clears instead of loading (row and
// column disagree on a zmask bit above the 64-wide tile: sk.zero_skip) are not written —
// K2 never reads them, so a controlled-phase layer's expansion writes ~1/32 of the plane.
__global__ void __launch_bounds__(256) expand_t_kernel(const __grid_constant__ LayerDesc d, int N,
                                                       double* __restrict__ out, int planes, int skip_zero) {
    const size_t plane = static_cast<size_t>(N) * N;
    const size_t pairs = plane / 2;
    const uint32_t half_n = static_cast<uint32_t>(N) / 2;
    const uint32_t skip_mask = skip_zero ? (d.zmask & ~63u) : 0u;
    for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < pairs;
         p += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint32_t n = static_cast<uint32_t>(p / half_n);
        const uint32_t k = static_cast<uint32_t>(p % half_n) * 2;
        if ((k ^ n) & skip_mask) continue;
        double r0, i0, r1, i1;
        layer_entry(d, k, n, r0, i0);
        layer_entry(d, k + 1, n, r1, i1);
        reinterpret_cast<double2*>(out)[p] = make_double2(r0, r1);
        reinterpret_cast<double2*>(out + plane)[p] = make_double2(i0, i1);
        if (planes == 3)
            reinterpret_cast<double2*>(out + 2 * plane)[p] = make_double2(__dadd_rn(r0, i0), __dadd_rn(r1, i1));
    }
}

int launch_expand_t(const LayerDesc& layer, int N, double* out, int planes, void* stream, int skip_zero) {
    const size_t pairs = static_cast<size_t>(N) * N / 2;
    int blocks = static_cast<int>((pairs + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    expand_t_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(layer, N, out, planes, skip_zero);
    return static_cast<int>(cudaGetLastError());
}

int gemm_tile_b_planes(int tile) { return tile == kTileWs3MS || tile == kTileWs3M ? 3 : 2; }

// Co-resident clusters of the warp-specialised kernel per split size (index log2 s),
// from the occupancy API at configure time: clusters must fit inside a GPC, so
// e.g. clusters of 8 do not tile 148 SMs.
static int g_ws_clusters[4] = {148, 74, 37, 18};

int ws_max_active_clusters(int splits) {
    const int i = splits >= 8 ? 3 : (splits >= 4 ? 2 : (splits >= 2 ? 1 : 0));
    return g_ws_clusters[i];
}

static void query_ws_clusters() {
    using C = WsCfg<true, true>;
    for (int i = 1; i < 4; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1, 1, 1 << i);
        cfg.blockDim = dim3(C::THREADS, 1, 1);
        cfg.dynamicSmemBytes = C::SMEM;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1 << i;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, zgemm_ws_kernel<true, true, false, false>, &cfg) == cudaSuccess && n > 0)
            g_ws_clusters[i] = n;
        else
            cudaGetLastError();
    }
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_ws_clusters[0] = sms;
}

int gemm_tile_rows(int tile) {
    switch (tile) {
    case kTile128x64: return 128;
    case kTile64x64: return 64;
    case kTileWs4M: return WsCfg<false>::BM;
    case kTileWs3M: return WsCfg<true>::BM;
    case kTileWs3MS: return WsCfg<true, true>::BM;
    default: return 32;
    }
}
int gemm_tile_planes(int tile) { return tile == kTileWs3MS ? 3 : 2; }

int ws_partial_values(int tile) {
    // accumulators per consumer thread: NACC x 4 x NT x 2 (4M: 2 x 4 x 4 x 2, 3M: 3 x 4 x 2 x 2)
    return tile == kTileWs4M ? 64 : 48;
}

int gemm_tile_cols(int tile) {
    switch (tile) {
    case kTile32x32: return 32;
    case kTileWs4M: return WsCfg<false>::BN;
    case kTileWs3M: return WsCfg<true>::BN;
    case kTileWs3MS: return WsCfg<true, true>::BN;
    default: return 64;
    }
}

template <int BM, int BN>
static int configure_zgemm_t() {
    return static_cast<int>(cudaFuncSetAttribute(zgemm_gen_kernel<BM, BN>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 GemmCfg<BM, BN>::SMEM));
}

template <int BM, int BN>
static int launch_zgemm_t(const GemmArgs& a, void* stream) {
    using C = GemmCfg<BM, BN>;
    dim3 grid(a.N / BN, a.M / BM);
    zgemm_gen_kernel<BM, BN><<<grid, C::THREADS, C::SMEM, static_cast<cudaStream_t>(stream)>>>(
        *static_cast<const CUtensorMap*>(a.tmap), *a.layer, a.out, a.M, a.N);
    return static_cast<int>(cudaGetLastError());
}

int launch_zgemm(const GemmArgs& a, int tile, int /*gemm_mode*/, void* stream) {
    switch (tile) {
    case kTileWs4M: return launch_ws_any<false, false>(a, stream);
    case kTileWs3M: return launch_ws_any<true, false>(a, stream);
    case kTileWs3MS: return launch_ws_any<true, true>(a, stream);
    case kTile128x64: return launch_zgemm_t<128, 64>(a, stream);
    case kTile64x64: return launch_zgemm_t<64, 64>(a, stream);
    default: return launch_zgemm_t<32, 32>(a, stream);
    }
}

// ----------------------------------------------------------------------------
// K2c: the whole GEMM chain of a plan in ONE persistent launch, dataflow across layers
// ----------------------------------------------------------------------------
//
// P persistent CTAs (one per SM, all co-resident) take units u = c, c + P, c + 2P, ...
// of the chain's unit list, GEMM-major: unit = (GEMM l, output tile t = (tm, tn), k-split
// s of S, KT / S k-tiles each). Rows tm of V_{l+1} = V_l L_l depend only on rows tm of
// V_l (the row-block independence of SURVEY 8(e), at tile granularity), so a unit of
// GEMM l loads its A rows as soon as row_done[tm] >= l * tiles_n — every tile of row
// block tm of GEMM l-1 stored — while GEMM l-1 is still running on other row blocks:
// no grid-wide barrier, no per-GEMM launch, pipeline fill or tail wave. The same
// counter orders the overwrite of V_{l-1} (read only by units of row tm of GEMM l-1).
// Split-K: the unit holding the LAST k-split finishes the tile — it waits for the other
// splits' partials (tile_flags, monotonic over the chain) and adds them to its own in
// split order (a fixed order: the same bits every run). Every wait targets a lower unit index and every CTA runs its
// units in increasing order, so the lowest unfinished unit can always proceed: no
// deadlock while all P CTAs are resident (one stream per device).
// Each GEMM runs as 3M (complex layer) or as two real products (real layer) by a
// run-time, CTA-uniform branch on layers[l].real; stages use the 3M sum-plane layout
// for both (a real layer fills two A planes and one B plane of it). Operator tiles are
// always generated in shared memory (chains with a layer that needs materialising
// keep the per-GEMM launches).
struct ChainCfg {
    using C3 = WsCfg<true, true, false>;
    using CR = WsCfg<true, true, true>;
    static constexpr int THREADS = C3::THREADS;
    static constexpr int STAGE = C3::STAGE;
    static constexpr int STAGES = C3::STAGES;
    static constexpr int SMEM = C3::SMEM;
    static constexpr int NT = C3::NT;
    static constexpr int NV = 3 * 4 * NT * 2;  // accumulator values per consumer thread
    static constexpr int CT = 32 * C3::CONSUMER_WARPS;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(ChainCfg::THREADS, 1)
    zgemm_chain_kernel(const __grid_constant__ CUtensorMap tm3_0, const __grid_constant__ CUtensorMap tm3_1,
                       const __grid_constant__ CUtensorMap tm2_0, const __grid_constant__ CUtensorMap tm2_1,
                       const LayerDesc* __restrict__ layers, int n_gemms, double* __restrict__ v0,
                       double* __restrict__ v1, int M, int N, int S, double* __restrict__ ws,
                       int* __restrict__ tile_flags, int* __restrict__ row_done) {
    using C = ChainCfg::C3;
    constexpr int BM = C::BM, BN = C::BN, NT = ChainCfg::NT, NV = ChainCfg::NV, CT = ChainCfg::CT;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sBase = smem_u32(smem);
    const uint32_t sFull = sBase + C::STAGES * C::STAGE;
    const uint32_t sEmpty = sFull + 8 * C::STAGES;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int tiles_n = N / BN;
    const int T = (M / BM) * tiles_n;
    const long long U1 = static_cast<long long>(T) * S;
    const long long U = U1 * n_gemms;
    const int KS = (N / C::BK) / S;
    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(sFull + 8 * s, 1 + C::PRODUCER_WARPS);
            mbar_init(sEmpty + 8 * s, C::CONSUMER_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm3_0)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm3_1)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm2_0)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm2_1)) : "memory");
    }
    __syncthreads();

    if (warp >= C::CONSUMER_WARPS) {
        // ------------------------------ producer warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::PRODUCER_REGS));
        const int ptid = tid - 32 * C::CONSUMER_WARPS;
        int kc = 0;
        for (long long u = blockIdx.x; u < U; u += gridDim.x) {
            const int l = static_cast<int>(u / U1);
            const int rem = static_cast<int>(u % U1);
            const int tile = rem / S, sp = rem % S;
            const int tm = tile / tiles_n;
            const int m0 = tm * BM, n0 = (tile % tiles_n) * BN;
            const LayerDesc& L = layers[l];
            const bool real = L.real != 0;
            if (l > 0 && ptid == 0) {
                // rows tm of V_l are complete (every tile of row block tm of GEMM l-1 stored)
                const int need = l * tiles_n;
                while (ld_acquire(row_done + tm) < need) __nanosleep(64);
                // generic-proxy stores of other CTAs, acquired above, before our async-proxy (TMA) reads
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            const CUtensorMap* ta = real ? ((l & 1) ? &tm2_1 : &tm2_0) : ((l & 1) ? &tm3_1 : &tm3_0);
            const uint32_t a_bytes = real ? ChainCfg::CR::A_TMA_BYTES : C::A_TMA_BYTES;
            for (int ktg = sp * KS; ktg < (sp + 1) * KS; ++ktg, ++kc) {
                const int s = kc % C::STAGES;
                if (kc >= C::STAGES) mbar_wait(sEmpty + 8 * s, ((kc / C::STAGES) & 1) ^ 1);
                const uint32_t stage = sBase + s * C::STAGE;
                const uint32_t tma_bar = sFull + 8 * s;
                if (ptid == 0) {
                    mbar_expect_tx(tma_bar, a_bytes);
                    tma_load_3d(stage, ta, tma_bar, ktg * C::BK, m0, 0);
                }
                // (the real and 3M variants clear different B sizes: no zero-stage reuse across them)
                if (real) {
                    uint32_t none = 0;
                    ws_produce_b<true, true, true>(L, stage + C::A_BYTES, ptid, ktg, n0, s, none);
                } else {
                    uint32_t none = 0;
                    ws_produce_b<true, true, false>(L, stage + C::A_BYTES, ptid, ktg, n0, s, none);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(sFull + 8 * s);
            }
        }
        return;
    }

    // ------------------------------ consumer warpgroups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::CONSUMER_REGS));
    const int g = lane >> 2;
    const int t = lane & 3;
    const int wm = warp / C::CWN;
    const int wn = warp % C::CWN;
    const size_t plane = static_cast<size_t>(M) * N;
    int kc = 0;
    int pending = -1;  // stage released after the next block boundary (see zgemm_ws_kernel)
    auto vidx = [](int a, int i, int j, int e) { return ((a * 4 + i) * NT + j) * 2 + e; };
    for (long long u = blockIdx.x; u < U; u += gridDim.x) {
        const int l = static_cast<int>(u / U1);
        const int rem = static_cast<int>(u % U1);
        const int tile = rem / S, sp = rem % S;
        const int tm = tile / tiles_n;
        const int m0 = tm * BM, n0 = (tile % tiles_n) * BN;
        const bool real = layers[l].real != 0;
        double acc[3][4][NT][2];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[a][i][j][0] = acc[a][i][j][1] = 0.0;
        for (int k = 0; k < KS; ++k, ++kc) {
            if (pending >= 0) {
                __syncwarp();
                if (lane == 0) mbar_arrive(sEmpty + 8 * pending);
            }
            const int s = kc % C::STAGES;
            mbar_wait(sFull + 8 * s, (kc / C::STAGES) & 1);
            pending = s;
            const uint32_t aRe = sBase + s * C::STAGE;
            const uint32_t aIm = aRe + BM * 128;
            const uint32_t aSm = aIm + BM * 128;
            const uint32_t bRe = aRe + C::A_BYTES;
            const uint32_t bIm = bRe + BN * 128;
            const uint32_t bSm = bIm + BN * 128;
            if (real)
                ws_consume_stage<true, true, true>(aRe, aIm, aSm, bRe, bIm, bSm, wm, wn, g, t, acc);
            else
                ws_consume_stage<true, true, false>(aRe, aIm, aSm, bRe, bIm, bSm, wm, wn, g, t, acc);
        }
        if (pending >= 0) {
            __syncwarp();
            if (lane == 0) mbar_arrive(sEmpty + 8 * pending);
            pending = -1;
        }
        if (S > 1) {
            double* slot = ws + static_cast<size_t>(tile) * (S - 1) * NV * CT + tid;
            if (sp < S - 1) {
                // contributor: publish the partial, then count it in (release)
                double* dst = slot + static_cast<size_t>(sp) * NV * CT;
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < NT; ++j)
#pragma unroll
                            for (int e = 0; e < 2; ++e) __stcg(dst + vidx(a, i, j, e) * CT, acc[a][i][j][e]);
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
                if (tid == 0) {
                    __threadfence();
                    atomicAdd(tile_flags + tile, 1);
                }
                continue;
            }
            // finisher: its own k range plus the other splits' partials
            const int need = (l + 1) * (S - 1);
            while (ld_acquire(tile_flags + tile) < need) __nanosleep(32);
            for (int q = 0; q < S - 1; ++q) {  // fixed order: own + p_0 + p_1 + ... (deterministic)
                const double* src = slot + static_cast<size_t>(q) * NV * CT;
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < NT; ++j)
#pragma unroll
                            for (int e = 0; e < 2; ++e) acc[a][i][j][e] += __ldcg(src + vidx(a, i, j, e) * CT);
            }
        }
        // store the tile: re, im and the sum plane (the next GEMM may be 3M)
        double* out = (l & 1) ? v0 : v1;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int row = m0 + wm * 32 + i * 8 + g;
                const int col = n0 + wn * C::WT_N + j * 8 + 2 * t;
                const size_t o = static_cast<size_t>(row) * N + col;
                double r0, r1, i0, i1;
                if (real) {
                    r0 = acc[0][i][j][0];
                    r1 = acc[0][i][j][1];
                    i0 = acc[1][i][j][0];
                    i1 = acc[1][i][j][1];
                } else {
                    r0 = acc[0][i][j][0] - acc[1][i][j][0];
                    r1 = acc[0][i][j][1] - acc[1][i][j][1];
                    i0 = acc[2][i][j][0] - acc[0][i][j][0] - acc[1][i][j][0];
                    i1 = acc[2][i][j][1] - acc[0][i][j][1] - acc[1][i][j][1];
                }
                *reinterpret_cast<double2*>(out + o) = make_double2(r0, r1);
                *reinterpret_cast<double2*>(out + plane + o) = make_double2(i0, i1);
                *reinterpret_cast<double2*>(out + 2 * plane + o) = make_double2(__dadd_rn(r0, i0), __dadd_rn(r1, i1));
            }
        // publish: the tile counts towards row block tm of V_{l+1} (release); the proxy fence
        // orders these generic stores before the async-proxy (TMA) reads that consume them
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(CT) : "memory");
        if (tid == 0) {
            __threadfence();
            atomicAdd(row_done + tm, 1);
        }
    }
}

size_t chain_ws_bytes(int M, int N, int S) {
    const size_t T = static_cast<size_t>(M / ChainCfg::C3::BM) * (N / ChainCfg::C3::BN);
    return S > 1 ? T * (S - 1) * ChainCfg::NV * ChainCfg::CT * sizeof(double) : 0;
}

int launch_chain(const ChainArgs& a, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int T = (a.M / ChainCfg::C3::BM) * (a.N / ChainCfg::C3::BN);
    int e;
    if ((e = static_cast<int>(cudaMemsetAsync(a.row_done, 0, sizeof(int) * (a.M / ChainCfg::C3::BM), s)))) return e;
    if (a.splits > 1 && (e = static_cast<int>(cudaMemsetAsync(a.tile_flags, 0, sizeof(int) * T, s)))) return e;
    const unsigned P = static_cast<unsigned>(ws_max_active_clusters(1));
    zgemm_chain_kernel<<<P, ChainCfg::THREADS, ChainCfg::SMEM, s>>>(
        *static_cast<const CUtensorMap*>(a.tmap3[0]), *static_cast<const CUtensorMap*>(a.tmap3[1]),
        *static_cast<const CUtensorMap*>(a.tmap2[0]), *static_cast<const CUtensorMap*>(a.tmap2[1]), a.layers,
        a.n_gemms, a.v[0], a.v[1], a.M, a.N, a.splits, a.ws, a.tile_flags, a.row_done);
    return static_cast<int>(cudaGetLastError());
}

// ----------------------------------------------------------------------------
// K2s: whole circuit in one CTA (2^n <= 32): launch-latency bound sizes.
// ----------------------------------------------------------------------------

// Operator rows generated per chunk: the whole operator up to N = 64, 32 rows at N = 128, 16 at N = 256.
__host__ __device__ constexpr int small_kc(int N) { return N <= 64 ? N : (N == 128 ? 32 : 16); }

size_t small_circuit_smem_bytes(int M, int N) {
    return sizeof(double) * (2 * static_cast<size_t>(M) * N * 2 + 2 * static_cast<size_t>(small_kc(N)) * N);
}

// The whole chain for N <= 256 in one launch, no inter-CTA exchange: CTA b owns
// rows [b R, b R + R) of V for every layer (rows of V <- V L depend only on the
// same rows of V). V and V' ping-pong in shared memory; each layer operator is
// generated KC rows at a time into shared memory (every CTA generates the whole
// operator — cheap next to the products), and every thread accumulates its
// outputs over the chunks. N is a template parameter: index arithmetic by
// constants and fully unrolled inner loops. x == nullptr means psi0 = |0...0>:
// psi = V[:, 0] (the reference's matvec with e_0 adds only exact zeros to V[i][0]).
template <int N>
__global__ void __launch_bounds__(1024) small_circuit_kernel(const SmallLayerDesc* __restrict__ layers, int nlayers,
                                                            int transpose, uint32_t row_begin, int M,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ v_out,
                                                            double* __restrict__ psi) {
    constexpr int KC = small_kc(N);
    constexpr int MAXQ = 2;  // outputs per thread (R N <= 2048 with 1024 threads)
    extern __shared__ double sm[];
    // Layer descriptors are staged in shared memory one ahead (cp.async), so the
    // generator's field reads never chase pointers through global memory.
    __shared__ __align__(16) SmallLayerDesc desc[2];
    constexpr int DESC_WORDS = static_cast<int>(sizeof(SmallLayerDesc) / 8);
    static_assert(sizeof(SmallLayerDesc) % 8 == 0, "SmallLayerDesc is copied in 8-byte words");
    const int R = M / gridDim.x;
    const int cta_row = blockIdx.x * R;
    row_begin += static_cast<uint32_t>(cta_row);
    const int out_plane = M * N;
    v_out += static_cast<size_t>(cta_row) * N;
    psi += cta_row;
    const int psi_plane = M;
    const int MN = R * N;
    double* lr = sm + 4 * MN;
    double* li = lr + KC * N;
    const int tid = threadIdx.x;
    auto fetch = [&](int l, int slot) {
        const uint64_t* src = reinterpret_cast<const uint64_t*>(layers + l);
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&desc[slot]));
        for (int w = tid; w < DESC_WORDS; w += blockDim.x)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8 * w), "l"(src + w) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    fetch(0, 0);
    if (nlayers > 1) {
        fetch(1, 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // layer 0 has landed
    } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    for (int e = tid; e < MN; e += blockDim.x) {
        const uint32_t r = row_begin + e / N, c = e % N;
        layer_entry(desc[0], transpose ? c : r, transpose ? r : c, sm[e], sm[MN + e]);
    }
    int cur = 0;  // V in planes [2 cur, 2 cur + 1] of sm
    for (int l = 1; l < nlayers; ++l) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();  // desc[l & 1] has landed; every thread is done with desc[(l - 1) & 1]
        if (l + 1 < nlayers) fetch(l + 1, (l + 1) & 1);
        const SmallLayerDesc& d = desc[l & 1];
        const double* vr = sm + (2 * cur) * MN;
        const double* vi = vr + MN;
        double* tr = sm + (2 * (cur ^ 1)) * MN;
        double* ti = tr + MN;
        double accr[MAXQ], acci[MAXQ];
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) accr[q] = acci[q] = 0.0;
        for (int k0 = 0; k0 < N; k0 += KC) {
            if (k0 > 0) __syncthreads();  // the previous chunk is consumed
            for (int e = tid; e < KC * N; e += blockDim.x) {
                const uint32_t r = static_cast<uint32_t>(k0 + e / N), c = static_cast<uint32_t>(e % N);
                layer_entry(d, transpose ? c : r, transpose ? r : c, lr[e], li[e]);
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < MAXQ; ++q) {
                const int e = tid + q * blockDim.x;
                if (e >= MN) break;
                const int i = e / N, j = e % N;
                double sr = accr[q], si = acci[q];
#pragma unroll
                for (int k = 0; k < KC; ++k) {
                    const double ar = vr[i * N + k0 + k], ai = vi[i * N + k0 + k];
                    const double br = lr[k * N + j], bi = li[k * N + j];
                    sr = fma(ar, br, fma(-ai, bi, sr));
                    si = fma(ar, bi, fma(ai, br, si));
                }
                accr[q] = sr;
                acci[q] = si;
            }
        }
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
            const int e = tid + q * blockDim.x;
            if (e < MN) {
                tr[e] = accr[q];
                ti[e] = acci[q];
            }
        }
        cur ^= 1;
        __syncthreads();
    }
    const double* vr = sm + (2 * cur) * MN;
    const double* vi = vr + MN;
    for (int e = tid; e < MN; e += blockDim.x) {
        v_out[e] = vr[e];
        v_out[out_plane + e] = vi[e];
    }
    for (int i = tid; i < R; i += blockDim.x) {
        if (x == nullptr) {
            psi[i] = vr[i * N];
            psi[psi_plane + i] = vi[i * N];
            continue;
        }
        double sr = 0.0, si = 0.0;
        for (int k = 0; k < N; ++k) {
            const double a_r = vr[i * N + k], a_i = vi[i * N + k];
            sr += a_r * x[k] - a_i * x[N + k];
            si += a_r * x[N + k] + a_i * x[k];
        }
        psi[i] = sr;
        psi[psi_plane + i] = si;
    }
}

// 8 <= N <= 64: the whole chain on the FP64 tensor cores, 8 rows of V per CTA.
// The operators of a batch of layers are generated together into shared memory
// (every entry independent: one generation latency per batch, not per layer),
// transposed, LT[n][k]; then each layer is V <- V L with DMMA m8n8k4 (4M):
// warp w owns output columns [8w, 8w + 8) and walks k in steps of 4 on two
// accumulator sets (even / odd steps). Row stride S = N + 4 doubles makes every
// fragment load two wavefronts (the minimum for 32 doubles). Operator entries are
// the bit-exact layer_entry values; only the summation order of products differs
// from the reference's k-sequential loop (within the 1e-10 contract).
constexpr size_t kSmallSmemMax = 227 * 1024;

template <int N>
__host__ __device__ constexpr int small_stride() { return N + 4; }

template <int N>
__host__ __device__ constexpr size_t small_v_bytes() {
    return sizeof(double) * 4 * 8 * static_cast<size_t>(small_stride<N>());  // V, V' (re, im), 8 rows
}

template <int N>
__host__ __device__ constexpr size_t small_op_bytes() {
    // LT re, im + the layer's descriptor (generation reads it from shared memory)
    return sizeof(double) * 2 * N * static_cast<size_t>(small_stride<N>()) + sizeof(SmallLayerDesc);
}

template <int N>
__global__ void __launch_bounds__(1024) small_dmma_kernel(const SmallLayerDesc* __restrict__ layers, int nlayers,
                                                        int batch, int transpose, uint32_t row_begin, int M,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ v_out, double* __restrict__ psi) {
    static_assert(N >= 8 && N <= 64, "DMMA small path: 8 <= N <= 64");
    extern __shared__ __align__(16) double sm[];
    constexpr int S = small_stride<N>();
    constexpr int VP = 8 * S;          // one plane of V
    constexpr int OP = N * S;          // one plane of an operator
    const int cta_row = blockIdx.x * 8;
    row_begin += static_cast<uint32_t>(cta_row);
    const int out_plane = M * N;
    v_out += static_cast<size_t>(cta_row) * N;
    psi += cta_row;
    double* ops = sm + 4 * VP;        // [batch][re | im][N][S]
    SmallLayerDesc* descs = reinterpret_cast<SmallLayerDesc*>(ops + static_cast<size_t>(batch) * 2 * OP);  // [batch]
    static_assert(sizeof(SmallLayerDesc) % 8 == 0, "descriptors are staged in 8-byte words");
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    for (int e = tid; e < 8 * N; e += blockDim.x) {
        const int i = e / N, j = e % N;
        const uint32_t r = row_begin + i, c = j;
        layer_entry(layers[0], transpose ? c : r, transpose ? r : c, sm[i * S + j], sm[VP + i * S + j]);
    }
    int cur = 0;
    for (int l0 = 1; l0 < nlayers; l0 += batch) {
        const int nb = min(batch, nlayers - l0);
        __syncthreads();  // the previous batch's operators are consumed (and V0 is written)
        {
            constexpr int W = static_cast<int>(sizeof(SmallLayerDesc) / 8);
            const unsigned long long* src = reinterpret_cast<const unsigned long long*>(layers + l0);
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(descs);
            for (int w = tid; w < nb * W; w += blockDim.x) dst[w] = __ldg(src + w);
        }
        __syncthreads();
        // Zero the batch's operator planes, then evaluate only the candidate entries:
        // (k, c) can be nonzero only where k and c agree on the layer's zmask, i.e.
        // c = (k & zmask) | (any combination of the free bits) — N 2^f of N^2 entries
        // (f = 1 for a gate or a controlled gate). A group of threads per layer.
        {
            double2* z = reinterpret_cast<double2*>(ops);
            const int nz = nb * OP;  // double2 words of nb x 2 planes
            for (int w = tid; w < nz; w += blockDim.x) z[w] = make_double2(0.0, 0.0);
        }
        __syncthreads();
        {
            const int gsz = static_cast<int>(blockDim.x) / nb;
            const int grp = tid / gsz, gl = tid - grp * gsz;
            if (grp < nb) {
                const SmallLayerDesc& d = descs[grp];
                const uint32_t fmask = ~d.zmask & static_cast<uint32_t>(N - 1);
                const int f = __popc(fmask);
                double* o = ops + static_cast<size_t>(grp) * 2 * OP;
                for (int idx = gl; idx < (N << f); idx += gsz) {
                    const uint32_t k = static_cast<uint32_t>(idx) >> f;
                    uint32_t sub = static_cast<uint32_t>(idx) & ((1u << f) - 1u);
                    uint32_t c = k & ~fmask, fb = fmask;
                    while (fb) {  // deposit sub's bits at fmask's positions
                        const uint32_t lb = fb & (0u - fb);
                        if (sub & 1u) c |= lb;
                        sub >>= 1;
                        fb ^= lb;
                    }
                    double* e = o + c * S + k;
                    // the operand's entry (k, c): L(k, c), or L(c, k) for column blocks (operand L^T)
                    layer_entry(d, transpose ? c : k, transpose ? k : c, e[0], e[OP]);
                }
            }
        }
        __syncthreads();
        for (int b = 0; b < nb; ++b) {
            if (warp < N / 8) {
                const double* ltr = ops + static_cast<size_t>(b) * 2 * OP + (8 * warp + g) * S + t;
                const double* lti = ltr + OP;
                const double* vr = sm + (2 * cur) * VP + g * S + t;
                const double* vi = vr + VP;
                double cr0[2] = {0.0, 0.0}, ci0[2] = {0.0, 0.0}, cr1[2] = {0.0, 0.0}, ci1[2] = {0.0, 0.0};
#pragma unroll
                for (int ks = 0; ks < N / 4; ++ks) {
                    const double ar = vr[4 * ks], ai = vi[4 * ks];
                    const double br = ltr[4 * ks], bi = lti[4 * ks];
                    if (ks & 1) {
                        dmma(cr1, ar, br);
                        dmma(cr1, ai, neg(bi));
                        dmma(ci1, ar, bi);
                        dmma(ci1, ai, br);
                    } else {
                        dmma(cr0, ar, br);
                        dmma(cr0, ai, neg(bi));
                        dmma(ci0, ar, bi);
                        dmma(ci0, ai, br);
                    }
                }
                double* tr = sm + (2 * (cur ^ 1)) * VP + g * S + 8 * warp + 2 * t;
                *reinterpret_cast<double2*>(tr) = make_double2(cr0[0] + cr1[0], cr0[1] + cr1[1]);
                *reinterpret_cast<double2*>(tr + VP) = make_double2(ci0[0] + ci1[0], ci0[1] + ci1[1]);
            }
            cur ^= 1;
            __syncthreads();
        }
    }
    __syncthreads();
    const double* vr = sm + (2 * cur) * VP;
    const double* vi = vr + VP;
    for (int e = tid; e < 8 * N; e += blockDim.x) {
        const int i = e / N, j = e % N;
        v_out[e] = vr[i * S + j];
        v_out[out_plane + e] = vi[i * S + j];
    }
    for (int i = tid; i < 8; i += blockDim.x) {
        if (x == nullptr) {
            psi[i] = vr[i * S];
            psi[M + i] = vi[i * S];
            continue;
        }
        double sr = 0.0, si = 0.0;
        for (int k = 0; k < N; ++k) {
            const double a_r = vr[i * S + k], a_i = vi[i * S + k];
            sr += a_r * x[k] - a_i * x[N + k];
            si += a_r * x[N + k] + a_i * x[k];
        }
        psi[i] = sr;
        psi[M + i] = si;
    }
}

template <int N>
static int launch_small_t(const SmallLayerDesc* d_layers, int nlayers, int transpose, uint32_t row_begin, int M,
                          const double* x, double* v, double* psi, cudaStream_t st) {
    // rows per CTA: 8 from N = 32 (several SMs), all of them below
    const int R = (N >= 32 && M % 8 == 0) ? 8 : M;
    if (N >= 8 && N <= 64 && M % 8 == 0 && !std::getenv("QSB_SMALL_FMA")) {
        constexpr int NT = (N >= 8 && N <= 64) ? N : 8;
        int batch = static_cast<int>((kSmallSmemMax - small_v_bytes<NT>()) / small_op_bytes<NT>());
        batch = std::max(1, std::min(batch, std::max(1, nlayers - 1)));
        const size_t smem = small_v_bytes<NT>() + static_cast<size_t>(batch) * small_op_bytes<NT>();
        small_dmma_kernel<NT><<<M / 8, 1024, smem, st>>>(d_layers, nlayers, batch, transpose, row_begin, M, x, v, psi);
        return static_cast<int>(cudaGetLastError());
    }
    const size_t smem = small_circuit_smem_bytes(R, N);
    int threads = R * N;
    if (threads > 1024) threads = 1024;
    threads = (threads + 31) / 32 * 32;
    small_circuit_kernel<N><<<M / R, threads, smem, st>>>(d_layers, nlayers, transpose, row_begin, M, x, v, psi);
    return static_cast<int>(cudaGetLastError());
}

// K2m: the one-launch chain for N = 64, 128 and 256 (n = 6, 7, 8). Per layer, a
// K2 GEMM of this size is ~15 us of fixed cost (launch, prologue, split-K
// reduction) for < 1 us of DMMA work. Here the whole chain runs in one launch:
// a cluster of CS CTAs owns 8 rows of V; CTA r of the cluster computes output
// columns [r N/CS, (r+1) N/CS) of every layer, generating only those columns of
// the operator (transposed, in shared memory, candidate entries only, in KCH
// k chunks when the columns do not fit whole), K split
// over KSPLIT warp groups whose partials are added in fixed order, and stores
// its 8 x N/CS block of V' into the V' buffer of every CTA of the cluster
// (st.shared::cluster); one cluster barrier per layer hands the full rows over.
// Descriptors are staged in shared memory up front when they fit, else the next
// one is fetched into registers during the DMMAs. DBUF (whole columns, every
// descriptor staged): two operator buffers, the next layer's generated while
// this layer's partials are reduced and stored.
template <int N, int CS, int KSPLIT, int KCH, bool DBUF = false>
struct MidCfg {
    static constexpr int NC = N / CS;               // output columns per CTA
    static constexpr int KC = N / KCH;              // k rows of the operator per generated chunk
    static constexpr int SK = KC + 4;               // operator column stride
    static constexpr int CB = NC / 8;               // 8-column DMMA blocks per CTA
    static constexpr int WARPS = CB * KSPLIT;
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int S = N + 4;                 // row stride (bank-conflict-free fragments)
    static constexpr int VP = 8 * S;                // one plane of V
    static constexpr int OP = NC * SK;              // one plane of the operator chunk's columns
    static constexpr int KS = KC / 4 / KSPLIT;      // m8n8k4 steps per warp per chunk
    static constexpr size_t RED = static_cast<size_t>(KSPLIT - 1) * CB * 32 * 4;  // partials
    static constexpr int NOPS = DBUF ? 2 : 1;       // operator buffers (DBUF: next layer's made early)
    static constexpr size_t BASE = sizeof(double) * (4 * VP + NOPS * 2 * OP + RED);  // + descriptor slots
    static constexpr size_t SMEM = BASE + 2 * sizeof(SmallLayerDesc);          // with a 2-slot ring
    static_assert(THREADS <= 1024 && SMEM <= kSmallSmemMax, "K2m configuration does not fit one SM");
    static_assert(KC % (4 * KSPLIT) == 0 && NC % 8 == 0, "K2m tiling");
    static_assert(!DBUF || KCH == 1, "double-buffered operators: whole columns");
};

__device__ __forceinline__ void st_cluster_v2(uint32_t local_addr, uint32_t rank, double a, double b) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(remote), "d"(a), "d"(b) : "memory");
}

template <int N, int CS, int KSPLIT, int KCH, bool DBUF>
__global__ void __launch_bounds__(MidCfg<N, CS, KSPLIT, KCH, DBUF>::THREADS, 1)
    mid_dmma_kernel(const SmallLayerDesc* __restrict__ layers, int nlayers, int all_staged, int transpose,
                    uint32_t row_begin, int M, const double* __restrict__ x, double* __restrict__ v_out,
                    double* __restrict__ psi, int three_m) {
    using C = MidCfg<N, CS, KSPLIT, KCH, DBUF>;
    constexpr int S = C::S, VP = C::VP, OP = C::OP, NC = C::NC, KC = C::KC, SK = C::SK;
    constexpr int DW = static_cast<int>(sizeof(SmallLayerDesc) / 8);
    static_assert(sizeof(SmallLayerDesc) % 8 == 0, "descriptors move in 8-byte words");
    extern __shared__ __align__(16) double sm[];
    double* ops = sm + 4 * VP;                       // [NOPS][re | im][NC][SK], transposed: (column, k)
    double* red = ops + C::NOPS * 2 * OP;            // [KSPLIT-1][CB][32 lanes][4]
    // descriptor slots: every layer's (all_staged: read once, up front — short chains,
    // where a per-layer fetch would sit on the critical path), or a 2-slot ring
    SmallLayerDesc* descs = reinterpret_cast<SmallLayerDesc*>(red + C::RED);
    const int rank = blockIdx.x;                     // cluster (CS, 1, 1) spans gridDim.x
    const int c0 = rank * NC;
    const int cta_row = blockIdx.y * 8;
    row_begin += static_cast<uint32_t>(cta_row);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int cb = warp % C::CB, kp = warp / C::CB;
    const unsigned long long* lsrc = reinterpret_cast<const unsigned long long*>(layers);
    // V0 = the first operand's rows (every CTA holds full rows); descriptor 1 staged
    for (int e = tid; e < 8 * N; e += C::THREADS) {
        const int i = e / N, j = e % N;
        const uint32_t r = row_begin + i, c = j;
        layer_entry(layers[0], transpose ? c : r, transpose ? r : c, sm[i * S + j], sm[VP + i * S + j]);
    }
    if (all_staged) {
        unsigned long long* dst = reinterpret_cast<unsigned long long*>(descs);
        for (int w = tid; w < nlayers * DW; w += C::THREADS) dst[w] = __ldg(lsrc + w);
    } else if (nlayers > 1 && tid < DW) {
        reinterpret_cast<unsigned long long*>(descs + 1)[tid] = __ldg(lsrc + DW + tid);
    }
    {
        double2* z = reinterpret_cast<double2*>(ops);
        for (int w = tid; w < C::NOPS * OP; w += C::THREADS) z[w] = make_double2(0.0, 0.0);  // 2 planes each
    }
    // The operator buffer is all zeros between chunks: a chunk writes its candidate
    // entries, and after its DMMAs clears just those again (or the whole buffer
    // when the candidates outnumber it) — no full memset per chunk.
    auto candidates = [&](const SmallLayerDesc& d, uint32_t fmask, int f, uint32_t k0, bool clear, double* ob) {
        // candidate entries of this CTA's columns: k agrees with c on zmask (and lies in the chunk)
        for (int idx = tid; idx < (NC << f); idx += C::THREADS) {
            const int cl = idx >> f;
            const uint32_t c = static_cast<uint32_t>(c0 + cl);
            uint32_t sub = static_cast<uint32_t>(idx) & ((1u << f) - 1u);
            uint32_t k = c & ~fmask, fb = fmask;
            while (fb) {
                const uint32_t lb = fb & (0u - fb);
                if (sub & 1u) k |= lb;
                sub >>= 1;
                fb ^= lb;
            }
            if (KCH > 1 && k - k0 >= static_cast<uint32_t>(KC)) continue;
            double* e = ob + cl * SK + (k - k0);
            if (clear) {
                e[0] = 0.0;
                e[OP] = 0.0;
            } else {
                layer_entry(d, transpose ? c : k, transpose ? k : c, e[0], e[OP]);
            }
        }
    };
    auto wipe = [&](const SmallLayerDesc& d, uint32_t fmask, int f, uint32_t k0, double* ob) {
        if ((NC << f) > OP / 2) {
            double2* z = reinterpret_cast<double2*>(ob);
            for (int w = tid; w < OP; w += C::THREADS) z[w] = make_double2(0.0, 0.0);
        } else {
            candidates(d, fmask, f, k0, true, ob);
        }
    };
    auto free_bits = [](const SmallLayerDesc& d) { return ~d.zmask & static_cast<uint32_t>(N - 1); };
    if (DBUF) {  // every descriptor is staged: layer 1's operator is made before the loop
        __syncthreads();
        if (nlayers > 1) {
            const uint32_t fm = free_bits(descs[1]);
            candidates(descs[1], fm, __popc(fm), 0, false, ops + 2 * OP);
        }
    }
    cluster_sync();  // every CTA of the cluster runs before any remote store
    int cur = 0;
    for (int l = 1; l < nlayers; ++l) {
        const SmallLayerDesc& d = descs[all_staged ? l : (l & 1)];
        unsigned long long next = 0;  // descriptor l + 1, in flight during this layer
        if (!all_staged && l + 1 < nlayers && tid < DW) next = __ldg(lsrc + static_cast<size_t>(l + 1) * DW + tid);
        double cr0[2] = {0.0, 0.0}, ci0[2] = {0.0, 0.0}, cr1[2] = {0.0, 0.0}, ci1[2] = {0.0, 0.0};
        double t2a[2] = {0.0, 0.0}, t2b[2] = {0.0, 0.0};  // 3M: the Ai Bi products
        const uint32_t fmask = ~d.zmask & static_cast<uint32_t>(N - 1);
        const int f = __popc(fmask);
        double* ob = DBUF ? ops + (l & 1) * 2 * OP : ops;  // this layer's operator
#pragma unroll 1
        for (int ch = 0; ch < KCH; ++ch) {
            const uint32_t k0 = static_cast<uint32_t>(ch * KC);
            if (!DBUF) {  // (DBUF: made during the previous layer's store phase)
                if (ch > 0) {
                    __syncthreads();  // the previous chunk's operator is consumed
                    wipe(d, fmask, f, k0 - KC, ob);
                    __syncthreads();
                }
                candidates(d, fmask, f, k0, false, ob);
                __syncthreads();
            }
            const int kl = kp * C::KS;  // this warp's k steps within the chunk
            const double* ltr = ob + (8 * cb + g) * SK + t + 4 * kl;
            const double* lti = ltr + OP;
            const double* vr = sm + (2 * cur) * VP + g * S + t + static_cast<int>(k0) + 4 * kl;
            const double* vi = vr + VP;
            if (d.real) {  // exact zero imaginary plane: the products with it add signed zeros
#pragma unroll
                for (int ks = 0; ks < C::KS; ++ks) {
                    const double br = ltr[4 * ks];
                    dmma((ks & 1) ? cr1 : cr0, vr[4 * ks], br);
                    dmma((ks & 1) ? ci1 : ci0, vi[4 * ks], br);
                }
            } else if (three_m) {
                // 3M: T1 += Ar Br, T2 += Ai Bi, T3 += (Ar + Ai)(Br + Bi); Cr = T1 - T2,
                // Ci = T3 - T1 - T2 (the sums in registers: two DADDs for one DMMA less)
#pragma unroll
                for (int ks = 0; ks < C::KS; ++ks) {
                    const double ar = vr[4 * ks], ai = vi[4 * ks];
                    const double br = ltr[4 * ks], bi = lti[4 * ks];
                    dmma((ks & 1) ? cr1 : cr0, ar, br);
                    dmma((ks & 1) ? t2b : t2a, ai, bi);
                    dmma((ks & 1) ? ci1 : ci0, __dadd_rn(ar, ai), __dadd_rn(br, bi));
                }
            } else {
#pragma unroll
                for (int ks = 0; ks < C::KS; ++ks) {
                    const double ar = vr[4 * ks], ai = vi[4 * ks];
                    const double br = ltr[4 * ks], bi = lti[4 * ks];
                    dmma((ks & 1) ? cr1 : cr0, ar, br);
                    dmma((ks & 1) ? cr1 : cr0, ai, neg(bi));
                    dmma((ks & 1) ? ci1 : ci0, ar, bi);
                    dmma((ks & 1) ? ci1 : ci0, ai, br);
                }
            }
        }
        if (three_m && !d.real) {  // (cr, ci) hold (T1, T3): combine with T2
            const double t2[2] = {t2a[0] + t2b[0], t2a[1] + t2b[1]};
            const double t1[2] = {cr0[0] + cr1[0], cr0[1] + cr1[1]};
            const double t3[2] = {ci0[0] + ci1[0], ci0[1] + ci1[1]};
            cr0[0] = t1[0] - t2[0];
            cr0[1] = t1[1] - t2[1];
            ci0[0] = t3[0] - t1[0] - t2[0];
            ci0[1] = t3[1] - t1[1] - t2[1];
            cr1[0] = cr1[1] = ci1[0] = ci1[1] = 0.0;
        }
        double o[4] = {cr0[0] + cr1[0], cr0[1] + cr1[1], ci0[0] + ci1[0], ci0[1] + ci1[1]};
        if (KSPLIT > 1 && kp > 0) {
            double* r = red + ((static_cast<size_t>(kp - 1) * C::CB + cb) * 32 + lane) * 4;
            *reinterpret_cast<double4*>(r) = make_double4(o[0], o[1], o[2], o[3]);
        }
        __syncthreads();  // every DMMA of the layer is done: partials visible, operator free
        wipe(d, fmask, f, static_cast<uint32_t>((KCH - 1) * KC), ob);
        if (DBUF && l + 1 < nlayers) {  // the next layer's operator, into the other buffer
            const uint32_t fm = free_bits(descs[l + 1]);
            candidates(descs[l + 1], fm, __popc(fm), 0, false, ops + ((l + 1) & 1) * 2 * OP);
        }
        if (KSPLIT > 1) {
            if (kp == 0) {
#pragma unroll
                for (int q = 1; q < KSPLIT; ++q) {  // fixed k order: deterministic
                    const double4 p = *reinterpret_cast<const double4*>(
                        red + ((static_cast<size_t>(q - 1) * C::CB + cb) * 32 + lane) * 4);
                    o[0] += p.x;
                    o[1] += p.y;
                    o[2] += p.z;
                    o[3] += p.w;
                }
            }
        }
        if (kp == 0) {
            double* tr = sm + (2 * (cur ^ 1)) * VP + g * S + c0 + 8 * cb + 2 * t;
            const uint32_t ar = static_cast<uint32_t>(__cvta_generic_to_shared(tr));
            const uint32_t ai = static_cast<uint32_t>(__cvta_generic_to_shared(tr + VP));
#pragma unroll
            for (int q = 0; q < CS; ++q) {
                st_cluster_v2(ar, static_cast<uint32_t>(q), o[0], o[1]);
                st_cluster_v2(ai, static_cast<uint32_t>(q), o[2], o[3]);
            }
        }
        if (!all_staged && l + 1 < nlayers && tid < DW)
            reinterpret_cast<unsigned long long*>(descs + ((l + 1) & 1))[tid] = next;
        cluster_sync();  // V' rows complete in every CTA; ops and descs[l & 1] free
        cur ^= 1;
    }
    const double* vr = sm + (2 * cur) * VP;
    const double* vi = vr + VP;
    const int out_plane = M * N;
    for (int e = tid; e < 8 * NC; e += C::THREADS) {
        const int i = e / NC, j = c0 + e % NC;
        v_out[static_cast<size_t>(cta_row + i) * N + j] = vr[i * S + j];
        v_out[out_plane + static_cast<size_t>(cta_row + i) * N + j] = vi[i * S + j];
    }
    if (rank == 0) {
        for (int i = tid; i < 8; i += C::THREADS) {
            if (x == nullptr) {
                psi[cta_row + i] = vr[i * S];
                psi[M + cta_row + i] = vi[i * S];
                continue;
            }
            double sr = 0.0, si = 0.0;
            for (int k = 0; k < N; ++k) {
                const double a_r = vr[i * S + k], a_i = vi[i * S + k];
                sr += a_r * x[k] - a_i * x[N + k];
                si += a_r * x[N + k] + a_i * x[k];
            }
            psi[cta_row + i] = sr;
            psi[M + cta_row + i] = si;
        }
    }
}

// K2m complex layers: 3M (three DMMAs and two DADDs per k-step) or 4M (four DMMAs).
// 3M measured faster where complex layers dominate (QFT-8 264 -> 251 us, QFT-7 77.9 ->
// 75.9 us; real-layer chains unchanged: profiles/R2p_mid3m_ab.txt). QSB_MID_3M=0 / 1.
constexpr int kMid3MDefault = 1;
int mid_three_m() {
    const char* e3 = std::getenv("QSB_MID_3M");
    return e3 && *e3 ? std::atoi(e3) : kMid3MDefault;
}

template <int N, int CS, int KSPLIT, int KCH, bool DBUF = false>
static int launch_mid_t(const SmallLayerDesc* d_layers, int nlayers, int transpose, uint32_t row_begin, int M,
                        const double* x, double* v, double* psi, cudaStream_t st) {
    using C = MidCfg<N, CS, KSPLIT, KCH, DBUF>;
    if (M % 8 != 0) return static_cast<int>(cudaErrorInvalidValue);
    const int all_staged = C::BASE + sizeof(SmallLayerDesc) * static_cast<size_t>(nlayers) <= kSmallSmemMax;
    static_assert(C::THREADS * 8 >= static_cast<int>(sizeof(SmallLayerDesc)), "ring: one word per thread");
    if (DBUF && !all_staged) return static_cast<int>(cudaErrorInvalidValue);  // caller checks mid_dbuf_fits
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, M / 8, 1);
    cfg.blockDim = dim3(C::THREADS, 1, 1);
    cfg.dynamicSmemBytes = all_staged ? C::BASE + sizeof(SmallLayerDesc) * std::max(nlayers, 2) : C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int three_m = mid_three_m();  // complex layers as 3M (1) or 4M (0)
    return static_cast<int>(cudaLaunchKernelEx(&cfg, mid_dmma_kernel<N, CS, KSPLIT, KCH, DBUF>, d_layers, nlayers, all_staged,
                                               transpose, row_begin, M, x, v, psi, three_m));
}

// Fallback configurations (launch_small_circuit picks DBUF / fewer-warp variants
// first). N = 128: clusters of 4 (32 columns per CTA, K over 8 warp groups), 16
// row blocks (clusters of 8 with K over 16 groups measured slower: QFT-7 103 ->
// 178 us, r79). N = 256: clusters of 4 (64 columns per CTA, K over 4 warp groups,
// operator in two k chunks), 32 row blocks: 128 CTAs, one wave.
#define QSB_MID_128 128, 4, 8, 1
#define QSB_MID_256 256, 4, 4, 2
// N = 64: clusters of 2, K over 8 warp groups (2 m8n8k4 steps each). Measured
// against K2s (r76): QFT-6 57.9 -> 57.5 us, DJ-6 22.7 -> 14.5 us; for N <= 32
// K2s's batched generation wins (QFT-4 8.4 vs 16.5 us) and stays.
#define QSB_MID_64 64, 2, 8, 1

// Double-buffered operators (the next layer's generated while this layer's
// partials are reduced and stored: one barrier per layer less) need every
// descriptor staged next to two operator buffers. QSB_MID_NODBUF turns it off.
static bool mid_dbuf(int nlayers, size_t base) {
    return !std::getenv("QSB_MID_NODBUF") &&
           base + sizeof(SmallLayerDesc) * static_cast<size_t>(std::max(nlayers, 2)) <= kSmallSmemMax;
}

int launch_small_circuit(const SmallLayerDesc* d_layers, int nlayers, int max_free_bits, int transpose,
                         uint32_t row_begin, int M, int N, const double* x, double* v, double* psi, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // K2m thread count: DMMA-bound layers run best with few warps (short barriers, small
    // reductions; r82: QFT-8 303 -> 262 us with K over 1 group instead of 4, QFT-7
    // 82 -> 76.5 us with 2 instead of 4), while layers with many candidate entries per
    // operator column (DJ's H on every qubit) need every thread for their generation
    // (DJ-7 22.6 us with 8 groups, 36.9 with 2).
    const bool dense = max_free_bits >= 4;
    switch (N) {
    case 128:
        if (!dense && mid_dbuf(nlayers, MidCfg<128, 4, 2, 1, true>::BASE))
            return launch_mid_t<128, 4, 2, 1, true>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
        if (mid_dbuf(nlayers, MidCfg<128, 4, 8, 1, true>::BASE))
            return launch_mid_t<128, 4, 8, 1, true>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
        if (mid_dbuf(nlayers, MidCfg<128, 4, 4, 1, true>::BASE))
            return launch_mid_t<128, 4, 4, 1, true>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
        return launch_mid_t<QSB_MID_128>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    case 256:
        if (!dense) return launch_mid_t<256, 4, 1, 2>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
        return launch_mid_t<QSB_MID_256>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    default: break;
    }
    const bool classic = std::getenv("QSB_SMALL_CLASSIC") != nullptr;  // K2s instead of K2m
    if (!classic) {
        if (N == 64 && mid_dbuf(nlayers, MidCfg<64, 2, 8, 1, true>::BASE))
            return launch_mid_t<64, 2, 8, 1, true>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
        if (N == 64) return launch_mid_t<QSB_MID_64>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    }
    switch (N) {
    case 2: return launch_small_t<2>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    case 4: return launch_small_t<4>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    case 8: return launch_small_t<8>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    case 16: return launch_small_t<16>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    case 32: return launch_small_t<32>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    case 64: return launch_small_t<64>(d_layers, nlayers, transpose, row_begin, M, x, v, psi, st);
    default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

// ----------------------------------------------------------------------------
// K3: psi = V * x, one warp per row
// ----------------------------------------------------------------------------

__global__ void __launch_bounds__(256) matvec_kernel(const double* __restrict__ v, int M, int N,
                                                     const double* __restrict__ x, double* __restrict__ psi) {
    const int warps = blockDim.x >> 5;
    const int lane = threadIdx.x & 31;
    const size_t plane = static_cast<size_t>(M) * N;
    for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < M; row += gridDim.x * warps) {
        const double2* vr = reinterpret_cast<const double2*>(v + static_cast<size_t>(row) * N);
        const double2* vi = reinterpret_cast<const double2*>(v + plane + static_cast<size_t>(row) * N);
        const double2* xr = reinterpret_cast<const double2*>(x);
        const double2* xi = reinterpret_cast<const double2*>(x + N);
        double sr = 0.0, si = 0.0;
        for (int k = lane; k < N / 2; k += 32) {
            const double2 a = __ldg(vr + k), b = __ldg(vi + k), c = __ldg(xr + k), d = __ldg(xi + k);
            sr += a.x * c.x - b.x * d.x;
            si += a.x * d.x + b.x * c.x;
            sr += a.y * c.y - b.y * d.y;
            si += a.y * d.y + b.y * c.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sr += __shfl_xor_sync(0xffffffffu, sr, o);
            si += __shfl_xor_sync(0xffffffffu, si, o);
        }
        if (lane == 0) {
            psi[row] = sr;
            psi[M + row] = si;
        }
    }
}

// Column blocks: V holds U[:, cols]^T (rows i <-> columns col0 + i of U), so the
// shard's share of psi = U psi0 is psi[k] = sum_i V[i][k] x[col0 + i] over the rows
// [i0, i0 + count) of the shard; one thread per k (coalesced over k), i ascending.
__global__ void __launch_bounds__(256) matvec_t_kernel(const double* __restrict__ v, int M, int N, int i0, int count,
                                                       int col0, const double* __restrict__ x,
                                                       double* __restrict__ psi) {
    const size_t plane = static_cast<size_t>(M) * N;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
        double sr = 0.0, si = 0.0;
        for (int i = i0; i < i0 + count; ++i) {
            const double ar = v[static_cast<size_t>(i) * N + k], ai = v[plane + static_cast<size_t>(i) * N + k];
            const double xr = x[col0 + i - i0], xi = x[N + col0 + i - i0];
            sr += ar * xr - ai * xi;
            si += ar * xi + ai * xr;
        }
        psi[k] = sr;
        psi[N + k] = si;
    }
}

int launch_matvec_t(const double* v, int M, int N, int i0, int count, int col0, const double* x, double* psi,
                    void* stream) {
    int blocks = (N + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    matvec_t_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(v, M, N, i0, count, col0, x, psi);
    return static_cast<int>(cudaGetLastError());
}

int launch_matvec(const double* v, int M, int N, const double* x, double* psi, void* stream) {
    int blocks = (M + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    matvec_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(v, M, N, x, psi);
    return static_cast<int>(cudaGetLastError());
}

// ----------------------------------------------------------------------------
// K4: probabilities + deterministic norm
// ----------------------------------------------------------------------------

__global__ void __launch_bounds__(256) probs_kernel(const double* __restrict__ psi, int64_t dim,
                                                    double* __restrict__ p, double* __restrict__ partial) {
    __shared__ double warp_sums[8];
    double s = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < dim;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double re = psi[i], im = psi[dim + i];
        const double v = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
        p[i] = v;
        s += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = threadIdx.x < (blockDim.x >> 5) ? warp_sums[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (threadIdx.x == 0) partial[blockIdx.x] = w;
    }
}

__global__ void reduce_partials_kernel(const double* __restrict__ partial, int n, double* __restrict__ out) {
    __shared__ double warp_sums[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double w = threadIdx.x < (blockDim.x >> 5) ? warp_sums[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if (threadIdx.x == 0) out[0] = w;
    }
}

int launch_probabilities(const double* psi, int64_t dim, double* p, double* partial, int partial_cap,
                         double* norm, void* stream) {
    int blocks = static_cast<int>((dim + 255) / 256);
    if (blocks > partial_cap) blocks = partial_cap;
    if (blocks < 1) blocks = 1;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    probs_kernel<<<blocks, 256, 0, s>>>(psi, dim, p, partial);
    reduce_partials_kernel<<<1, 1024, 0, s>>>(partial, blocks, norm);
    return static_cast<int>(cudaGetLastError());
}

template <int N>
static int configure_small_t() {
    return static_cast<int>(cudaFuncSetAttribute(small_dmma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kSmallSmemMax)));
}

template <int N, int CS, int KSPLIT, int KCH, bool DBUF = false>
static int configure_mid_t() {
    return static_cast<int>(cudaFuncSetAttribute(mid_dmma_kernel<N, CS, KSPLIT, KCH, DBUF>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kSmallSmemMax)));
}

// Kernel attributes, set once per device before any launch or graph capture.
int configure_kernels() {
    int e;
    if ((e = configure_zgemm_t<128, 64>())) return e;
    if ((e = configure_zgemm_t<64, 64>())) return e;
    if ((e = configure_zgemm_t<32, 32>())) return e;
    if ((e = configure_ws_t<false, false>())) return e;
    if ((e = configure_ws_t<true, false>())) return e;
    if ((e = configure_ws_t<true, true>())) return e;
    if ((e = static_cast<int>(cudaFuncSetAttribute(zgemm_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   ChainCfg::SMEM))))
        return e;
    query_ws_clusters();
    if ((e = configure_small_t<8>()) || (e = configure_small_t<16>()) || (e = configure_small_t<32>()) ||
        (e = configure_small_t<64>()))
        return e;
    if ((e = configure_mid_t<QSB_MID_64>()) || (e = configure_mid_t<QSB_MID_128>()) ||
        (e = configure_mid_t<QSB_MID_256>()) || (e = configure_mid_t<64, 2, 8, 1, true>()) ||
        (e = configure_mid_t<128, 4, 8, 1, true>()) || (e = configure_mid_t<128, 4, 4, 1, true>()) ||
        (e = configure_mid_t<256, 4, 1, 2>()) || (e = configure_mid_t<128, 4, 2, 1, true>()))
        return e;
    if ((e = static_cast<int>(cudaFuncSetAttribute(small_circuit_kernel<32>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024))))
        return e;
    if ((e = static_cast<int>(cudaFuncSetAttribute(small_circuit_kernel<64>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(small_circuit_smem_bytes(8, 64))))))
        return e;
    return 0;
}

}  // namespace qsb
