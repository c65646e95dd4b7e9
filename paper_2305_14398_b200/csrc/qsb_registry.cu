// qsb_registry.cu — registry validation on the GPU:
// is_unitary(A, tol) = max_ij |(A^H A - I)_ij| <= tol, the O(N^3) check
// GateRegistry::register_function runs on every registered matrix
// (gates.cpp:112-125 -> linalg.cpp:131-155; the DJ oracle is 2^n x 2^n).
//
//   transpose_kernel   T = A^T (both planes; 32x32 shared-memory tiles), so
//                      both Gram operands are K-major rows of T
//   gram_kernel        G = conj(T) T^T on the DMMA pipe (mma.sync m8n8k4 f64),
//                      both tiles staged by TMA (SWIZZLE_128B, mbarrier
//                      pipeline), upper-triangular tile pairs only (G is
//                      Hermitian: |G_ji| = |G_ij|); the epilogue reduces
//                      max(|Re G_ij - d_ij|, |Im G_ij|) and never writes G
//   gram_small_kernel  N < 64: one thread per entry, the reference's loop
//
// The reference's verdict is "every |entry| <= tol" (linalg.cpp:145-151); the
// maximum deviation is the same test. NaN entries fail no comparison there and
// are skipped by fmax here.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace qsb {

namespace reg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
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

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar, int c0, int c1, int c2) {
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

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(c[0]), "+d"(c[1])
        : "d"(a), "d"(b));
}

__device__ __forceinline__ double neg(double x) {
    return __longlong_as_double(__double_as_longlong(x) ^ static_cast<long long>(0x8000000000000000ULL));
}

// Non-negative doubles order like their bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
    atomicMax(p, static_cast<unsigned long long>(__double_as_longlong(v)));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

constexpr int BT = 64;  // tile rows = cols
constexpr int BK = 16;  // one 128-byte swizzle line of doubles
constexpr int STAGES = 4;
constexpr int TILE_BYTES = 2 * BT * BK * 8;  // re + im planes
constexpr int STAGE_BYTES = 2 * TILE_BYTES;  // A and B tiles
constexpr int THREADS = 128;                 // 4 warps, 2 x 2 warp tiles of 32 x 32
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 64;

__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ re, const double* __restrict__ im,
                                                      double* __restrict__ t, int N) {
    __shared__ double tile[2][32][33];
    const size_t plane = static_cast<size_t>(N) * N;
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        tile[0][r][threadIdx.x] = re[static_cast<size_t>(by + r) * N + bx + threadIdx.x];
        tile[1][r][threadIdx.x] = im[static_cast<size_t>(by + r) * N + bx + threadIdx.x];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        t[static_cast<size_t>(bx + r) * N + by + threadIdx.x] = tile[0][threadIdx.x][r];
        t[plane + static_cast<size_t>(bx + r) * N + by + threadIdx.x] = tile[1][threadIdx.x][r];
    }
}

// G tile (bi, bj), bi <= bj, of conj(T) T^T: G_ij = sum_k conj(T_ik) T_jk.
// Smem tiles are [plane][rows][16 doubles] with the TMA 128-byte swizzle; lane
// (g, t) reads chunks 2t, 2t+1 of line g (k-permutation 4t + s for both operands).
__global__ void __launch_bounds__(THREADS, 1) gram_kernel(const __grid_constant__ CUtensorMap tmT, int N,
                                                         unsigned long long* __restrict__ maxdev) {
    const int bi = blockIdx.y, bj = blockIdx.x;
    if (bi > bj) return;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sBase = smem_u32(smem);
    const uint32_t sBar = sBase + STAGES * STAGE_BYTES;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;
    const int m0 = bi * BT, n0 = bj * BT;
    const int KT = N / BK;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(sBar + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int kt) {
        const int s = kt % STAGES;
        const uint32_t st = sBase + s * STAGE_BYTES;
        mbar_expect_tx(sBar + 8 * s, STAGE_BYTES);
        tma_load_3d(st, &tmT, sBar + 8 * s, kt * BK, m0, 0);
        tma_load_3d(st + TILE_BYTES, &tmT, sBar + 8 * s, kt * BK, n0, 0);
    };
    double gr[4][4][2], gi[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) gr[i][j][0] = gr[i][j][1] = gi[i][j][0] = gi[i][j][1] = 0.0;
    if (tid == 0)
        for (int kt = 0; kt < STAGES - 1 && kt < KT; ++kt) issue(kt);
    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        mbar_wait(sBar + 8 * s, (kt / STAGES) & 1);
        const uint32_t aRe = sBase + s * STAGE_BYTES, aIm = aRe + BT * 128;
        const uint32_t bRe = aRe + TILE_BYTES, bIm = bRe + BT * 128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t choff = static_cast<uint32_t>(((2 * t + h) ^ g) << 4);
            double2 ar[4], ai[4], br[4], bi2[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t line = static_cast<uint32_t>(wm * 32 + i * 8 + g) * 128 + choff;
                ar[i] = lds128(aRe + line);
                ai[i] = lds128(aIm + line);
                const uint32_t lb = static_cast<uint32_t>(wn * 32 + i * 8 + g) * 128 + choff;
                br[i] = lds128(bRe + lb);
                bi2[i] = lds128(bIm + lb);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double xr = e ? ar[i].y : ar[i].x, xi = e ? ai[i].y : ai[i].x;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double yr = e ? br[j].y : br[j].x, yi = e ? bi2[j].y : bi2[j].x;
                        // conj(x) y = (xr yr + xi yi) + i (xr yi - xi yr)
                        dmma(gr[i][j], xr, yr);
                        dmma(gr[i][j], xi, yi);
                        dmma(gi[i][j], xr, yi);
                        dmma(gi[i][j], neg(xi), yr);
                    }
                }
        }
        __syncthreads();  // every warp is done with stage s before it is refilled
        if (tid == 0 && kt + STAGES - 1 < KT) issue(kt + STAGES - 1);
    }
    double dev = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + wm * 32 + i * 8 + g;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + wn * 32 + j * 8 + 2 * t + e;
                const double d = gr[i][j][e] - (row == col ? 1.0 : 0.0);
                dev = fmax(dev, fmax(fabs(d), fabs(gi[i][j][e])));
            }
    }
    dev = warp_max(dev);
    if (lane == 0) atomic_max_nonneg(maxdev, dev);
}

// Dimensions that are not a multiple of the 64-wide tile (N < 64 for the
// power-of-two registry matrices): the reference's triple loop (linalg.cpp:138-151),
// one thread per entry, 64-bit indices, every product and sum separately rounded
// in the reference's order (x86-64 without FMA contraction), so a verdict at the
// tolerance boundary is the reference's.
__global__ void gram_small_kernel(const double* __restrict__ re, const double* __restrict__ im, int64_t N,
                                  unsigned long long* __restrict__ maxdev) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double dev = 0.0;
    if (idx < N * N) {
        const int64_t i = idx / N, j = idx % N;
        double sr = 0.0, si = 0.0;
        for (int64_t k = 0; k < N; ++k) {
            const double air = re[k * N + i], aii = im[k * N + i], ajr = re[k * N + j], aji = im[k * N + j];
            sr = __dadd_rn(sr, __dadd_rn(__dmul_rn(air, ajr), __dmul_rn(aii, aji)));
            si = __dadd_rn(si, __dsub_rn(__dmul_rn(air, aji), __dmul_rn(aii, ajr)));
        }
        if (i == j) sr = __dsub_rn(sr, 1.0);
        dev = fmax(fabs(sr), fabs(si));
    }
    dev = warp_max(dev);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(maxdev, dev);
}

}  // namespace reg

int registry_configure() {
    return static_cast<int>(
        cudaFuncSetAttribute(reg::gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, reg::SMEM));
}

int gram_tile() { return reg::BT; }

int launch_transpose(const double* re, const double* im, double* t, int N, void* stream) {
    dim3 grid(N / 32, N / 32), block(32, 8);
    reg::transpose_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(re, im, t, N);
    return static_cast<int>(cudaGetLastError());
}

int launch_gram(const void* tmapT, int N, unsigned long long* maxdev, void* stream) {
    const int T = N / reg::BT;
    dim3 grid(T, T);
    reg::gram_kernel<<<grid, reg::THREADS, reg::SMEM, static_cast<cudaStream_t>(stream)>>>(
        *static_cast<const CUtensorMap*>(tmapT), N, maxdev);
    return static_cast<int>(cudaGetLastError());
}

int launch_gram_small(const double* re, const double* im, int N, unsigned long long* maxdev, void* stream) {
    const int64_t blocks = (static_cast<int64_t>(N) * N + 255) / 256;
    if (blocks > 0x7fffffff) return static_cast<int>(cudaErrorInvalidValue);
    reg::gram_small_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        re, im, static_cast<int64_t>(N), maxdev);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace qsb
