// Does compute-sanitizer racecheck model mbarrier arrive / wait ordering?
// Thread 0 of warp 1 writes shared memory and arrives (release.cta) on an mbarrier of
// count 1; the threads of warp 0 wait on it (acquire.cta, try_wait.parity) and read.
// Correct by the PTX memory model. Variant 1 writes from all 32 lanes of warp 1 and
// lets lane 0 arrive after __syncwarp() — the K2 producer's publication pattern.
// Any hazard racecheck reports here is a hazard it reports for correct code.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(bar), "r"(parity) : "memory");
}

__global__ void k(int variant, double* out) {
    __shared__ double buf[64];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        mbar_init(b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 1) {
        if (variant == 0) {
            if (lane == 0) {
                for (int i = 0; i < 64; ++i) buf[i] = i;
                mbar_arrive(b);
            }
        } else {
            buf[lane] = lane;
            buf[lane + 32] = lane + 32;
            __syncwarp();
            if (lane == 0) mbar_arrive(b);
        }
    } else {
        mbar_wait(b, 0);
        out[threadIdx.x] = buf[lane] + buf[lane + 32];
    }
}

int main() {
    double* d;
    cudaMalloc(&d, 64 * sizeof(double));
    for (int v = 0; v < 2; ++v) {
        k<<<1, 64>>>(v, d);
        cudaError_t e = cudaDeviceSynchronize();
        double h[32];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        std::printf("variant %d: %s, out[5] = %g (expect 42)\n", v, cudaGetErrorString(e), h[5]);
    }
    return 0;
}
