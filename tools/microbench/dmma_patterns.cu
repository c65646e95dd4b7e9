// Which consumer-loop pattern keeps the DMMA pipe busy? Each variant runs the
// inner loop of a K2 consumer warp on fixed shared-memory tiles (no producer),
// 8 consumer warps per CTA, 1 CTA per SM. Reports DMMA-pipe TFLOP/s (DMMA
// count x 512 FLOP) and the per-warp instruction mix.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;} } while (0)

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds128(unsigned addr) {
  double2 v; asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr)); return v;
}

// MI x NI tiles per warp, NACC accumulator sets, PL A-planes & B-planes loaded, DADD for sum plane
template <int MI, int NI, int NACC, int APL, int BPL, bool ADD, bool LOADS>
__global__ void __launch_bounds__(256, 1) pattern(double* out, int iters) {
  __shared__ __align__(16) double sm[6 * 64 * 16];
  for (int i = threadIdx.x; i < 6 * 64 * 16; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[NACC][MI][NI][2];
#pragma unroll
  for (int a = 0; a < NACC; ++a)
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) acc[a][i][j][0] = acc[a][i][j][1] = 0;
  double2 A[APL][MI], B[BPL][NI];
#pragma unroll
  for (int p = 0; p < APL; ++p)
#pragma unroll
    for (int i = 0; i < MI; ++i) A[p][i] = lds128(base + ((p * 64 + i * 8 + g) * 128) + (((2 * t) ^ g) << 4));
#pragma unroll
  for (int p = 0; p < BPL; ++p)
#pragma unroll
    for (int j = 0; j < NI; ++j) B[p][j] = lds128(base + 3 * 64 * 128 + ((p * 64 + j * 8 + g) * 128) + (((2 * t) ^ g) << 4));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (LOADS) {
        const unsigned ch = ((2 * t + h) ^ g) << 4;
#pragma unroll
        for (int p = 0; p < APL; ++p)
#pragma unroll
          for (int i = 0; i < MI; ++i) A[p][i] = lds128(base + ((p * 64 + i * 8 + g) * 128) + ch);
#pragma unroll
        for (int p = 0; p < BPL; ++p)
#pragma unroll
          for (int j = 0; j < NI; ++j) B[p][j] = lds128(base + 3 * 64 * 128 + ((p * 64 + j * 8 + g) * 128) + ch);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double x[3][MI], y[3][NI];
#pragma unroll
        for (int p = 0; p < 3; ++p) {
#pragma unroll
          for (int i = 0; i < MI; ++i) x[p][i] = p < APL ? (e ? A[p][i].y : A[p][i].x) : 0.0;
#pragma unroll
          for (int j = 0; j < NI; ++j) y[p][j] = p < BPL ? (e ? B[p][j].y : B[p][j].x) : 0.0;
        }
        if (ADD) {
#pragma unroll
          for (int i = 0; i < MI; ++i) x[2][i] = x[0][i] + x[1][i];
        }
#pragma unroll
        for (int a = 0; a < NACC; ++a)
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NI; ++j) dmma(acc[a][i][j], x[a % 3][i], y[a % 3][j]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < NACC; ++a)
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) s += acc[a][i][j][0] + acc[a][i][j][1];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
int run(const char* name, K k, int dmma_per_iter) {
  double* d; CK(cudaMalloc(&d, 64));
  int iters = 2000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148, 256>>>(d, iters); CK(cudaDeviceSynchronize());
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); k<<<148, 256>>>(d, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 512.0 * dmma_per_iter * iters * 8.0 * 148;
  printf("%-48s %7.2f TFLOP/s (DMMA pipe)\n", name, flops / (best * 1e-3) / 1e12);
  cudaFree(d);
  return 0;
}

int main() {
  // dmma per iter per warp = NACC * MI * NI * 4 (2 h x 2 e)
  run("4M 4x4 (2 acc, 2+2 planes, loads)", pattern<4, 4, 2, 2, 2, false, true>, 2 * 16 * 4 * 2);
  run("4M 4x4 as 4 products (4 acc-equiv uses)", pattern<4, 4, 4, 2, 2, false, true>, 4 * 16 * 4);
  run("3M 4x2 (3 acc, A 2pl+DADD, B 3pl, loads)", pattern<4, 2, 3, 2, 3, true, true>, 3 * 8 * 4);
  run("3M 4x2 (3 acc, A 3pl, B 3pl, loads, no DADD)", pattern<4, 2, 3, 3, 3, false, true>, 3 * 8 * 4);
  run("3M 4x2 no loads, DADD", pattern<4, 2, 3, 2, 3, true, false>, 3 * 8 * 4);
  run("3M 4x2 no loads, no DADD", pattern<4, 2, 3, 3, 3, false, false>, 3 * 8 * 4);
  run("3M 2x4 (3 acc, loads, DADD)", pattern<2, 4, 3, 2, 3, true, true>, 3 * 8 * 4);
  run("3M 2x4 no loads no DADD", pattern<2, 4, 3, 3, 3, false, false>, 3 * 8 * 4);
  run("3M 4x3 (3 acc, loads, DADD)", pattern<4, 3, 3, 2, 3, true, true>, 3 * 12 * 4);
  run("3M 4x4 (3 acc, loads, no DADD) [192 acc regs]", pattern<4, 4, 3, 3, 3, false, true>, 3 * 16 * 4);
  run("2 acc 4x2 no loads", pattern<4, 2, 2, 3, 3, false, false>, 2 * 8 * 4);
  run("4 acc 4x2 no loads", pattern<4, 2, 4, 3, 3, false, false>, 4 * 8 * 4);
  return 0;
}
