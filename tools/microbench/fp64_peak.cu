// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA vs cuBLAS ZGEMM/DGEMM.
// Used once to fix the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int ACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dmma16_loop(double* out, int iters) {
  // m16n8k16: A 8 regs(doubles), B 4, C 4
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
  double c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[0] = s;
}

template <int ACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-9;
  double c[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
double time_kernel(K kernel, int blocks, int threads, int iters, double flop_per_thread_iter, double* d) {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kernel<<<blocks, threads>>>(d, iters); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0)); kernel<<<blocks, threads>>>(d, iters); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
  }
  return flop_per_thread_iter * (double)blocks * threads * iters / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms %d clock(kHz) %d\n", p.name, p.multiProcessorCount, p.clockRate);
  double* d; CK(cudaMalloc(&d, 64));
  int sms = p.multiProcessorCount;
  // DMMA m8n8k4: per warp 512 FLOP per mma -> per thread 16 FLOP per mma
  for (int threads : {128, 256, 512}) {
    printf("dmma m8n8k4   acc8  blocks %d x %d threads: %.2f TFLOP/s\n", sms * 2, threads,
           time_kernel(dmma_loop<8>, sms * 2, threads, 20000, 8 * 16.0, d));
    printf("dmma m8n8k4   acc16 blocks %d x %d threads: %.2f TFLOP/s\n", sms * 2, threads,
           time_kernel(dmma_loop<16>, sms * 2, threads, 10000, 16 * 16.0, d));
    printf("dmma m16n8k16 acc4  blocks %d x %d threads: %.2f TFLOP/s\n", sms * 2, threads,
           time_kernel(dmma16_loop<4>, sms * 2, threads, 5000, 4 * 2.0 * 16 * 8 * 16 / 32.0, d));
    printf("dfma          acc8  blocks %d x %d threads: %.2f TFLOP/s\n", sms * 2, threads,
           time_kernel(dfma_loop<8>, sms * 2, threads, 20000, 8 * 2.0, d));
  }
  cublasHandle_t h; cublasCreate(&h);
  for (int n : {2048, 4096, 8192}) {
    size_t bytes = (size_t)n * n * 16;
    void *A, *B, *C; CK(cudaMalloc(&A, bytes)); CK(cudaMalloc(&B, bytes)); CK(cudaMalloc(&C, bytes));
    CK(cudaMemset(A, 0, bytes)); CK(cudaMemset(B, 0, bytes));
    cuDoubleComplex one = {1, 0}, zero = {0, 0};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
      auto run = [&]() {
        if (mode == 0) cublasZgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, (cuDoubleComplex*)A, n, (cuDoubleComplex*)B, n, &zero, (cuDoubleComplex*)C, n);
        else if (mode == 1) cublasZgemm3m(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, (cuDoubleComplex*)A, n, (cuDoubleComplex*)B, n, &zero, (cuDoubleComplex*)C, n);
        else { double o = 1, z = 0; cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &o, (double*)A, n, (double*)B, n, &z, (double*)C, n); }
      };
      run(); CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) { cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
      double flop = (mode < 2 ? 8.0 : 2.0) * n * (double)n * n;
      printf("cublas %s n=%d: %.3f ms  %.2f TFLOP/s (credited %s)\n", mode == 0 ? "Zgemm" : mode == 1 ? "Zgemm3m" : "Dgemm", n, best, flop / (best * 1e-3) / 1e12, mode < 2 ? "8N^3" : "2N^3");
    }
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  return 0;
}
