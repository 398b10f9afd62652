// Microbenchmark: FP64 DFMA pipe vs DMMA (mma.sync f64) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 1.0000001, 1e-9);
  double s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}

// m8n8k4: A 1 double, B 1 double, C/D 2 doubles per thread.
__global__ void k_dmma884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[8][2];
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (s == 1.2345) out[0] = s;
}

// one dependent DMMA chain per warp (latency probe) and two chains
template <int CH>
__global__ void k_dmma_chain(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[CH][2];
  for (int k = 0; k < CH; ++k) d[k][0] = d[k][1] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CH; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < CH; ++k) s += d[k][0] + d[k][1];
  if (s == 1.2345) out[0] = s;
}

// m16n8k4: A 2 doubles, B 1, C/D 4.
__global__ void k_dmma1684(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double d[4][4];
  for (int k = 0; k < 4; ++k) d[k][0] = d[k][1] = d[k][2] = d[k][3] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(d[k][0]), "+d"(d[k][1]), "+d"(d[k][2]), "+d"(d[k][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
  if (s == 1.2345) out[0] = s;
}

// m16n8k16: A 8 doubles, B 4, C/D 4.
__global__ void k_dmma16816(double* out, int iters) {
  double a[8], b[4];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < 4; ++k) b[k] = 1.0 - threadIdx.x * 1e-4 * k;
  double d[4][4];
  for (int k = 0; k < 4; ++k) d[k][0] = d[k][1] = d[k][2] = d[k][3] = k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(d[k][0]), "+d"(d[k][1]), "+d"(d[k][2]), "+d"(d[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
  if (s == 1.2345) out[0] = s;
}

// DDIV / DSQRT throughput (IEEE, as in the flux)
__global__ void k_div(double* out, int iters) {
  double a[4];
  for (int k = 0; k < 4; ++k) a[k] = 1.5 + threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = 1.0 / a[k] + 1.0;
  double s = 0;
  for (int k = 0; k < 4; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_sqrt(double* out, int iters) {
  double a[4];
  for (int k = 0; k < 4; ++k) a[k] = 1.5 + threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = sqrt(a[k]) + 1.0;
  double s = 0;
  for (int k = 0; k < 4; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}

template <class K>
float timeit(K k, int blocks, int threads, int iters, double* d) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<blocks, threads>>>(d, 16);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k<<<blocks, threads>>>(d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int it = 4096;
  // warps per SM sub-partition: 1, 2, 4 (one block per SM) and the saturated case
  for (int wpb : {4, 8, 16, 32}) {
    int blocks = sms, threads = 32 * wpb;
    double n = double(blocks) * threads;
    float t = timeit(k_dfma, blocks, threads, it, d);
    printf("warps/blk %2d  DFMA      %.2f TFLOP/s\n", wpb, 2.0 * 8 * it * n / (t * 1e-3) / 1e12);
    t = timeit(k_dmma884, blocks, threads, it, d);
    printf("warps/blk %2d  DMMA 884  %.2f TFLOP/s\n", wpb, 2.0 * 8 * it * (n / 32) * 256 / (t * 1e-3) / 1e12);
    t = timeit(k_dmma1684, blocks, threads, it, d);
    printf("warps/blk %2d  DMMA 1684 %.2f TFLOP/s\n", wpb, 2.0 * 4 * it * (n / 32) * 512 / (t * 1e-3) / 1e12);
    t = timeit(k_dmma16816, blocks, threads, it, d);
    printf("warps/blk %2d  DMMA16816 %.2f TFLOP/s\n", wpb, 2.0 * 4 * it * (n / 32) * 2048 / (t * 1e-3) / 1e12);
    t = timeit(k_dmma_chain<1>, blocks, threads, it, d);
    printf("warps/blk %2d  DMMA 1 chain  %.2f TFLOP/s  (%.1f cycles per DMMA per warp at 1.965 GHz)\n", wpb,
           2.0 * it * (n / 32) * 256 / (t * 1e-3) / 1e12, t * 1e-3 * 1.965e9 / it);
    t = timeit(k_dmma_chain<2>, blocks, threads, it, d);
    printf("warps/blk %2d  DMMA 2 chains %.2f TFLOP/s\n", wpb, 2.0 * 2 * it * (n / 32) * 256 / (t * 1e-3) / 1e12);
    t = timeit(k_dmma_chain<4>, blocks, threads, it, d);
    printf("warps/blk %2d  DMMA 4 chains %.2f TFLOP/s\n", wpb, 2.0 * 4 * it * (n / 32) * 256 / (t * 1e-3) / 1e12);
    t = timeit(k_div, blocks, threads, it, d);
    printf("warps/blk %2d  DDIV      %.3f Gop/s (%.1f DFMA-equiv)\n", wpb, 4.0 * it * n / (t * 1e-3) / 1e9, 0.0);
    t = timeit(k_sqrt, blocks, threads, it, d);
    printf("warps/blk %2d  DSQRT     %.3f Gop/s\n", wpb, 4.0 * it * n / (t * 1e-3) / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
}
