// HBM bandwidth of the p=1 stage kernel's access pattern: each thread (one element) reads R rows
// of a [R][ld] SoA array (coalesced across elements, rows ld apart) and writes R rows, grid-stride
// like k_element (592 blocks x 128 threads); compared with the same bytes in an AoSoA layout
// [ld/32][R][32] (each warp's rows contiguous) and with a plain contiguous copy.
#include <cstdio>
#include <cuda_runtime.h>

template <int R, bool AOSOA>
__global__ void __launch_bounds__(128, 4) k_rows(const double* __restrict__ in, double* __restrict__ out, int n, long long ld) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    double v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long i = AOSOA ? (static_cast<long long>(e >> 5) * R + r) * 32 + (e & 31) : r * ld + e;
      v[r] = __ldg(in + i);
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s = fma(v[r], 1.0000001, s);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long i = AOSOA ? (static_cast<long long>(e >> 5) * R + r) * 32 + (e & 31) : r * ld + e;
      out[i] = v[r] + s * 1e-30;
    }
  }
}

template <class K>
float timeit(K k, int grid, const double* a, double* b, int n, long long ld) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<<<grid, 128>>>(a, b, n, ld);
  float best = 1e9;
  for (int it = 0; it < 10; ++it) {
    cudaEventRecord(e0);
    k<<<grid, 128>>>(a, b, n, ld);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const int n = 1002528;
  const long long ld = (n + 31) / 32 * 32;
  const int R = 12;
  double *a, *b;
  cudaMalloc(&a, R * ld * 8);
  cudaMalloc(&b, R * ld * 8);
  cudaMemset(a, 0, R * ld * 8);
  const double gb = 2.0 * R * n * 8 / 1e9;
  for (int grid : {592, 1184, 2368, 7832}) {
    const float t0 = timeit(k_rows<R, false>, grid, a, b, n, ld);
    const float t1 = timeit(k_rows<R, true>, grid, a, b, n, ld);
    printf("grid %5d  SoA [12][ld]: %.4f ms %.0f GB/s   AoSoA [ld/32][12][32]: %.4f ms %.0f GB/s\n", grid, t0,
           gb / (t0 * 1e-3), t1, gb / (t1 * 1e-3));
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
