// Precision of the MUFU double seeds (rcp.approx.ftz.f64, rsqrt.approx.ftz.f64) and of the
// Newton-refined reciprocal / square root variants used by the flux (element_impl.cuh), against
// IEEE 1/x and sqrt(x) over log-uniform arguments in [1e-6, 1e6].
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__device__ double rcp_seed(double x) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ double rsq_seed(double x) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ double sqrt_it(double a, int iters) {
  double y = rsq_seed(a);
  const double h = 0.5 * a;
  for (int i = 0; i < iters; ++i) y = y * fma(-h * y, y, 1.5);
  const double s = a * y;
  return fma(0.5 * y, fma(-s, s, a), s);
}
__device__ double rcp_it(double x, int iters) {
  double r = rcp_seed(x);
  for (int i = 0; i < iters; ++i) { double e = fma(-x, r, 1.0); r = fma(r, e, r); }
  return r;
}
__device__ unsigned long long ulps(double a, double b) {
  long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  return x > y ? x - y : y - x;
}
__global__ void k(unsigned long long n, unsigned long long* out, double* relmax) {
  unsigned long long s = 0x9e3779b97f4a7c15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  double rs = 0, rr = 0;
  unsigned long long u1 = 0, u2 = 0, r1 = 0, r2 = 0, d1 = 0, d2 = 0;
  for (unsigned long long i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double t = (s >> 11) * (1.0 / 9007199254740992.0);
    const double x = exp((t * 2 - 1) * 13.8);
    rs = fmax(rs, fabs(rsq_seed(x) * sqrt(x) - 1.0));
    rr = fmax(rr, fabs(rcp_seed(x) * x - 1.0));
    const double sq = sqrt(x), rc = 1.0 / x;
    const unsigned long long a1 = ulps(sqrt_it(x, 1), sq), a2 = ulps(sqrt_it(x, 2), sq);
    const unsigned long long b1 = ulps(rcp_it(x, 1), rc), b2 = ulps(rcp_it(x, 2), rc);
    u1 = max(u1, a1); u2 = max(u2, a2); r1 = max(r1, b1); r2 = max(r2, b2);
    d1 += a1 != 0; d2 += a2 != 0;
  }
  atomicMax(out + 0, u1); atomicMax(out + 1, u2); atomicMax(out + 2, r1); atomicMax(out + 3, r2);
  atomicAdd(out + 4, d1); atomicAdd(out + 5, d2);
  atomicMax(reinterpret_cast<unsigned long long*>(relmax), __double_as_longlong(rs));
  atomicMax(reinterpret_cast<unsigned long long*>(relmax + 1), __double_as_longlong(rr));
}
int main() {
  unsigned long long* o; double* r;
  cudaMallocManaged(&o, 6 * 8); cudaMallocManaged(&r, 2 * 8);
  for (int i = 0; i < 6; ++i) o[i] = 0;
  r[0] = r[1] = 0;
  const unsigned long long n = 4096;
  k<<<1184, 256>>>(n, o, r);
  cudaDeviceSynchronize();
  const double total = 1184.0 * 256 * n;
  printf("samples %.3g\n", total);
  printf("rsqrt seed max rel err %.3e (2^%.1f)\n", r[0], log2(r[0]));
  printf("rcp   seed max rel err %.3e (2^%.1f)\n", r[1], log2(r[1]));
  printf("sqrt_nr 1 rsqrt iteration + correction: max %llu ulp, %.3g%% differ from IEEE sqrt\n", o[0], 100.0 * o[4] / total);
  printf("sqrt_nr 2 rsqrt iterations + correction: max %llu ulp, %.3g%% differ\n", o[1], 100.0 * o[5] / total);
  printf("rcp 1 Newton step: max %llu ulp; 2 steps: max %llu ulp\n", o[2], o[3]);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
