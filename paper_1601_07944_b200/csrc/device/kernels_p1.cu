// Kernels for polynomial degree 1 (see kernels_tu.cuh) plus the p = 1
// Barth-Jespersen limiter with the positivity guard (solver.cpp:286-425).
#define DGB_P 1
#include <cstdlib>

#include "kernels_tu.cuh"

namespace dgbk {

namespace {
__constant__ LimTab c_lim;
constexpr int kLimNE = 6, kLimNPT = 12;  // p = 1 tables: 2 points per edge, 3 interior
constexpr int kLim4PerSm = 128;          // latency-form limiter up to this many elements per SM

__device__ __forceinline__ double ref_pressure(double rho, double mx, double my, double E, double g1) {
  return g1 * (E - __dmul_rn(0.5, fma(my, my, __dmul_rn(mx, mx))) / rho);
}
}  // namespace

namespace {
// One thread per element, in place on modes 1..2 (mode 0 is never written, so
// reading the neighbours' means while limiting is race-free, solver.cpp:419-422).
// NE / NPT: edge points and all check points as compile-time constants (0: read from c_lim),
// so the point loops unroll onto immediate constant-bank operands.
#ifndef DGB_LIMIT_MINB
#define DGB_LIMIT_MINB 6  // 80 registers: 0.120 ms per stage on the 2M DMR vs 0.128 at 64, 0.126 at 72 (measured)
#endif
#ifndef DGB_LIMIT_CFL_PREFETCH
#define DGB_LIMIT_CFL_PREFETCH 1
#endif
// EPI: epilogues compiled into the instance (1: CFL bound, 2: residual), the launch passes
// a.want_lambda / a.want_resid; the intermediate-stage instance carries neither.

// Loads of the limiter's inputs.  The standalone kernel reads its own coefficients through L1
// and the neighbours' means read-only; inside the fused stage + limiter kernel every read of the
// stage output must bypass L1 (ld.global.cg): other SMs write it during the same launch, and an
// L1 sector fetched for one neighbour may hold a not-yet-published element next to it.
template <bool Coherent>
__device__ __forceinline__ double lim_ld(const double* p) {
  if constexpr (Coherent) return __ldcg(p); else return *p;
}
template <bool Coherent>
__device__ __forceinline__ double lim_ldg(const double* p) {
  if constexpr (Coherent) return __ldcg(p); else return __ldg(p);
}

// Barth-Jespersen + positivity guard of one element (solver.cpp:286-425), in place on modes
// 1..2, with the residual and CFL epilogues of the last stage.  Every product-sum is written as
// an explicit fma / __dmul_rn: left to the compiler, the contraction of e.g. c1 phi1 + c2 phi2
// differed between kernel instances (measured: the EPI=2 and EPI=3 limiters gave slopes one
// ulp apart), and the limiter must give the same bits in every instance and launch form.
template <int NE, int NPT, int EPI, bool Coherent>
__device__ __forceinline__ void limit_element(const Geo& geo, const LimArgs& a, int e, double& lam_min,
                                              double& res_max) {
  const bool want_lambda = (EPI & 1) && a.want_lambda, want_resid = (EPI & 2) && a.want_resid;
  constexpr int NP = 3;
  const long long ld = geo.ld;
  const double g1 = geo.gamma - 1.0;
  const double sqrt2 = sqrt(2.0);
  Scalars* sc = a.sc;
  const LimTab& L = c_lim;
  const Tab<1>& T = c_tab;
  const int n_edge = NE ? NE : L.n_edge;
  const int e_begin = NE ? NPT - NE - 3 : L.edge_begin;
  const int n_pts = NPT ? NPT : L.n_pts;
  {
    double c0[4], c1[4], c2[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      c0[m] = lim_ld<Coherent>(a.c + (m * NP + 0) * ld + e);
      c1[m] = lim_ld<Coherent>(a.c + (m * NP + 1) * ld + e);
      c2[m] = lim_ld<Coherent>(a.c + (m * NP + 2) * ld + e);
    }
    int nb[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) nb[q] = __ldg(geo.nbr + q * ld + e);
#if DGB_LIMIT_CFL_PREFETCH
    // the CFL epilogue's edge normals and inradius, requested with the neighbour means
    int ed3[3] = {0, 0, 0};
    double enx3[3] = {0.0, 0.0, 0.0}, eny3[3] = {0.0, 0.0, 0.0}, rin = 0.0;
    if (want_lambda) {
#pragma unroll
      for (int q = 0; q < 3; ++q) ed3[q] = __ldg(geo.eid + q * ld + e);
      rin = __ldg(geo.inradius + e);
    }
#endif
    // the neighbours' means, all requested at once (mode 0 is never written here,
    // so the read-only path is safe)
    double nm[3][4];
    if (!Coherent && a.means) {  // the same values from the stage kernel's compact means: 2 loads per neighbour
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double2* mp = reinterpret_cast<const double2*>(a.means + 4 * static_cast<long long>(nb[q] >= 0 ? nb[q] : e));
        const double2 lo = __ldg(mp), hi = __ldg(mp + 1);
        nm[q][0] = nb[q] >= 0 ? lo.x : 0.0;
        nm[q][1] = nb[q] >= 0 ? lo.y : 0.0;
        nm[q][2] = nb[q] >= 0 ? hi.x : 0.0;
        nm[q][3] = nb[q] >= 0 ? hi.y : 0.0;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int m = 0; m < 4; ++m) nm[q][m] = nb[q] >= 0 ? lim_ldg<Coherent>(a.c + (m * NP) * ld + nb[q]) : 0.0;
    }
#if DGB_LIMIT_CFL_PREFETCH
    if (want_lambda) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        enx3[q] = __ldg(geo.enx + ed3[q]);
        eny3[q] = __ldg(geo.eny + ed3[q]);
      }
    }
#endif

    // Barth-Jespersen per conserved variable against the neighbours' centroid range
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double uc = __dmul_rn(c0[m], sqrt2);
      double umax = uc, umin = uc;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (nb[q] < 0) continue;
        const double un = __dmul_rn(nm[q][m], sqrt2);
        umax = std_max(umax, un);
        umin = std_min(umin, un);
      }
      const double tol = 1e-13 * (fabs(uc) + (umax - umin));
      // min over the edge points of clamp((umax-uc)/d) for d > tol and clamp((umin-uc)/d) for
      // d < -tol (solver.cpp:348-358).  The numerators have fixed signs and correctly rounded
      // division is monotone in the divisor, so the minimum is the quotient by the extreme d:
      // two divisions per variable instead of one per point.  tol >= 0, so the extreme d
      // beyond +-tol is the extreme of all d when that clears the threshold (and NaN d are
      // skipped by the selects as by the comparisons): bit-identical.
      double dpos = 0.0, dneg = 0.0;
#pragma unroll
      for (int k = e_begin; k < e_begin + n_edge; ++k) {
        const double d = fma(c2[m], L.phi2[k], __dmul_rn(c1[m], L.phi1[k]));
        dpos = d > dpos ? d : dpos;  // a NaN d is skipped, as by the reference's comparisons
        dneg = d < dneg ? d : dneg;
      }
      double alpha = 1.0;
      if (dpos > tol) alpha = std_min(alpha, std_clamp01((umax - uc) / dpos));
      if (dneg < -tol) alpha = std_min(alpha, std_clamp01((umin - uc) / dneg));
      c1[m] *= alpha;
      c2[m] *= alpha;
    }

    // positivity guard toward the cell mean (solver.cpp:363-417)
    const double mr = __dmul_rn(c0[0], sqrt2), mmx = __dmul_rn(c0[1], sqrt2), mmy = __dmul_rn(c0[2], sqrt2),
                 mE = __dmul_rn(c0[3], sqrt2);
    const double p_mean = ref_pressure(mr, mmx, mmy, mE, g1);
    if (mr > 0.0 && p_mean > 0.0) {
      const double eps_rho = 1e-8 * mr;
      const double eps_p = 1e-8 * p_mean;
      double dev[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) dev[m] = fma(fabs(c2[m]), L.max_phi2, __dmul_rn(fabs(c1[m]), L.max_phi1));
      const double rho_floor = mr - dev[0];
      bool safe = rho_floor > eps_rho;
      if (safe) {
        const double mx_peak = fabs(mmx) + dev[1];
        const double my_peak = fabs(mmy) + dev[2];
        const double p_floor =
            g1 * ((mE - dev[3]) - __dmul_rn(0.5, fma(my_peak, my_peak, __dmul_rn(mx_peak, mx_peak))) / rho_floor);
        safe = p_floor > eps_p;
      }
      if (!safe) {
        double rho_min = mr;
        for (int k = 0; k < n_pts; ++k)
          rho_min = fmin(rho_min, fma(c2[0], L.phi2[k], fma(c1[0], L.phi1[k], __dmul_rn(c0[0], sqrt2))));
        if (rho_min < eps_rho) {
          const double th = fmin(fmax((mr - eps_rho) / (mr - rho_min), 0.0), 1.0);
          c1[0] *= th;
          c2[0] *= th;
        }
        double th_p = 1.0;
        for (int k = 0; k < n_pts; ++k) {
          double u[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) u[m] = fma(c2[m], L.phi2[k], fma(c1[m], L.phi1[k], __dmul_rn(c0[m], sqrt2)));
          if (u[0] <= 0.0) {
            th_p = 0.0;
            break;
          }
          const double pk = ref_pressure(u[0], u[1], u[2], u[3], g1);
          if (pk < eps_p) th_p = fmin(th_p, (p_mean - eps_p) / (p_mean - pk));
        }
        if (th_p < 1.0) {
          th_p = fmax(th_p, 0.0);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            c1[m] *= th_p;
            c2[m] *= th_p;
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      a.c[(m * NP + 1) * ld + e] = c1[m];
      a.c[(m * NP + 2) * ld + e] = c2[m];
    }
    if (want_resid) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        res_max = std_max(res_max, fabs(__ldg(a.u + (m * NP + 0) * ld + e) - c0[m]));
        res_max = std_max(res_max, fabs(__ldg(a.u + (m * NP + 1) * ld + e) - c1[m]));
        res_max = std_max(res_max, fabs(__ldg(a.u + (m * NP + 2) * ld + e) - c2[m]));
      }
    }
    if (want_lambda) {  // CFL bound of the limited state (solver.cpp:439-457)
      double lam = 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        double U[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) U[m] = fma(T.phm[q][2], c2[m], fma(T.phm[q][1], c1[m], T.phm[q][0] * c0[m]));
#if DGB_LIMIT_CFL_PREFETCH
        const double nxq = enx3[q], nyq = eny3[q];
#else
        const int ed = __ldg(geo.eid + q * ld + e);
        const double nxq = __ldg(geo.enx + ed), nyq = __ldg(geo.eny + ed);
#endif
        bool ok;
        const double ws = wave_speed_ieee(U, nxq, nyq, geo.gamma, ok);
        if (!ok) {
          record_error(sc, err_key(a.seq, kPassDt, __ldg(geo.ref_id + e), q + 1));
          continue;
        }
        lam = std_max(lam, ws);
      }
#if DGB_LIMIT_CFL_PREFETCH
      lam_min = std_min(lam_min, 2.0 * rin / (3.0 * lam));
#else
      lam_min = std_min(lam_min, 2.0 * __ldg(geo.inradius + e) / (3.0 * lam));
#endif
    }
  }
}

// The latency form of limit_element: four lanes per element, lane v owning conserved variable
// v, for launches that leave the GPU mostly idle (small meshes: a stage then costs one element's
// dependency chain, not bandwidth).  Barth-Jespersen of variable v runs on lane v with exactly
// the operations of limit_element's loop body for m = v; the positivity guard gathers the four
// means and deviations by shuffles and every lane of the quad evaluates it redundantly (the same
// operations on the same operands, so the same decision and factors); the CFL epilogue evaluates
// midpoint q on lane q.  Bit-identical to limit_element (tests/test_gpu_parity.py).
// The geometry limit_element4 reads (it does not depend on the state, so the fused kernel
// requests it before waiting for the neighbours' stage output).
struct LimGeo4 {
  int nb[3];
  double enx, eny, rin;
};
template <int EPI>
__device__ __forceinline__ LimGeo4 lim_geo4(const Geo& geo, const LimArgs& a, int e, int v) {
  LimGeo4 r;
  const long long ld = geo.ld;
#pragma unroll
  for (int q = 0; q < 3; ++q) r.nb[q] = __ldg(geo.nbr + q * ld + e);
  r.enx = r.eny = r.rin = 0.0;
  if ((EPI & 1) && a.want_lambda) {  // CFL epilogue operands of midpoint q = v
    const int ed = __ldg(geo.eid + (v < 3 ? v : 2) * ld + e);
    r.rin = __ldg(geo.inradius + e);
    r.enx = __ldg(geo.enx + ed);
    r.eny = __ldg(geo.eny + ed);
  }
  return r;
}

template <int NE, int NPT, int EPI, bool Coherent = false>
__device__ __forceinline__ void limit_element4(const Geo& geo, const LimArgs& a, int e, bool valid, int v,
                                               double& lam_min, double& res_max, const LimGeo4* pre = nullptr) {
  const bool want_lambda = (EPI & 1) && a.want_lambda, want_resid = (EPI & 2) && a.want_resid;
  constexpr int NP = 3;
  const long long ld = geo.ld;
  const double g1 = geo.gamma - 1.0;
  const double sqrt2 = sqrt(2.0);
  Scalars* sc = a.sc;
  const LimTab& L = c_lim;
  const Tab<1>& T = c_tab;
  const int n_edge = NE ? NE : L.n_edge;
  const int e_begin = NE ? NPT - NE - 3 : L.edge_begin;
  const int n_pts = NPT ? NPT : L.n_pts;
  const double* __restrict__ cv = a.c + static_cast<long long>(v) * NP * ld;
  const double c0 = lim_ld<Coherent>(cv + e);
  double c1 = lim_ld<Coherent>(cv + ld + e), c2 = lim_ld<Coherent>(cv + 2 * ld + e);
  const LimGeo4 gg = pre ? *pre : lim_geo4<EPI>(geo, a, e, v);
  const int nb[3] = {gg.nb[0], gg.nb[1], gg.nb[2]};
  const double enx = gg.enx, eny = gg.eny, rin = gg.rin;
  double nm[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) nm[q] = nb[q] >= 0 ? lim_ldg<Coherent>(cv + nb[q]) : 0.0;

  // Barth-Jespersen of variable v (limit_element, loop body for m = v)
  {
    const double uc = __dmul_rn(c0, sqrt2);
    double umax = uc, umin = uc;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (nb[q] < 0) continue;
      const double un = __dmul_rn(nm[q], sqrt2);
      umax = std_max(umax, un);
      umin = std_min(umin, un);
    }
    const double tol = 1e-13 * (fabs(uc) + (umax - umin));
    double dpos = 0.0, dneg = 0.0;
#pragma unroll
    for (int k = e_begin; k < e_begin + n_edge; ++k) {
      const double d = fma(c2, L.phi2[k], __dmul_rn(c1, L.phi1[k]));
      dpos = d > dpos ? d : dpos;
      dneg = d < dneg ? d : dneg;
    }
    double alpha = 1.0;
    if (dpos > tol) alpha = std_min(alpha, std_clamp01((umax - uc) / dpos));
    if (dneg < -tol) alpha = std_min(alpha, std_clamp01((umin - uc) / dneg));
    c1 *= alpha;
    c2 *= alpha;
  }

  // positivity guard toward the cell mean (solver.cpp:363-417) on the gathered quad
  const double dv = fma(fabs(c2), L.max_phi2, __dmul_rn(fabs(c1), L.max_phi1));
  double C0[4], dev[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    C0[m] = __shfl_sync(kFull, c0, m, 4);
    dev[m] = __shfl_sync(kFull, dv, m, 4);
  }
  const double mr = __dmul_rn(C0[0], sqrt2), mmx = __dmul_rn(C0[1], sqrt2), mmy = __dmul_rn(C0[2], sqrt2),
               mE = __dmul_rn(C0[3], sqrt2);
  const double p_mean = ref_pressure(mr, mmx, mmy, mE, g1);
  const bool guard = mr > 0.0 && p_mean > 0.0;
  const double eps_rho = 1e-8 * mr;
  const double eps_p = 1e-8 * p_mean;
  bool safe = true;
  if (guard) {
    const double rho_floor = mr - dev[0];
    safe = rho_floor > eps_rho;
    if (safe) {
      const double mx_peak = fabs(mmx) + dev[1];
      const double my_peak = fabs(mmy) + dev[2];
      const double p_floor =
          g1 * ((mE - dev[3]) - __dmul_rn(0.5, fma(my_peak, my_peak, __dmul_rn(mx_peak, mx_peak))) / rho_floor);
      safe = p_floor > eps_p;
    }
  }
  const bool slow = guard && !safe;
  if (__any_sync(kFull, slow)) {  // shuffles by the whole warp, the sweep only where needed
    double C1[4], C2[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      C1[m] = __shfl_sync(kFull, c1, m, 4);
      C2[m] = __shfl_sync(kFull, c2, m, 4);
    }
    if (slow) {
      double rho_min = mr;
      for (int k = 0; k < n_pts; ++k)
        rho_min = fmin(rho_min, fma(C2[0], L.phi2[k], fma(C1[0], L.phi1[k], __dmul_rn(C0[0], sqrt2))));
      if (rho_min < eps_rho) {
        const double th = fmin(fmax((mr - eps_rho) / (mr - rho_min), 0.0), 1.0);
        C1[0] *= th;
        C2[0] *= th;
        if (v == 0) {
          c1 = C1[0];
          c2 = C2[0];
        }
      }
      double th_p = 1.0;
      for (int k = 0; k < n_pts; ++k) {
        double u[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) u[m] = fma(C2[m], L.phi2[k], fma(C1[m], L.phi1[k], __dmul_rn(C0[m], sqrt2)));
        if (u[0] <= 0.0) {
          th_p = 0.0;
          break;
        }
        const double pk = ref_pressure(u[0], u[1], u[2], u[3], g1);
        if (pk < eps_p) th_p = fmin(th_p, (p_mean - eps_p) / (p_mean - pk));
      }
      if (th_p < 1.0) {
        th_p = fmax(th_p, 0.0);
        c1 *= th_p;
        c2 *= th_p;
      }
    }
  }
  if (valid) {
    double* __restrict__ cw = a.c + static_cast<long long>(v) * NP * ld;
    cw[ld + e] = c1;
    cw[2 * ld + e] = c2;
    if (want_resid) {
      const double* __restrict__ uv = a.u + static_cast<long long>(v) * NP * ld;
      res_max = std_max(res_max, fabs(__ldg(uv + e) - c0));
      res_max = std_max(res_max, fabs(__ldg(uv + ld + e) - c1));
      res_max = std_max(res_max, fabs(__ldg(uv + 2 * ld + e) - c2));
    }
  }
  if (want_lambda) {  // CFL bound of the limited state (solver.cpp:439-457), midpoint q on lane q
    double U[4];
#pragma unroll
    for (int q = 0; q < 3; ++q) U[q] = fma(T.phm[q][2], c2, fma(T.phm[q][1], c1, T.phm[q][0] * c0));
    U[3] = U[0];
    transpose4(U, v);  // lane q: the four variables at midpoint q
    bool ok;
    const double ws = wave_speed_ieee(U, enx, eny, geo.gamma, ok);
    double lam = 0.0;
    if (v < 3) {
      if (ok) {
        lam = ws;
      } else if (valid) {
        record_error(sc, err_key(a.seq, kPassDt, __ldg(geo.ref_id + e), v + 1));
      }
    }
    lam = std_max(lam, __shfl_xor_sync(kFull, lam, 1));
    lam = std_max(lam, __shfl_xor_sync(kFull, lam, 2));
    if (valid && v == 0) lam_min = std_min(lam_min, 2.0 * rin / (3.0 * lam));
  }
}

template <int NE, int NPT, int EPI>
__global__ void __launch_bounds__(kBlock) k_limit4(Geo geo, LimArgs a) {
  Scalars* sc = a.sc;
  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  __syncthreads();
  if (s_stop) return;
  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;
  const int n4 = ((a.e1 - a.e0) * 4 + 31) & ~31;  // whole warps: the quads shuffle warp-wide
  for (int tid = blockIdx.x * blockDim.x + threadIdx.x; tid < n4; tid += gridDim.x * blockDim.x) {
    int e = a.e0 + (tid >> 2);
    const bool valid = e < a.e1;
    if (!valid) e = a.e1 - 1;
    limit_element4<NE, NPT, EPI>(geo, a, e, valid, tid & 3, lam_min, res_max);
  }
  const bool want_lambda = (EPI & 1) && a.want_lambda, want_resid = (EPI & 2) && a.want_resid;
  const int par = a.step & 1;
  if (want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
  if (want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
}

template <int NE, int NPT, int EPI>
__global__ void __launch_bounds__(kBlock, DGB_LIMIT_MINB) k_limit(Geo geo, LimArgs a) {
  Scalars* sc = a.sc;
  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  __syncthreads();
  if (s_stop) return;
  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;
  for (int e = a.e0 + blockIdx.x * blockDim.x + threadIdx.x; e < a.e1; e += gridDim.x * blockDim.x)
    limit_element<NE, NPT, EPI, false>(geo, a, e, lam_min, res_max);
  const bool want_lambda = (EPI & 1) && a.want_lambda, want_resid = (EPI & 2) && a.want_resid;
  const int par = a.step & 1;
  if (want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
  if (want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
}

constexpr unsigned long long kFuseTimeoutKey = (7ull << 35) | 1ull;  // sorts before every solver error

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

#ifndef DGB_FUSE_MINB
#define DGB_FUSE_MINB 4  // blocks per SM of the fused kernel (the stage body's register budget)
#endif

// Stage + limiter in one launch.  A cooperative grid of warps, each
// running a fixed sequence of 32-element tiles (FuseArgs): the stage of tile i (the element
// kernel's body, no epilogues), published with a release add to its chunk counter, then the
// limiter of tile j = i - lag once every chunk holding a neighbour of j has published (acquire,
// one chunk per lane).  The limiter reads the fresh stage output from L2 (ld.global.cg), so the
// unlimited state never makes an HBM round trip between two kernels, and the limiter's
// instructions overlap other warps' stage work.  No deadlock: every warp is resident
// (cooperative launch); a warp in its k-th tile waits only for stage parts of tiles <= i - W
// (lag >= reach + W), i.e. of other warps' earlier iterations, and a stage part never waits.
// No early exit once running (an error recorded by another warp of this launch must not make a
// block skip tiles others wait for): only errors of earlier launches (sequence < a.seq) and the
// drivers' stop rules, both grid-uniform, end the launch at its start.
template <int FLUX, int VAR, int EPI>
__global__ void __launch_bounds__(kBlock, DGB_FUSE_MINB) k_stage_limit(Geo geo, StageArgs a, LimArgs la,
                                                                      FuseArgs f) {
  __shared__ int s_stop;
  Scalars* sc = a.sc;
  if (threadIdx.x == 0) {
    const unsigned long long k = sc->err_key;
    s_stop = ((k != kNoError && (k >> 38) < a.seq) || sc->halt) ? 1 : 0;
  }
  __syncthreads();
  double t0 = a.t_host, dt = 0.0;
  const bool run = !s_stop && stage_prologue(a, sc, t0, dt);
  const double tstage = fma(a.tcoef, dt, t0);
  double lam_min = __longlong_as_double(0x7ff0000000000000ll), res_max = 0.0;
  double st_lam = lam_min, st_res = 0.0;  // the stage body's epilogues are off (VAR has no kVarLambda)
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * (blockDim.x >> 5);
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  bool timed_out = false;
  if (run) {
    for (int i = w; i < f.n_tiles + f.lag; i += W) {
      if (i < f.n_tiles) {
        const int e = a.e0 + i * kFuseTile + lane;
        if (e < a.e1) g1_element<1, kModeStage, FLUX, VAR>(c_tab, geo, a, e, dt, tstage, st_lam, st_res);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(f.count + i / kFuseChunk, 1ull);  // after the fence: a release
      }
      const int j = i - f.lag;
      if (j >= 0) {
        const int2 r = __ldg(f.range + j);
        for (int c = r.x + lane; c <= r.y; c += 32) {
          const unsigned long long need = f.epoch * min(kFuseChunk, f.n_tiles - c * kFuseChunk);
          long long spins = 0;
          while (ld_acquire_gpu(f.count + c) < need) {
            __nanosleep(64);
            if (++spins > (1ll << 26)) {  // seconds: a broken launch, never a hang
              timed_out = true;
              break;
            }
          }
        }
        __syncwarp();
        __threadfence();
        const int e = la.e0 + j * kFuseTile + lane;
        if (e < la.e1) limit_element<kLimNE, kLimNPT, EPI, true>(geo, la, e, lam_min, res_max);
      }
    }
  }
  if (timed_out) record_error(sc, kFuseTimeoutKey);
  const int par = la.step & 1;
  if ((EPI & 1) && la.want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
  if ((EPI & 2) && la.want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
}

// Latency form of k_stage_limit for small meshes (a grid with one warp per 8-element subtile):
// warp w runs the stage of subtile w first (four lanes per element, g4_element), then limiter
// subtiles w, w + W, ... (four lanes per element, limit_element4), each once the chunks holding
// its neighbours have published (4 subtiles per 32-element tile).  Stage parts never wait and
// every warp is resident, so no warp waits on work that cannot start.  Bit-identical to the
// other forms.
template <int FLUX, int VAR, int EPI>
__global__ void __launch_bounds__(kBlock, DGB_FUSE_MINB) k_stage_limit4(Geo geo, StageArgs a, LimArgs la,
                                                                       FuseArgs f) {
  __shared__ int s_stop;
  Scalars* sc = a.sc;
  if (threadIdx.x == 0) {
    const unsigned long long k = sc->err_key;
    s_stop = ((k != kNoError && (k >> 38) < a.seq) || sc->halt) ? 1 : 0;
  }
  __syncthreads();
  double t0 = a.t_host, dt = 0.0;
  const bool run = !s_stop && stage_prologue(a, sc, t0, dt);
  const double tstage = fma(a.tcoef, dt, t0);
  double lam_min = __longlong_as_double(0x7ff0000000000000ll), res_max = 0.0;
  double st_lam = lam_min, st_res = 0.0;
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * (blockDim.x >> 5);
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  bool timed_out = false;
  if (run) {
    if (w < 4 * f.n_tiles) {
      int e = a.e0 + w * 8 + (lane >> 2);
      const bool valid = e < a.e1;
      if (!valid) e = a.e1 - 1;
      g4_element<1, kModeStage, FLUX, VAR>(c_tab, geo, a, e, valid, lane & 3, dt, tstage, st_lam, st_res);
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(f.count + (w >> 2) / kFuseChunk, 1ull);
    }
    for (int j4 = w; j4 < 4 * f.n_tiles; j4 += W) {
      int e = la.e0 + j4 * 8 + (lane >> 2);
      const bool valid = e < la.e1;
      if (!valid) e = la.e1 - 1;
      const LimGeo4 gg = lim_geo4<EPI>(geo, la, e, lane & 3);  // in flight during the wait
      const int2 r = __ldg(f.range + (j4 >> 2));
      for (int c = r.x + lane; c <= r.y; c += 32) {
        const unsigned long long need = 4 * f.epoch * min(kFuseChunk, f.n_tiles - c * kFuseChunk);
        long long spins = 0;
        while (ld_acquire_gpu(f.count + c) < need) {
          __nanosleep(32);
          if (++spins > (1ll << 26)) {
            timed_out = true;
            break;
          }
        }
      }
      __syncwarp();
      __threadfence();
      limit_element4<kLimNE, kLimNPT, EPI, true>(geo, la, e, valid, lane & 3, lam_min, res_max, &gg);
    }
  }
  if (timed_out) record_error(sc, kFuseTimeoutKey);
  const int par = la.step & 1;
  if ((EPI & 1) && la.want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
  if ((EPI & 2) && la.want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
}

// host copy of (n_edge, n_pts) of the table uploaded to each device's bank (packed in one
// atomic word: the limiter may be launched from several host threads)
std::atomic<int> g_lim_pts[kMaxDevices];
}  // namespace

cudaError_t upload_limtab(const LimTab& t, cudaStream_t s) {
  const int npt = t.edge_begin + t.n_edge + 3 == t.n_pts ? t.n_pts : 0;
  g_lim_pts[current_device()].store(t.n_edge | (npt << 16));
  return cudaMemcpyToSymbolAsync(c_lim, &t, sizeof(t), 0, cudaMemcpyHostToDevice, s);
}


cudaError_t preload_limit() {
  cudaError_t err = cudaSuccess;
  auto touch = [&](auto k) {
    cudaFuncAttributes fa;
    const cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) err = e;
  };
  touch(k_limit<0, 0, 3>);
  touch(k_limit<kLimNE, kLimNPT, 0>);
  touch(k_limit<kLimNE, kLimNPT, 1>);
  touch(k_limit<kLimNE, kLimNPT, 2>);
  touch(k_limit<kLimNE, kLimNPT, 3>);
  touch(k_limit4<kLimNE, kLimNPT, 0>);
  touch(k_limit4<kLimNE, kLimNPT, 1>);
  touch(k_limit4<kLimNE, kLimNPT, 2>);
  touch(k_limit4<kLimNE, kLimNPT, 3>);
  return err;
}

int limit_resident_blocks() {
  static std::atomic<int> occ{0};
  int o = occ.load(std::memory_order_relaxed);
  if (!o) occ.store(o = occupancy(k_limit<kLimNE, kLimNPT, 3>), std::memory_order_relaxed);
  return o;
}

int stage_limit_grid() {
  static std::atomic<int> occ{0};
  int o = occ.load(std::memory_order_relaxed);
  if (!o) occ.store(o = occupancy(k_stage_limit<kFluxRoe, kVarRk4 | kVarBoundary, 3>), std::memory_order_relaxed);
  return o * sm_count();
}

namespace {
int stage_limit4_grid() {  // co-resident blocks of the latency form (its own register budget)
  static std::atomic<int> occ{0};
  int o = occ.load(std::memory_order_relaxed);
  if (!o) occ.store(o = occupancy(k_stage_limit4<kFluxRoe, kVarRk4 | kVarBoundary, 3>), std::memory_order_relaxed);
  return o * sm_count();
}
}  // namespace

cudaError_t launch_stage_limit(int grid, const Geo& g, const StageArgs& a, const LimArgs& la, const FuseArgs& f,
                               cudaStream_t s) {
  if (a.e1 <= a.e0) return cudaSuccess;
  if (g_lim_pts[current_device()].load() != (kLimNE | (kLimNPT << 16))) return cudaErrorInvalidValue;
  if (grid <= 0) grid = stage_limit_grid();
  const int var = (g.has_bnd ? kVarBoundary : 0) | (a.kmode != 0 ? kVarRk4 : 0);
  const bool last = la.want_lambda || la.want_resid;
  cudaError_t err = cudaSuccess;
  // latency form: one warp per stage tile and per 8-element limiter subtile fit in one wave
  const int wpb = kBlock / 32;
  const bool lat = f.n_tiles > 0 && 4 * f.n_tiles <= stage_limit4_grid() * wpb &&
                   (g.lat_limit_n >= 0 ? a.e1 - a.e0 <= g.lat_limit_n : true);
  if (lat) grid = (4 * f.n_tiles + wpb - 1) / wpb;
  auto go = [&](auto k) {  // cooperative: every warp of the grid is resident (the tiles' waits need it)
    void* args[] = {const_cast<Geo*>(&g), const_cast<StageArgs*>(&a), const_cast<LimArgs*>(&la),
                    const_cast<FuseArgs*>(&f)};
    err = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(grid), dim3(kBlock), args, 0, s);
  };
  if (lat) {
    const bool roe = g.flux == kFluxRoe;
    switch (var | (last ? 8 : 0) | (roe ? 16 : 0)) {
      case 0: go(k_stage_limit4<kFluxLLF, 0, 0>); break;
      case 1: go(k_stage_limit4<kFluxLLF, 1, 0>); break;
      case 4: go(k_stage_limit4<kFluxLLF, 4, 0>); break;
      case 5: go(k_stage_limit4<kFluxLLF, 5, 0>); break;
      case 8: go(k_stage_limit4<kFluxLLF, 0, 3>); break;
      case 9: go(k_stage_limit4<kFluxLLF, 1, 3>); break;
      case 12: go(k_stage_limit4<kFluxLLF, 4, 3>); break;
      case 13: go(k_stage_limit4<kFluxLLF, 5, 3>); break;
      case 16: go(k_stage_limit4<kFluxRoe, 0, 0>); break;
      case 17: go(k_stage_limit4<kFluxRoe, 1, 0>); break;
      case 20: go(k_stage_limit4<kFluxRoe, 4, 0>); break;
      case 21: go(k_stage_limit4<kFluxRoe, 5, 0>); break;
      case 24: go(k_stage_limit4<kFluxRoe, 0, 3>); break;
      case 25: go(k_stage_limit4<kFluxRoe, 1, 3>); break;
      case 28: go(k_stage_limit4<kFluxRoe, 4, 3>); break;
      default: go(k_stage_limit4<kFluxRoe, 5, 3>); break;
    }
    return err;
  }
  if (g.flux == kFluxRoe) {
    switch (var | (last ? 8 : 0)) {
      case 0: go(k_stage_limit<kFluxRoe, 0, 0>); break;
      case 1: go(k_stage_limit<kFluxRoe, 1, 0>); break;
      case 4: go(k_stage_limit<kFluxRoe, 4, 0>); break;
      case 5: go(k_stage_limit<kFluxRoe, 5, 0>); break;
      case 8: go(k_stage_limit<kFluxRoe, 0, 3>); break;
      case 9: go(k_stage_limit<kFluxRoe, 1, 3>); break;
      case 12: go(k_stage_limit<kFluxRoe, 4, 3>); break;
      default: go(k_stage_limit<kFluxRoe, 5, 3>); break;
    }
  } else {
    switch (var | (last ? 8 : 0)) {
      case 0: go(k_stage_limit<kFluxLLF, 0, 0>); break;
      case 1: go(k_stage_limit<kFluxLLF, 1, 0>); break;
      case 4: go(k_stage_limit<kFluxLLF, 4, 0>); break;
      case 5: go(k_stage_limit<kFluxLLF, 5, 0>); break;
      case 8: go(k_stage_limit<kFluxLLF, 0, 3>); break;
      case 9: go(k_stage_limit<kFluxLLF, 1, 3>); break;
      case 12: go(k_stage_limit<kFluxLLF, 4, 3>); break;
      default: go(k_stage_limit<kFluxLLF, 5, 3>); break;
    }
  }
  return err;
}

// Elements up to which a limiter launch takes the four-lane latency form (k_limit4): below
// this the one-thread form leaves most of the GPU idle and the launch costs one element's
// dependency chain.  DGB_LIM4_MAXN overrides (0: never).
int limit_latency_max_n() {
  static std::atomic<int> v{-1};
  int n = v.load(std::memory_order_relaxed);
  if (n < 0) {
    const char* env = std::getenv("DGB_LIM4_MAXN");
    n = env ? std::atoi(env) : kLim4PerSm * sm_count();
    v.store(n, std::memory_order_relaxed);
  }
  return n;
}

cudaError_t launch_limit(int grid, const Geo& g, const LimArgs& a, cudaStream_t s) {
  if (a.e1 <= a.e0) return cudaSuccess;
  const int epi = (a.want_lambda ? 1 : 0) | (a.want_resid ? 2 : 0);
  if (a.e1 - a.e0 <= (g.lat_limit_n >= 0 ? g.lat_limit_n : limit_latency_max_n()) && g_lim_pts[current_device()].load() == (kLimNE | (kLimNPT << 16))) {
    if (grid <= 0) grid = grid_for(static_cast<long long>(a.e1 - a.e0) * 4, 16);
    switch (epi) {
      case 0: k_limit4<kLimNE, kLimNPT, 0><<<grid, kBlock, 0, s>>>(g, a); break;
      case 1: k_limit4<kLimNE, kLimNPT, 1><<<grid, kBlock, 0, s>>>(g, a); break;
      case 2: k_limit4<kLimNE, kLimNPT, 2><<<grid, kBlock, 0, s>>>(g, a); break;
      default: k_limit4<kLimNE, kLimNPT, 3><<<grid, kBlock, 0, s>>>(g, a); break;
    }
    return cudaGetLastError();
  }
  if (grid <= 0) grid = grid_for(a.e1 - a.e0, limit_resident_blocks());
  if (g_lim_pts[current_device()].load() == (kLimNE | (kLimNPT << 16))) {
    switch (epi) {
      case 0: k_limit<kLimNE, kLimNPT, 0><<<grid, kBlock, 0, s>>>(g, a); break;
      case 1: k_limit<kLimNE, kLimNPT, 1><<<grid, kBlock, 0, s>>>(g, a); break;
      case 2: k_limit<kLimNE, kLimNPT, 2><<<grid, kBlock, 0, s>>>(g, a); break;
      default: k_limit<kLimNE, kLimNPT, 3><<<grid, kBlock, 0, s>>>(g, a); break;
    }
  } else {
    k_limit<0, 0, 3><<<grid, kBlock, 0, s>>>(g, a);
  }
  return cudaGetLastError();
}

}  // namespace dgbk
