// Kernels for polynomial degree 1 (see kernels_tu.cuh) plus the p = 1
// Barth-Jespersen limiter with the positivity guard (solver.cpp:286-425).
#define DGB_P 1
#include "kernels_tu.cuh"

namespace dgbk {

namespace {
__constant__ LimTab c_lim;

__device__ __forceinline__ double ref_pressure(double rho, double mx, double my, double E, double g1) {
  return g1 * (E - 0.5 * (mx * mx + my * my) / rho);
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
template <int NE, int NPT, int EPI>
__global__ void __launch_bounds__(kBlock, DGB_LIMIT_MINB) k_limit(Geo geo, LimArgs a) {
  const bool want_lambda = (EPI & 1) && a.want_lambda, want_resid = (EPI & 2) && a.want_resid;
  constexpr int NP = 3;
  const long long ld = geo.ld;
  const double g1 = geo.gamma - 1.0;
  const double sqrt2 = sqrt(2.0);
  Scalars* sc = a.sc;
  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  __syncthreads();
  if (s_stop) return;

  const LimTab& L = c_lim;
  const Tab<1>& T = c_tab;
  const int n_edge = NE ? NE : L.n_edge;
  const int e_begin = NE ? NPT - NE - 3 : L.edge_begin;
  const int n_pts = NPT ? NPT : L.n_pts;
  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;

  for (int e = a.e0 + blockIdx.x * blockDim.x + threadIdx.x; e < a.e1; e += gridDim.x * blockDim.x) {
    double c0[4], c1[4], c2[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      c0[m] = a.c[(m * NP + 0) * ld + e];
      c1[m] = a.c[(m * NP + 1) * ld + e];
      c2[m] = a.c[(m * NP + 2) * ld + e];
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
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int m = 0; m < 4; ++m) nm[q][m] = nb[q] >= 0 ? __ldg(a.c + (m * NP) * ld + nb[q]) : 0.0;
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
      const double uc = c0[m] * sqrt2;
      double umax = uc, umin = uc;
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        if (nb[q] < 0) continue;
        const double un = nm[q][m] * sqrt2;
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
        const double d = c1[m] * L.phi1[k] + c2[m] * L.phi2[k];
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
    const double mr = c0[0] * sqrt2, mmx = c0[1] * sqrt2, mmy = c0[2] * sqrt2, mE = c0[3] * sqrt2;
    const double p_mean = ref_pressure(mr, mmx, mmy, mE, g1);
    if (mr > 0.0 && p_mean > 0.0) {
      const double eps_rho = 1e-8 * mr;
      const double eps_p = 1e-8 * p_mean;
      double dev[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) dev[m] = fabs(c1[m]) * L.max_phi1 + fabs(c2[m]) * L.max_phi2;
      const double rho_floor = mr - dev[0];
      bool safe = rho_floor > eps_rho;
      if (safe) {
        const double mx_peak = fabs(mmx) + dev[1];
        const double my_peak = fabs(mmy) + dev[2];
        const double p_floor = g1 * (mE - dev[3] - 0.5 * (mx_peak * mx_peak + my_peak * my_peak) / rho_floor);
        safe = p_floor > eps_p;
      }
      if (!safe) {
        double rho_min = mr;
        for (int k = 0; k < n_pts; ++k)
          rho_min = fmin(rho_min, c0[0] * sqrt2 + c1[0] * L.phi1[k] + c2[0] * L.phi2[k]);
        if (rho_min < eps_rho) {
          const double th = fmin(fmax((mr - eps_rho) / (mr - rho_min), 0.0), 1.0);
          c1[0] *= th;
          c2[0] *= th;
        }
        double th_p = 1.0;
        for (int k = 0; k < n_pts; ++k) {
          double u[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) u[m] = c0[m] * sqrt2 + c1[m] * L.phi1[k] + c2[m] * L.phi2[k];
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
    if (a.push && e >= geo.send_begin) {
      const double v[4][NP] = {{c0[0], c1[0], c2[0]}, {c0[1], c1[1], c2[1]}, {c0[2], c1[2], c2[2]}, {c0[3], c1[3], c2[3]}};
      push_element<NP, 4>(geo, a.peers, a.out_buf, e, 0, v);
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
  const int par = a.step & 1;
  if (want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
  if (want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
  if (a.push) __threadfence_system();
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

constexpr int kLimNE = 6, kLimNPT = 12;  // p = 1 tables: 2 points per edge, 3 interior

int limit_resident_blocks() {
  static std::atomic<int> occ{0};
  int o = occ.load(std::memory_order_relaxed);
  if (!o) occ.store(o = occupancy(k_limit<kLimNE, kLimNPT, 3>), std::memory_order_relaxed);
  return o;
}

cudaError_t launch_limit(int grid, const Geo& g, const LimArgs& a, cudaStream_t s) {
  if (a.e1 <= a.e0) return cudaSuccess;
  if (grid <= 0) grid = grid_for(a.e1 - a.e0, limit_resident_blocks());
  const int epi = (a.want_lambda ? 1 : 0) | (a.want_resid ? 2 : 0);
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
