// Templated device code shared by the per-degree translation units
// (kernels_p1.cu .. kernels_p5.cu).  Each unit defines its own constant bank
// `c_tab` and includes this file.
#pragma once

#include <cuda_runtime.h>

#include "dg_kernels.cuh"

namespace dgbk {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double bits_to_double(unsigned long long b) { return __longlong_as_double(static_cast<long long>(b)); }
__device__ __forceinline__ unsigned long long double_to_bits(double d) {
  return static_cast<unsigned long long>(__double_as_longlong(d));
}

__device__ __forceinline__ unsigned long long err_key(unsigned long long seq, int pass, long long id, int point) {
  return (seq << 38) | (static_cast<unsigned long long>(pass) << 35) |
         (static_cast<unsigned long long>(id & 0x3fffffff) << 5) | static_cast<unsigned long long>(point & 31);
}

__device__ __forceinline__ void record_error(Scalars* sc, unsigned long long key) { atomicMin(&sc->err_key, key); }

// Select variable m of a full state without local-memory indexing.
__device__ __forceinline__ double pick4(const double (&v)[4], int m) {
  double r = v[0];
  r = (m == 1) ? v[1] : r;
  r = (m == 2) ? v[2] : r;
  r = (m == 3) ? v[3] : r;
  return r;
}

// Assemble the full state (rho, mx, my, E) from the G lanes of one element.
template <int G, int MG>
__device__ __forceinline__ void gather_state(const double (&own)[MG], double (&U)[4]) {
  if constexpr (G == 1) {
#pragma unroll
    for (int m = 0; m < 4; ++m) U[m] = own[m];
  } else {
#pragma unroll
    for (int m = 0; m < 4; ++m) U[m] = __shfl_sync(kFull, own[m % MG], m / MG, G);
  }
}

struct Prim {
  double inv, vx, vy, p;
};

// EOS (euler.hpp:29-31) through one reciprocal per state.
__device__ __forceinline__ Prim primitives(const double (&U)[4], double g1) {
  Prim w;
  w.inv = 1.0 / U[0];
  w.vx = U[1] * w.inv;
  w.vy = U[2] * w.inv;
  w.p = g1 * (U[3] - 0.5 * (U[1] * w.vx + U[2] * w.vy));
  return w;
}

__device__ __forceinline__ bool admissible(const double (&U)[4], const Prim& w) { return U[0] > 0.0 && w.p > 0.0; }

// Analytic flux (euler.hpp:43-50).
__device__ __forceinline__ void euler_flux(const double (&U)[4], const Prim& w, double (&f1)[4], double (&f2)[4]) {
  const double ep = U[3] + w.p;
  f1[0] = U[1];
  f1[1] = fma(U[1], w.vx, w.p);
  f1[2] = U[2] * w.vx;
  f1[3] = w.vx * ep;
  f2[0] = U[2];
  f2[1] = U[1] * w.vy;
  f2[2] = fma(U[2], w.vy, w.p);
  f2[3] = w.vy * ep;
}

// Local Lax-Friedrichs flux, normal from left to right (euler.hpp:59-71).
__device__ __forceinline__ void llf_flux(const double (&UL)[4], const double (&UR)[4], double nx, double ny,
                                         double gamma, double (&fn)[4]) {
  const double g1 = gamma - 1.0;
  const Prim wl = primitives(UL, g1), wr = primitives(UR, g1);
  double f1l[4], f2l[4], f1r[4], f2r[4];
  euler_flux(UL, wl, f1l, f2l);
  euler_flux(UR, wr, f1r, f2r);
  const double sl = fabs(wl.vx * nx + wl.vy * ny) + sqrt(gamma * wl.p * wl.inv);
  const double sr = fabs(wr.vx * nx + wr.vy * ny) + sqrt(gamma * wr.p * wr.inv);
  const double s = fmax(sl, sr);
#pragma unroll
  for (int m = 0; m < 4; ++m)
    fn[m] = 0.5 * (nx * (f1l[m] + f1r[m]) + ny * (f2l[m] + f2r[m])) - 0.5 * s * (UR[m] - UL[m]);
}

__device__ __forceinline__ void reflect(const double (&u)[4], double nx, double ny, double (&g)[4]) {
  const double mn = 2.0 * (u[1] * nx + u[2] * ny);
  g[0] = u[0];
  g[1] = u[1] - mn * nx;
  g[2] = u[2] - mn * ny;
  g[3] = u[3];
}

// ghost_state (euler.hpp:118-140) with the host closures replaced by tables.
template <int K>
__device__ __forceinline__ void ghost_state(const double (&ul)[4], int code, int ed, int kc, double nx, double ny,
                                            double t, const Geo& g, double (&ur)[4]) {
  switch (code) {
    case kReflecting:
      reflect(ul, nx, ny, ur);
      break;
    case kCurved: {
      const double* w = g.bwn + 2 * (static_cast<long long>(ed) * K + kc);
      reflect(ul, w[0], w[1], ur);
      break;
    }
    case kInflow:
      if (g.has_dir) {
        const double* s = g.bstate + 4 * (static_cast<long long>(ed) * K + kc);
#pragma unroll
        for (int m = 0; m < 4; ++m) ur[m] = s[m];
      } else {
#pragma unroll
        for (int m = 0; m < 4; ++m) ur[m] = g.inflow[m];
      }
      break;
    case kShock: {
      const double* x = g.bx + 2 * (static_cast<long long>(ed) * K + kc);
      const double front = g.sh_x0 + (x[1] * g.sh_cos + g.sh_speed * t) / g.sh_sin;
      const bool behind = x[0] < front;
#pragma unroll
      for (int m = 0; m < 4; ++m) ur[m] = behind ? g.sh_post[m] : g.sh_pre[m];
      break;
    }
    default:  // outflow (other codes are rejected on the host)
#pragma unroll
      for (int m = 0; m < 4; ++m) ur[m] = ul[m];
      break;
  }
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Block-wide min/max folded into one atomic per block (non-negative doubles
// compare like their bit patterns).
template <bool IsMin>
__device__ __forceinline__ void block_reduce_atomic(double v, unsigned long long* target) {
  __shared__ double red[32];
  v = IsMin ? warp_min(v) : warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    double r = lane < nw ? red[lane] : (IsMin ? __longlong_as_double(0x7ff0000000000000ll) : 0.0);
    r = IsMin ? warp_min(r) : warp_max(r);
    if (lane == 0) {
      if (IsMin)
        atomicMin(target, double_to_bits(r));
      else
        atomicMax(target, double_to_bits(r));
    }
  }
  __syncthreads();
}

// Trace of the neighbour's coefficients on its side S at the reversed points,
// streamed from global memory (the neighbour's column is an L1/L2 hit).  The
// FMA chain is the same as the one the neighbour uses for its own trace, so
// both sides of an edge see bit-identical values.
template <int P, int S, int MG>
__device__ __forceinline__ void neighbour_trace(const Tab<P>& T, const double* __restrict__ in, long long ld, int m0,
                                                int nb, double (&un)[Dim<P>::K][MG]) {
  constexpr int NP = Dim<P>::NP, K = Dim<P>::K;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
#pragma unroll
    for (int mm = 0; mm < MG; ++mm) {
      const double cn = __ldg(in + (static_cast<long long>(m0 + mm) * NP + j) * ld + nb);
#pragma unroll
      for (int ko = 0; ko < K; ++ko) {
        const double ph = T.phe[S][K - 1 - ko][j];
        un[ko][mm] = (j == 0) ? ph * cn : fma(ph, cn, un[ko][mm]);
      }
    }
  }
}

// The fused element kernel.  MODE selects what is written:
//   kModeVolume  -> volume integral only (eval_volume_pass)
//   kModeSurface -> per-side surface integrals into the slot buffer (eval_surface_pass)
//   kModeRhs     -> (volume + surface) / det (compute_rhs)
//   kModeStage   -> RK stage update with the fused epilogues
template <int P, int G, int MODE>
__device__ __forceinline__ void element_body(const Tab<P>& T, const Geo& geo, const StageArgs& a) {
  constexpr int NP = Dim<P>::NP, NQ = Dim<P>::NQ, K = Dim<P>::K, MG = 4 / G;
  const long long ld = geo.ld;
  const int gsize = geo.ld * G;
  const int stride = gridDim.x * blockDim.x;
  const double gamma = geo.gamma, g1 = gamma - 1.0;
  Scalars* sc = a.sc;

  // block-uniform early exit: an error or a stop rule fired in an earlier launch
  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  __syncthreads();
  if (s_stop) return;

  // ---- time and dt of this stage (every thread evaluates the same values)
  double t0 = a.t_host, dt = 0.0;
  if constexpr (MODE == kModeStage) {
    const int par = a.step & 1;
    t0 = sc->t[par];
    if (a.first) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (a.hist && a.step > 0) a.hist[a.step - 1] = bits_to_double(sc->resid[par ^ 1]);
      }
      bool stop = false;
      if (a.stop_at_t_end && !(t0 < a.t_end)) stop = true;
      if (a.stop_steady && a.step > 0 && bits_to_double(sc->resid[par ^ 1]) <= a.tol) stop = true;
      if (stop) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
          sc->halt = 1;
          sc->halt_step = a.step;
        }
        return;
      }
    }
    if (a.dt_mode == 0) {
      dt = a.dt_host;
    } else {
      dt = a.cfl * bits_to_double(sc->dtmin[par]);
      if (a.clip_t_end && t0 + dt > a.t_end) dt = a.t_end - t0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (a.first) {
        sc->dtmin[par ^ 1] = 0x7ff0000000000000ull;  // +inf
        sc->resid[par] = 0ull;
        sc->dt_used[par] = dt;
      }
      if (a.last) sc->t[par ^ 1] = t0 + dt;
    }
  }
  const double tstage = (MODE == kModeStage) ? fma(a.tcoef, dt, t0) : t0;

  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;

  for (int tid = blockIdx.x * blockDim.x + threadIdx.x; tid < gsize; tid += stride) {
    const int lane_g = (G == 1) ? 0 : (tid % G);
    const int m0 = lane_g * MG;
    int e = tid / G;
    const bool valid = e < geo.N;
    if (!valid) e = geo.N - 1;

    double c[MG][NP];
#pragma unroll
    for (int mm = 0; mm < MG; ++mm)
#pragma unroll
      for (int j = 0; j < NP; ++j) c[mm][j] = __ldg(a.in + (static_cast<long long>(m0 + mm) * NP + j) * ld + e);

    double acc[MG][NP];
#pragma unroll
    for (int mm = 0; mm < MG; ++mm)
#pragma unroll
      for (int j = 0; j < NP; ++j) acc[mm][j] = 0.0;

    // ------------------------------------------------------------ volume
    if constexpr (MODE != kModeSurface) {
      const double ta = __ldg(geo.tau + e), tb = __ldg(geo.tau + ld + e);
      const double tc = __ldg(geo.tau + 2 * ld + e), td = __ldg(geo.tau + 3 * ld + e);
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        double u[MG];
#pragma unroll
        for (int mm = 0; mm < MG; ++mm) {
          double s = T.phi[k][0] * c[mm][0];
#pragma unroll
          for (int j = 1; j < NP; ++j) s = fma(T.phi[k][j], c[mm][j], s);
          u[mm] = s;
        }
        double U[4];
        gather_state<G, MG>(u, U);
        Prim w = primitives(U, g1);
        if (!admissible(U, w)) {
          if (valid && lane_g == 0) record_error(sc, err_key(a.seq, kPassVolume, __ldg(geo.ref_id + e), k));
          U[0] = 1.0; U[1] = 0.0; U[2] = 0.0; U[3] = 2.5;  // placeholder (solver.cpp:129-132)
          w.inv = 1.0; w.vx = 0.0; w.vy = 0.0; w.p = 1.0;
        }
        double f1[4], f2[4];
        euler_flux(U, w, f1, f2);
#pragma unroll
        for (int mm = 0; mm < MG; ++mm) {
          const int m = m0 + mm;
          const double F1 = (G == 1) ? f1[mm] : pick4(f1, m);
          const double F2 = (G == 1) ? f2[mm] : pick4(f2, m);
          const double fr = ta * F1 + tb * F2;  // contravariant flux along r
          const double fs = tc * F1 + td * F2;  // along s
#pragma unroll
          for (int j = 0; j < NP; ++j) acc[mm][j] = fma(T.drw[k][j], fr, fma(T.dsw[k][j], fs, acc[mm][j]));
        }
      }
    }

    // ------------------------------------------------------------ surface
    double snx[3], sny[3];
    if constexpr (MODE != kModeVolume) {
      const int inf = __ldg(geo.info + e);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int nb = __ldg(geo.nbr + q * ld + e);
        const int ed = __ldg(geo.eid + q * ld + e);
        const int snb = (inf >> (2 * q)) & 3;
        const bool left = (inf >> (6 + q)) & 1;
        const double nx = __ldg(geo.enx + ed), ny = __ldg(geo.eny + ed), h = __ldg(geo.eh + ed);
        snx[q] = nx;
        sny[q] = ny;
        const bool bnd = nb < 0;

        double un[K][MG];
        if (!bnd) {
          switch (snb) {
            case 1: neighbour_trace<P, 0, MG>(T, a.in, ld, m0, nb, un); break;
            case 2: neighbour_trace<P, 1, MG>(T, a.in, ld, m0, nb, un); break;
            default: neighbour_trace<P, 2, MG>(T, a.in, ld, m0, nb, un); break;
          }
        } else {
#pragma unroll
          for (int ko = 0; ko < K; ++ko)
#pragma unroll
            for (int mm = 0; mm < MG; ++mm) un[ko][mm] = 0.0;
        }
        if constexpr (MODE == kModeSurface) {
#pragma unroll
          for (int mm = 0; mm < MG; ++mm)
#pragma unroll
            for (int j = 0; j < NP; ++j) acc[mm][j] = 0.0;
        }
#pragma unroll
        for (int ko = 0; ko < K; ++ko) {
          double uo[MG];
#pragma unroll
          for (int mm = 0; mm < MG; ++mm) {
            double s = T.phe[q][ko][0] * c[mm][0];
#pragma unroll
            for (int j = 1; j < NP; ++j) s = fma(T.phe[q][ko][j], c[mm][j], s);
            uo[mm] = s;
          }
          double Uo[4], Un[4];
          gather_state<G, MG>(uo, Uo);
          gather_state<G, MG>(un[ko], Un);
          double UL[4], UR[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            UL[m] = left ? Uo[m] : Un[m];
            UR[m] = left ? Un[m] : Uo[m];
          }
          const int kc = left ? ko : K - 1 - ko;
          if (bnd) ghost_state<K>(UL, nb, ed, kc, nx, ny, tstage, geo, UR);
          const Prim wl = primitives(UL, g1), wr = primitives(UR, g1);
          const bool okl = admissible(UL, wl), okr = admissible(UR, wr);
          double fn[4];
          if (okl && okr) {
            llf_flux(UL, UR, nx, ny, gamma, fn);
          } else {
            if (valid && lane_g == 0) record_error(sc, err_key(a.seq, kPassSurface, ed, kc));
#pragma unroll
            for (int m = 0; m < 4; ++m) fn[m] = 0.0;
          }
          const double wl_ = h * (left ? T.we[ko] : T.we[K - 1 - ko]);
#pragma unroll
          for (int mm = 0; mm < MG; ++mm) {
            const double f = (G == 1) ? fn[mm] : pick4(fn, m0 + mm);
            const double cf = left ? -(wl_ * f) : (wl_ * f);
#pragma unroll
            for (int j = 0; j < NP; ++j) acc[mm][j] = fma(cf, T.phe[q][ko][j], acc[mm][j]);
          }
        }
        if constexpr (MODE == kModeSurface) {
          if (valid) {
#pragma unroll
            for (int mm = 0; mm < MG; ++mm)
#pragma unroll
              for (int j = 0; j < NP; ++j)
                a.out[((static_cast<long long>(q) * 4 + m0 + mm) * NP + j) * ld + e] = acc[mm][j];
          }
        }
      }
    }

    // ------------------------------------------------------------ outputs
    if constexpr (MODE == kModeVolume) {
      if (valid) {
#pragma unroll
        for (int mm = 0; mm < MG; ++mm)
#pragma unroll
          for (int j = 0; j < NP; ++j) a.out[(static_cast<long long>(m0 + mm) * NP + j) * ld + e] = acc[mm][j];
      }
    } else if constexpr (MODE == kModeRhs) {
      const double idet = __ldg(geo.inv_det + e);
      if (valid) {
#pragma unroll
        for (int mm = 0; mm < MG; ++mm)
#pragma unroll
          for (int j = 0; j < NP; ++j)
            a.out[(static_cast<long long>(m0 + mm) * NP + j) * ld + e] = acc[mm][j] * idet;
      }
    } else if constexpr (MODE == kModeStage) {
      const double idet = __ldg(geo.inv_det + e);
      const double gdt = a.gcoef * dt;
      const double dt6 = dt / 6.0;
      const bool need_u = a.alpha != 0.0 || a.want_resid || a.kmode == 3;
#pragma unroll
      for (int mm = 0; mm < MG; ++mm) {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const long long idx = (static_cast<long long>(m0 + mm) * NP + j) * ld + e;
          const double d = acc[mm][j] * idet;
          const double uu = need_u ? __ldg(a.u + idx) : 0.0;
          double o;
          if (a.kmode == 3) {
            o = fma(dt6, __ldg(a.kacc + idx) + d, uu);
          } else {
            const double base = (a.alpha != 0.0) ? fma(a.alpha, uu, a.beta * c[mm][j]) : a.beta * c[mm][j];
            o = fma(gdt, d, base);
            if (a.kmode == 1 && valid) a.kacc[idx] = d;
            if (a.kmode == 2 && valid) a.kacc[idx] = fma(2.0, d, a.kacc[idx]);
          }
          if (valid) {
            a.out[idx] = o;
            if (a.want_resid) res_max = fmax(res_max, fabs(uu - o));
          }
          acc[mm][j] = o;  // keep the new stage for the CFL epilogue
        }
      }
      if (a.want_lambda) {
        double lam = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          double um[MG];
#pragma unroll
          for (int mm = 0; mm < MG; ++mm) {
            double s = T.phm[q][0] * acc[mm][0];
#pragma unroll
            for (int j = 1; j < NP; ++j) s = fma(T.phm[q][j], acc[mm][j], s);
            um[mm] = s;
          }
          double U[4];
          gather_state<G, MG>(um, U);
          const Prim w = primitives(U, g1);
          if (admissible(U, w)) {
            lam = fmax(lam, fabs(w.vx * snx[q] + w.vy * sny[q]) + sqrt(gamma * w.p * w.inv));
          } else if (valid && lane_g == 0) {
            record_error(sc, err_key(a.seq_next, kPassDt, __ldg(geo.ref_id + e), q + 1));
          }
        }
        if (valid) lam_min = fmin(lam_min, 2.0 * __ldg(geo.inradius + e) / ((2.0 * P + 1.0) * lam));
      }
    }
  }

  if constexpr (MODE == kModeStage) {
    const int par = a.step & 1;
    if (a.want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
    if (a.want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
  }
}

// stable_dt (solver.cpp:427-461) for a standalone call / the first step.
template <int P>
__device__ __forceinline__ void dt_body(const Tab<P>& T, const Geo& geo, const double* __restrict__ c, Scalars* sc,
                                        int slot, unsigned long long seq) {
  constexpr int NP = Dim<P>::NP;
  const long long ld = geo.ld;
  const double gamma = geo.gamma, g1 = gamma - 1.0;
  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < geo.ld; e += gridDim.x * blockDim.x) {
    if (e >= geo.N) continue;
    double lam = 0.0;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double U[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        double s = T.phm[q][0] * __ldg(c + (static_cast<long long>(m) * NP) * ld + e);
#pragma unroll
        for (int j = 1; j < NP; ++j) s = fma(T.phm[q][j], __ldg(c + (static_cast<long long>(m) * NP + j) * ld + e), s);
        U[m] = s;
      }
      const Prim w = primitives(U, g1);
      if (!admissible(U, w)) {
        record_error(sc, err_key(seq, kPassDt, __ldg(geo.ref_id + e), q + 1));
        continue;
      }
      const int ed = __ldg(geo.eid + q * ld + e);
      lam = fmax(lam, fabs(w.vx * __ldg(geo.enx + ed) + w.vy * __ldg(geo.eny + ed)) + sqrt(gamma * w.p * w.inv));
    }
    lam_min = fmin(lam_min, 2.0 * __ldg(geo.inradius + e) / ((2.0 * P + 1.0) * lam));
  }
  block_reduce_atomic<true>(lam_min, &sc->dtmin[slot]);
}

}  // namespace dgbk
