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

// std::max / std::min / std::clamp(x, 0, 1) as the reference evaluates them (plain
// compare-and-select): fmax/fmin carry NaN-propagation fix-ups (~6 instructions each on
// sm_100a), and the limiter's extreme searches are most of its instruction stream.
__device__ __forceinline__ double std_max(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double std_min(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double std_clamp01(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }

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

// Branch-free reciprocal / square root for the pointwise physics: the MUFU seed
// (rcp/rsqrt.approx.ftz.f64) refined by Newton steps to within ~1 ulp.  The IEEE
// `1.0 / x` and `sqrt(x)` carry a slow-path branch each and cost 8.5 / 14 DFMA
// slots (measured, profiles/r01_dmma_peak.txt); the flux evaluates 2 of each per
// edge point.  Arguments are positive whenever the state is admissible (the only
// case whose result is used); ~1 ulp differences are far inside the 1e-12 bar.
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// One Newton step on the 2^-20 MUFU seed (2^-40), then the square-root correction s + (a - s^2)
// y / 2 (2^-80 before rounding): equal to IEEE sqrt on all 1.2e9 log-uniform samples in
// [1e-6, 1e6] (tools/micro/mufu_prec.cu, profiles/r02_mufu_prec.txt), as was the two-step form.
__device__ __forceinline__ double sqrt_nr(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  const double s = a * y;
  return fma(0.5 * y, fma(-s, s, a), s);
}

struct Prim {
  double inv, vx, vy, p;
};

// EOS (euler.hpp:29-31) through one reciprocal per state.
__device__ __forceinline__ Prim primitives(const double (&U)[4], double g1) {
  Prim w;
  w.inv = rcp_nr(U[0]);
  w.vx = U[1] * w.inv;
  w.vy = U[2] * w.inv;
  w.p = g1 * (U[3] - 0.5 * (U[1] * w.vx + U[2] * w.vy));
  return w;
}

__device__ __forceinline__ bool admissible(const double (&U)[4], const Prim& w) { return U[0] > 0.0 && w.p > 0.0; }

// CFL wave speed |v.n| + c at a side midpoint with the reference's own operations
// (max_wave_speed / sound_speed / pressure, euler.hpp:29-55): IEEE division and square
// root, no Newton approximations, so the time step carries no approximation error
// relative to stable_dt (solver.cpp:427-461).  `ok` = admissible(u) as the reference
// tests it before the wave speed.
__device__ __forceinline__ double wave_speed_ieee(const double (&U)[4], double nx, double ny, double gamma, bool& ok) {
  const double p = (gamma - 1.0) * (U[3] - 0.5 * (U[1] * U[1] + U[2] * U[2]) / U[0]);
  ok = U[0] > 0.0 && p > 0.0;
  const double vn = (U[1] * nx + U[2] * ny) / U[0];
  return fabs(vn) + sqrt(gamma * p / U[0]);
}

// Contravariant fluxes fr = ta F1 + tb F2, fs = tc F1 + td F2 of the analytic flux
// (euler.hpp:43-50) through the contravariant velocities: 16 FP64 operations instead of
// forming F1, F2 and rotating them (26).
__device__ __forceinline__ void contravariant_flux(const double (&U)[4], const Prim& w, double ta, double tb, double tc,
                                                   double td, double (&fr)[4], double (&fs)[4]) {
  const double Vr = fma(ta, w.vx, tb * w.vy), Vs = fma(tc, w.vx, td * w.vy);
  const double ep = U[3] + w.p;
  fr[0] = fma(ta, U[1], tb * U[2]);
  fr[1] = fma(U[1], Vr, ta * w.p);
  fr[2] = fma(U[2], Vr, tb * w.p);
  fr[3] = ep * Vr;
  fs[0] = fma(tc, U[1], td * U[2]);
  fs[1] = fma(U[1], Vs, tc * w.p);
  fs[2] = fma(U[2], Vs, td * w.p);
  fs[3] = ep * Vs;
}

// Normal flux F(U).n and normal velocity.
__device__ __forceinline__ void normal_flux(const double (&U)[4], const Prim& w, double nx, double ny, double& vn,
                                            double (&f)[4]) {
  vn = fma(w.vx, nx, w.vy * ny);
  f[0] = fma(U[1], nx, U[2] * ny);
  f[1] = fma(U[1], vn, w.p * nx);
  f[2] = fma(U[2], vn, w.p * ny);
  f[3] = (U[3] + w.p) * vn;
}

// Local Lax-Friedrichs flux, normal from left to right (euler.hpp:59-71), on
// precomputed primitives: 0.5 (F(UL).n + F(UR).n) - 0.5 max(s_L, s_R) (UR - UL).
__device__ __forceinline__ void llf_flux(const double (&UL)[4], const Prim& wl, const double (&UR)[4], const Prim& wr,
                                         double nx, double ny, double gamma, double (&fn)[4]) {
  double fl[4], fr[4], vnl, vnr;
  normal_flux(UL, wl, nx, ny, vnl, fl);
  normal_flux(UR, wr, nx, ny, vnr, fr);
  const double sl = fabs(vnl) + sqrt_nr(gamma * wl.p * wl.inv);
  const double sr = fabs(vnr) + sqrt_nr(gamma * wr.p * wr.inv);
  const double hs = 0.5 * std_max(sl, sr);  // std::max as euler.hpp:64
#pragma unroll
  for (int m = 0; m < 4; ++m) fn[m] = fma(0.5, fl[m] + fr[m], -hs * (UR[m] - UL[m]));
}

// Roe flux with Harten's entropy fix on the acoustic waves (delta = 0.1 c~); not in the
// reference (it has LLF only) — same formulas as the oracle's roe() (oracle/dg2d_oracle.c),
// on the precomputed primitives.
__device__ __forceinline__ void roe_flux(const double (&UL)[4], const Prim& wl, const double (&UR)[4], const Prim& wr,
                                         double nx, double ny, double gamma, double (&fn)[4]) {
  const double epl = UL[3] + wl.p, epr = UR[3] + wr.p;
  const double HL = epl * wl.inv, HR = epr * wr.inv;
  const double sl = sqrt_nr(UL[0]), sr = sqrt_nr(UR[0]);
  const double isum = rcp_nr(sl + sr);
  const double u = (sl * wl.vx + sr * wr.vx) * isum, v = (sl * wl.vy + sr * wr.vy) * isum;
  const double H = (sl * HL + sr * HR) * isum;
  const double q2 = u * u + v * v;
  const double c = sqrt_nr((gamma - 1.0) * (H - 0.5 * q2)), rho = sl * sr;
  const double ic2 = rcp_nr(c * c);
  const double qn = u * nx + v * ny;
  const double du = wr.vx - wl.vx, dv = wr.vy - wl.vy, dqn = du * nx + dv * ny;
  const double dut = du - dqn * nx, dvt = dv - dqn * ny;
  const double dr = UR[0] - UL[0], dp = wr.p - wl.p;
  const double a1 = 0.5 * (dp - rho * c * dqn) * ic2, a2 = dr - dp * ic2, a3 = 0.5 * (dp + rho * c * dqn) * ic2;
  double l1 = fabs(qn - c), l3 = fabs(qn + c);
  const double l2 = fabs(qn), dd = 0.1 * c, i2d = 0.5 * rcp_nr(dd);
  if (l1 < dd) l1 = (l1 * l1 + dd * dd) * i2d;
  if (l3 < dd) l3 = (l3 * l3 + dd * dd) * i2d;
  const double b1 = l1 * a1, b2 = l2 * a2, b3 = l3 * a3, b4 = l2 * rho;
  const double D0 = b1 + b2 + b3;
  const double D1 = b1 * (u - c * nx) + b2 * u + b3 * (u + c * nx) + b4 * dut;
  const double D2 = b1 * (v - c * ny) + b2 * v + b3 * (v + c * ny) + b4 * dvt;
  const double D3 = b1 * (H - qn * c) + b2 * 0.5 * q2 + b3 * (H + qn * c) + b4 * (u * dut + v * dvt);
  double fl[4], fr[4], vnl, vnr;
  normal_flux(UL, wl, nx, ny, vnl, fl);
  normal_flux(UR, wr, nx, ny, vnr, fr);
  const double D[4] = {D0, D1, D2, D3};
#pragma unroll
  for (int m = 0; m < 4; ++m) fn[m] = 0.5 * ((fl[m] + fr[m]) - D[m]);
}

enum : int { kFluxLLF = 0, kFluxRoe = 1 };

// The numerical flux of the run, a template parameter of the element kernels: one
// instance per flux, so the LLF instance carries none of the Roe flux's registers
// (measured per stage: p=1 0.159 vs 0.175 ms, p=2 0.391 vs 0.421, p=4 1.046 vs 1.077).
template <int FLUX>
__device__ __forceinline__ void num_flux(const double (&UL)[4], const Prim& wl, const double (&UR)[4], const Prim& wr,
                                         double nx, double ny, double gamma, double (&fn)[4]) {
  if constexpr (FLUX == kFluxRoe)
    roe_flux(UL, wl, UR, wr, nx, ny, gamma, fn);
  else
    llf_flux(UL, wl, UR, wr, nx, ny, gamma, fn);
}

// The numerical flux times a signed quadrature weight w (-h w_k on the edge's left element, +h w_k
// on its right one).  LLF folds w into its two coefficients, cf = (w/2)(F(U_L).n + F(U_R).n) -
// (w hs)(U_R - U_L): 18 FP64 operations instead of 20 and no sign selects.  Exactly antisymmetric
// in the sign of w (IEEE negation commutes with products and fma), so the two elements of an edge
// still receive bitwise-opposite contributions.  Roe: w f.
template <int FLUX>
__device__ __forceinline__ void num_flux_w(const double (&UL)[4], const Prim& wl, const double (&UR)[4],
                                           const Prim& wr, double nx, double ny, double gamma, double w,
                                           double (&cf)[4]) {
  if constexpr (FLUX == kFluxRoe) {
    double f[4];
    roe_flux(UL, wl, UR, wr, nx, ny, gamma, f);
#pragma unroll
    for (int m = 0; m < 4; ++m) cf[m] = w * f[m];
  } else {
    double fl[4], fr[4], vnl, vnr;
    normal_flux(UL, wl, nx, ny, vnl, fl);
    normal_flux(UR, wr, nx, ny, vnr, fr);
    const double sl = fabs(vnl) + sqrt_nr(gamma * wl.p * wl.inv);
    const double sr = fabs(vnr) + sqrt_nr(gamma * wr.p * wr.inv);
    const double a = 0.5 * w, b = (0.5 * std_max(sl, sr)) * w;  // std::max as euler.hpp:64
#pragma unroll
    for (int m = 0; m < 4; ++m) cf[m] = fma(-b, UR[m] - UL[m], a * (fl[m] + fr[m]));
  }
}

// num_flux_w from the element's own view: UO = its own trace, UN = the neighbour's (or the
// ghost state), wmag = h w_k > 0, `left` = the element is the edge's left (canonical) element.
// LLF needs no orientation selects: with the canonical operands UL, UR = (UO, UN) or (UN, UO),
// F(UL).n + F(UR).n and max(s_L, s_R) are symmetric, U_R - U_L = +-(UN - UO) exactly, and
// fma(-p, q, c) = fma(p, -q, c) exactly, so cf = fma(hs wmag, UN - UO, +-(wmag/2)(F(UO).n + F(UN).n))
// is bitwise the value num_flux_w gives on the canonical operands.  Roe is not symmetric in its
// operand order and keeps the canonical selects.
template <int FLUX>
__device__ __forceinline__ void num_flux_own(const double (&UO)[4], const Prim& wo, const double (&UN)[4],
                                             const Prim& wn, double nx, double ny, double gamma, double wmag,
                                             bool left, double (&cf)[4]) {
  if constexpr (FLUX == kFluxRoe) {
    double UL[4], UR[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      UL[m] = left ? UO[m] : UN[m];
      UR[m] = left ? UN[m] : UO[m];
    }
    const Prim wl = left ? wo : wn, wr = left ? wn : wo;
    num_flux_w<FLUX>(UL, wl, UR, wr, nx, ny, gamma, left ? -wmag : wmag, cf);
  } else {
    double fo[4], fn[4], vno, vnn;
    normal_flux(UO, wo, nx, ny, vno, fo);
    normal_flux(UN, wn, nx, ny, vnn, fn);
    const double so = fabs(vno) + sqrt_nr(gamma * wo.p * wo.inv);
    const double sn = fabs(vnn) + sqrt_nr(gamma * wn.p * wn.inv);
    const double b = (0.5 * std_max(so, sn)) * wmag;  // std::max as euler.hpp:64
    const double a = left ? -(0.5 * wmag) : 0.5 * wmag;
#pragma unroll
    for (int m = 0; m < 4; ++m) cf[m] = fma(b, UN[m] - UO[m], a * (fo[m] + fn[m]));
  }
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

// cp.async of one double into shared memory (zero-filled when !pred); lane-private
// destinations, so the issuing lane's wait_group is the only synchronisation needed.
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool pred) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "r"(pred ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Cross-element software pipeline of the one-thread kernel (g1_element with PF): each thread
// owns shared-memory rows, row r at base[r * stride] (stride = blockDim.x: consecutive threads
// hit consecutive words, no bank conflicts).  Rows [0, 4NP) hold the element's own coefficient
// column, rows [4NP (1 + q), 4NP (2 + q)) the neighbour column of side q.  While element e is
// evaluated, the column of the thread's next element and, side by side as the slots free up,
// its neighbours' columns are in flight (cp.async, one commit group per slot, so every wait is
// wait_group 3: the slot needed now is the fourth-newest group).
struct G1Pipe {
  double* base;
  int stride;
  int e_next;     // next element of this thread (>= a.e1: none)
  int nb_next[3]; // its neighbours (BC code < 0: none)
};
template <int NP>
__device__ __forceinline__ void g1_fetch_col(const G1Pipe& pp, int slot, const double* __restrict__ in, long long ld,
                                             int col, bool ok) {
#pragma unroll
  for (int r = 0; r < 4 * NP; ++r)
    cp_async8(pp.base + (slot * 4 * NP + r) * pp.stride, ok ? in + static_cast<long long>(r) * ld + col : in, ok);
  cp_async_commit();
}

// neighbour_trace from the pipeline's shared-memory column (same FMA chain: bit-identical)
template <int P, int S>
__device__ __forceinline__ void neighbour_trace_s(const Tab<P>& T, const double* __restrict__ col, int stride,
                                                  double (&un)[Dim<P>::K][4]) {
  constexpr int NP = Dim<P>::NP, K = Dim<P>::K;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      const double cn = col[(mm * NP + j) * stride];
      const double p0 = T.phe[S][0][0] * cn;  // the mode-0 basis value is the same at every point
#pragma unroll
      for (int ko = 0; ko < K; ++ko) {
        const double ph = T.phe[S][K - 1 - ko][j];
        un[ko][mm] = (j == 0) ? p0 : fma(ph, cn, un[ko][mm]);
      }
    }
  }
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
      // the mode-0 basis value is the same double at every point (a constant function): one
      // product serves all K points, bit-identical to the per-point product
      const double p0 = T.phe[S][0][0] * cn;
#pragma unroll
      for (int ko = 0; ko < K; ++ko) {
        const double ph = T.phe[S][K - 1 - ko][j];
        un[ko][mm] = (j == 0) ? p0 : fma(ph, cn, un[ko][mm]);
      }
    }
  }
}

// 4x4 transpose across the 4 lanes of an element group: on entry lane g holds
// v[i] = (variable g) at point i; on exit lane g holds v[m] = (variable m) at
// point g.  Two butterfly rounds, 4 double shuffles.
__device__ __forceinline__ void transpose4(double (&v)[4], int g) {
  const bool b1 = g & 2, b0 = g & 1;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b1 ? v[i] : v[i + 2];
    const double r = __shfl_xor_sync(kFull, send, 2);
    if (b1) v[i] = r; else v[i + 2] = r;
  }
#pragma unroll
  for (int i = 0; i < 4; i += 2) {
    const double send = b0 ? v[i] : v[i + 1];
    const double r = __shfl_xor_sync(kFull, send, 1);
    if (b0) v[i] = r; else v[i + 1] = r;
  }
}

template <int K>
__device__ __forceinline__ double pick_weight(const double (&we)[K], int k) {
  double r = we[0];
#pragma unroll
  for (int i = 1; i < K; ++i) r = (k == i) ? we[i] : r;
  return r;
}

// Minimum registers per launch for the fused kernel (occupancy target per degree).
#ifndef DGB_MINB
#define DGB_MINB(P) ((P) == 1 ? 4 : (P) == 2 ? 3 : (P) == 3 ? 5 : (P) == 4 ? 4 : 3)  // p=1 0.129 vs 0.132 ms at 5, p=2 0.323 vs 0.328 at 4
#endif
#ifndef DGB_G1_SIDE_UNROLL
#define DGB_G1_SIDE_UNROLL 1  // sides of the one-thread-per-element kernel: runtime loop
#endif
constexpr int kG1SideUnroll = DGB_G1_SIDE_UNROLL;
#ifndef DGB_G1_MAXP
#define DGB_G1_MAXP 2
#endif
#ifndef DGB_G1_SIDE_PREFETCH
#define DGB_G1_SIDE_PREFETCH 1
#endif
#ifndef DGB_G1_RELOAD_MINP
// one-thread kernel, degrees >= this: re-read the coefficients after the volume integral
// instead of keeping them in registers (measured per stage: p=2 0.428 vs 0.446 ms, fewer
// spills; p=1 0.189 vs 0.182 ms, so p=1 keeps them)
#define DGB_G1_RELOAD_MINP 2
#endif
// Read-only global load the compiler may not merge with an earlier load of the same
// address (so a value can be re-read instead of being kept live in registers).
__device__ __forceinline__ double ld_nc(const double* p) {
  double r;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
#ifndef DGB_TRACE_P
// degrees with trace-buffer stage instances (kVarTrace) and the epilogue's trace write; measured
// per stage (interleaved, element-major traces): p=5 1.387 vs 1.549 ms, p=4 0.848 vs 0.980, p=3
// 0.657 vs 0.665, p=2 (one-thread kernel, large meshes) 0.281 vs 0.286; p=1 0.170 vs 0.117 (the
// trace bytes outweigh the three 12-row gathers they replace), so p=1 interpolates
#define DGB_TRACE_P(P) ((P) >= 2)
#endif
#ifndef DGB_G1_OWN_TRACE_READ
#define DGB_G1_OWN_TRACE_READ 1  // p=2: own traces read 0.281 ms, re-interpolated from the coefficients 0.304
#endif
#ifndef DGB_G1_HOIST_MAXP
#define DGB_G1_HOIST_MAXP 2  // one-thread kernel: mode-0 products formed once per variable (not per point)
#endif
#ifndef DGB_G1_PF_MAXP
#define DGB_G1_PF_MAXP 0  // one-thread kernel degrees with the cross-element pipeline (G1Pipe); measured at p=1:
                          // 0.161 vs 0.127 ms per stage (spills, L1 reduced to 64 KB): off
#endif
// Whether element_body_g1 runs the cross-element shared-memory pipeline (every mode that
// reads neighbour columns: the volume mode has no side loop to keep the group count).
template <int P, int MODE>
struct G1Prefetch {
  static constexpr bool value = P <= DGB_G1_PF_MAXP && MODE != kModeVolume;
};
// shared memory of the pipeline per thread (bytes): own column + three neighbour columns
template <int P>
constexpr int g1_pipe_bytes() {
  return G1Prefetch<P, kModeStage>::value ? 4 * 4 * Dim<P>::NP * 8 : 0;
}
// Degrees up to DGB_G1_MAXP use one thread per element, higher ones four lanes.
template <int P>
struct Lanes {
  static constexpr int value = P <= DGB_G1_MAXP ? 1 : 4;
};

#ifndef DGB_SIDE_UNROLL
#define DGB_SIDE_UNROLL 1
#endif
constexpr int kSideUnroll = DGB_SIDE_UNROLL;  // 1: sides processed in a runtime loop
#ifndef DGB_VOL_UNROLL
#define DGB_VOL_UNROLL 1
#endif
constexpr int kVolUnroll = DGB_VOL_UNROLL;  // 1: volume point groups in a runtime loop

template <int P>
struct MinBlocks {
  static constexpr int value = DGB_MINB(P);
};

// Stage prologue shared by the element kernels: step bookkeeping, stop rules, dt.
// Returns false when the step must not run (a stop rule fired).
__device__ __forceinline__ bool stage_prologue(const StageArgs& a, Scalars* sc, double& t0, double& dt) {
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
      return false;
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
  return true;
}

// The fused element kernel.  Four lanes per element, lane g owns conserved
// variable g (its n_p coefficients and accumulators).  Contractions are DFMA
// chains with constant-bank table operands (all lanes of a warp use the same
// table entry); every nonlinear pointwise evaluation (volume flux, numerical
// flux, wave speed) is done ONCE per point: the four lanes transpose four
// points' states, each lane evaluates one point, and the results are
// transposed back.  MODE selects what is written:
//   kModeVolume  -> volume integral only (eval_volume_pass)
//   kModeSurface -> per-side surface integrals into the slot buffer (eval_surface_pass)
//   kModeRhs     -> (volume + surface) / det (compute_rhs)
//   kModeStage   -> RK stage update with the fused epilogues
// The work of one element in the four-lane form (lane g = conserved variable g): element_body
// grid-strides over it, the fused latency-form stage + limiter kernel (kernels_p1.cu) calls it
// per scheduled 8-element subtile.
template <int P, int MODE, int FLUX, int VAR>
__device__ __forceinline__ void g4_element(const Tab<P>& T, const Geo& geo, const StageArgs& a, int e, bool valid,
                                           int g, double dt, double tstage, double& lam_min, double& res_max) {
  constexpr int NP = Dim<P>::NP, NQ = Dim<P>::NQ, K = Dim<P>::K;
  const long long ld = geo.ld;
  const double gamma = geo.gamma, g1 = gamma - 1.0;
  Scalars* sc = a.sc;
  constexpr bool RK4 = VAR & kVarRk4, LAM = VAR & kVarLambda, BND = VAR & kVarBoundary;
  const int kmode = RK4 ? a.kmode : 0;
  const bool want_lambda = LAM && a.want_lambda;
  {
  const long long row = static_cast<long long>(g) * NP * ld + e;  // (g, j=0, e)

  double c[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) c[j] = __ldg(a.in + row + j * ld);
  double acc[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) acc[j] = 0.0;

  // ------------------------------------------------------------ volume
  if constexpr (MODE != kModeSurface) {
    const double ta = __ldg(geo.tau + e), tb = __ldg(geo.tau + ld + e);
    const double tc = __ldg(geo.tau + 2 * ld + e), td = __ldg(geo.tau + 3 * ld + e);
#pragma unroll kVolUnroll
    for (int k0 = 0; k0 < NQ; k0 += 4) {
      const int nk = (NQ - k0) < 4 ? (NQ - k0) : 4;
      double v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nk) {
          double s = T.phi[k0 + i][0] * c[0];
#pragma unroll
          for (int j = 1; j < NP; ++j) s = fma(T.phi[k0 + i][j], c[j], s);
          v[i] = s;
        } else {
          v[i] = v[0];  // padding lane: duplicate of a real point
        }
      }
      transpose4(v, g);  // lane g: full state at point k0 + g
      Prim w = primitives(v, g1);
      if (!admissible(v, w)) {
        if (valid && g < nk) record_error(sc, err_key(a.seq, kPassVolume, __ldg(geo.ref_id + e), k0 + g));
        v[0] = 1.0; v[1] = 0.0; v[2] = 0.0; v[3] = 2.5;  // placeholder (solver.cpp:129-132)
        w.inv = 1.0; w.vx = 0.0; w.vy = 0.0; w.p = 1.0;
      }
      double fr[4], fs[4];  // contravariant fluxes along r and s
      contravariant_flux(v, w, ta, tb, tc, td, fr, fs);
      transpose4(fr, g);  // lane g: variable g at points k0..k0+3
      transpose4(fs, g);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < nk) {
#pragma unroll
          for (int j = 0; j < NP; ++j) acc[j] = fma(T.drw[k0 + i][j], fr[i], fma(T.dsw[k0 + i][j], fs[i], acc[j]));
        }
      }
    }
  }

  // ------------------------------------------------------------ surface
  double snx[3], sny[3];
  if constexpr (MODE != kModeVolume) {
    const int inf = __ldg(geo.info + e);
#pragma unroll kSideUnroll
    for (int q = 0; q < 3; ++q) {
      const int nb = __ldg(geo.nbr + q * ld + e);
      const int ed = __ldg(geo.eid + q * ld + e);
      const int snb = (inf >> (2 * q)) & 3;
      const bool left = (inf >> (6 + q)) & 1;
      const double nx = __ldg(geo.enx + ed), ny = __ldg(geo.eny + ed), h = __ldg(geo.eh + ed);
      snx[q] = nx;
      sny[q] = ny;
      const bool bnd = nb < 0;

      double un[K][1];
      if (!bnd) {
        switch (snb) {
          case 1: neighbour_trace<P, 0, 1>(T, a.in, ld, g, nb, un); break;
          case 2: neighbour_trace<P, 1, 1>(T, a.in, ld, g, nb, un); break;
          default: neighbour_trace<P, 2, 1>(T, a.in, ld, g, nb, un); break;
        }
      } else {
#pragma unroll
        for (int ko = 0; ko < K; ++ko) un[ko][0] = 0.0;
      }
      double uo[K];
#pragma unroll
      for (int ko = 0; ko < K; ++ko) {
        double s = T.phe[q][ko][0] * c[0];
#pragma unroll
        for (int j = 1; j < NP; ++j) s = fma(T.phe[q][ko][j], c[j], s);
        uo[ko] = s;
      }
      if constexpr (MODE == kModeSurface) {
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[j] = 0.0;
      }
#pragma unroll
      for (int k0 = 0; k0 < K; k0 += 4) {
        const int nk = (K - k0) < 4 ? (K - k0) : 4;
        double UO[4], UN[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ko = (i < nk) ? k0 + i : k0;
          UO[i] = uo[ko];
          UN[i] = un[ko][0];
        }
        transpose4(UO, g);  // lane g: full traces at own point k0 + g
        transpose4(UN, g);
        const int ko = (g < nk) ? k0 + g : k0;
        const int kc = left ? ko : K - 1 - ko;  // canonical (left-element) point index
        if (BND && bnd) ghost_state<K>(UO, nb, ed, kc, nx, ny, tstage, geo, UN);  // boundary: the element is left
        const Prim wo = primitives(UO, g1), wn = primitives(UN, g1);
        const double wl_ = h * pick_weight<K>(T.we, kc);
        double fn[4];
        if (admissible(UO, wo) && admissible(UN, wn)) {
          num_flux_own<FLUX>(UO, wo, UN, wn, nx, ny, gamma, wl_, left, fn);
        } else {
          if (valid && g < nk) record_error(sc, err_key(a.seq, kPassSurface, ed, kc));
#pragma unroll
          for (int m = 0; m < 4; ++m) fn[m] = 0.0;
        }
        transpose4(fn, g);  // lane g: weighted flux of variable g at points k0..k0+3
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (i < nk) {
#pragma unroll
            for (int j = 0; j < NP; ++j) acc[j] = fma(fn[i], T.phe[q][k0 + i][j], acc[j]);
          }
        }
      }
      if constexpr (MODE == kModeSurface) {
        if (valid) {
#pragma unroll
          for (int j = 0; j < NP; ++j) a.out[(static_cast<long long>(q) * 4 * NP + g * NP + j) * ld + e] = acc[j];
        }
      }
    }
  }

  // ------------------------------------------------------------ outputs
  if constexpr (MODE == kModeVolume) {
    if (valid) {
#pragma unroll
      for (int j = 0; j < NP; ++j) a.out[row + j * ld] = acc[j];
    }
  } else if constexpr (MODE == kModeRhs) {
    const double idet = __ldg(geo.inv_det + e);
    if (valid) {
#pragma unroll
      for (int j = 0; j < NP; ++j) a.out[row + j * ld] = acc[j] * idet;
    }
  } else if constexpr (MODE == kModeStage) {
    const double idet = __ldg(geo.inv_det + e);
    const double gdt = a.gcoef * dt;
    const double dt6 = dt / 6.0;
    const bool need_u = a.alpha != 0.0 || a.want_resid || kmode == 3;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const long long idx = row + j * ld;
      const double d = acc[j] * idet;
      const double uu = need_u ? __ldg(a.u + idx) : 0.0;
      double o;
      if (kmode == 3) {
        o = fma(dt6, __ldg(a.kacc + idx) + d, uu);
      } else {
        const double base = (a.alpha != 0.0) ? fma(a.alpha, uu, a.beta * c[j]) : a.beta * c[j];
        o = fma(gdt, d, base);
        if (kmode == 1 && valid) a.kacc[idx] = d;
        if (kmode == 2 && valid) a.kacc[idx] = fma(2.0, d, a.kacc[idx]);
      }
      if (valid) {
        a.out[idx] = o;
        if (a.want_resid) res_max = std_max(res_max, fabs(uu - o));
      }
      acc[j] = o;  // keep the new stage for the CFL epilogue
    }
    if (a.means && valid) a.means[4 * static_cast<long long>(e) + g] = acc[0];
    if (want_lambda) {
      double v[4];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        double s = T.phm[q][0] * acc[0];
#pragma unroll
        for (int j = 1; j < NP; ++j) s = fma(T.phm[q][j], acc[j], s);
        v[q] = s;
      }
      v[3] = v[0];
      transpose4(v, g);  // lane q < 3: state at the midpoint of side q
      const double nxq = g == 0 ? snx[0] : (g == 1 ? snx[1] : snx[2]);
      const double nyq = g == 0 ? sny[0] : (g == 1 ? sny[1] : sny[2]);
      double lam = 0.0;
      bool ok;
      const double ws = wave_speed_ieee(v, nxq, nyq, gamma, ok);
      if (ok) {
        lam = ws;
      } else if (valid && g < 3) {
        record_error(sc, err_key(a.seq_next, kPassDt, __ldg(geo.ref_id + e), g + 1));
      }
      if (g == 3) lam = 0.0;
      lam = std_max(lam, __shfl_xor_sync(kFull, lam, 1));
      lam = std_max(lam, __shfl_xor_sync(kFull, lam, 2));
      if (valid && g == 0) lam_min = std_min(lam_min, 2.0 * __ldg(geo.inradius + e) / ((2.0 * P + 1.0) * lam));
    }
  }
  }
}

template <int P, int MODE, int FLUX, int VAR>
__device__ __forceinline__ void element_body(const Tab<P>& T, const Geo& geo, const StageArgs& a) {
  const int gsize = ((a.e1 - a.e0 + 31) & ~31) * 4;  // whole warps (8 elements each), whole blocks
  const int stride = gridDim.x * blockDim.x;
  Scalars* sc = a.sc;
  constexpr bool LAM = VAR & kVarLambda;
  const bool want_lambda = LAM && a.want_lambda;

  // block-uniform early exit: an error or a stop rule fired in an earlier launch
  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  __syncthreads();
  if (s_stop) return;

  // ---- time and dt of this stage (every thread evaluates the same values)
  double t0 = a.t_host, dt = 0.0;
  if constexpr (MODE == kModeStage) {
    if (!stage_prologue(a, sc, t0, dt)) return;
  }
  const double tstage = (MODE == kModeStage) ? fma(a.tcoef, dt, t0) : t0;

  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;

  for (int tid = blockIdx.x * blockDim.x + threadIdx.x; tid < gsize; tid += stride) {
    const int g = tid & 3;  // conserved variable owned by this lane
    int e = a.e0 + (tid >> 2);
    const bool valid = e < a.e1;
    if (!valid) e = a.e1 - 1;
    g4_element<P, MODE, FLUX, VAR>(T, geo, a, e, valid, g, dt, tstage, lam_min, res_max);
  }

  if constexpr (MODE == kModeStage) {
    const int par = a.step & 1;
    if (want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
    if (a.want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
  }
}


// One thread per element (all four variables): the low-degree variant.  At
// p <= 2 the per-point work (reciprocals, square roots, shuffles) dominates the
// contractions, so spreading an element over lanes multiplies it; a thread per
// element evaluates every pointwise quantity exactly once with no exchange.
// The work of one element (one thread); element_body_g1 grid-strides over it, the fused
// stage + limiter kernel (kernels_p1.cu) calls it per scheduled tile.
template <int P, int MODE, int FLUX, int VAR, bool PF = false>
__device__ __forceinline__ void g1_element(const Tab<P>& T, const Geo& geo, const StageArgs& a, int e, double dt,
                                           double tstage, double& lam_min, double& res_max,
                                           const G1Pipe* pipe = nullptr) {
  constexpr int NP = Dim<P>::NP, NQ = Dim<P>::NQ, K = Dim<P>::K;
  const long long ld = geo.ld;
  const double gamma = geo.gamma, g1 = gamma - 1.0;
  Scalars* sc = a.sc;
  // instance variant (kernels_tu.cuh): paths the launch knows are unused compile away
  constexpr bool RK4 = VAR & kVarRk4, LAM = VAR & kVarLambda, BND = VAR & kVarBoundary;
  const int kmode = RK4 ? a.kmode : 0;
  const bool want_lambda = LAM && a.want_lambda;
  constexpr bool kHoist0 = P <= DGB_G1_HOIST_MAXP;
  // trace-buffer instance: the own and neighbour traces of the stage
  // input come from a.tr_in, element-major [e][side][var][point] (one contiguous 4K block per
  // side), instead of being interpolated from the coefficient columns
  constexpr bool kTrG = MODE == kModeStage && !PF && DGB_TRACE_P(P) && (VAR & kVarTrace) != 0;
  constexpr bool kTrOwn = kTrG && DGB_G1_OWN_TRACE_READ;  // own traces read too (else interpolated)
  constexpr int kTS = 12 * K;  // trace doubles per element
  {
    double c[4][NP];
    if constexpr (PF) {
      cp_async_wait<3>();  // this element's column (issued during the previous element)
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int j = 0; j < NP; ++j) c[m][j] = pipe->base[(m * NP + j) * pipe->stride];
      g1_fetch_col<NP>(*pipe, 0, a.in, ld, pipe->e_next, pipe->e_next < a.e1);
    } else {
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int j = 0; j < NP; ++j) c[m][j] = __ldg(a.in + (static_cast<long long>(m) * NP + j) * ld + e);
    }
    double acc[4][NP];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int j = 0; j < NP; ++j) acc[m][j] = 0.0;
#if DGB_G1_SIDE_PREFETCH
    // connectivity of the three sides, requested with the coefficients so that the side
    // loop's neighbour-column and normal loads do not wait for a dependent index load
    int nb3[3] = {0, 0, 0}, ed3[3] = {0, 0, 0}, inf0 = 0;
    if constexpr (MODE != kModeVolume) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        nb3[q] = __ldg(geo.nbr + q * ld + e);
        ed3[q] = __ldg(geo.eid + q * ld + e);
      }
      inf0 = __ldg(geo.info + e);
    }
#endif

    // mode-0 products of the interpolations and own traces (the mode-0 basis function is a
    // constant: every table holds the same double in column 0), formed once per variable
    double c0p[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) c0p[m] = kHoist0 ? T.phi[0][0] * c[m][0] : 0.0;
    // ------------------------------------------------------------ volume
    if constexpr (MODE != kModeSurface) {
      const double ta = __ldg(geo.tau + e), tb = __ldg(geo.tau + ld + e);
      const double tc = __ldg(geo.tau + 2 * ld + e), td = __ldg(geo.tau + 3 * ld + e);
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        double U[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          double s = kHoist0 ? c0p[m] : T.phi[k][0] * c[m][0];  // the same product at every point
#pragma unroll
          for (int j = 1; j < NP; ++j) s = fma(T.phi[k][j], c[m][j], s);
          U[m] = s;
        }
        Prim w = primitives(U, g1);
        if (!admissible(U, w)) {
          record_error(sc, err_key(a.seq, kPassVolume, __ldg(geo.ref_id + e), k));
          U[0] = 1.0; U[1] = 0.0; U[2] = 0.0; U[3] = 2.5;  // placeholder (solver.cpp:129-132)
          w.inv = 1.0; w.vx = 0.0; w.vy = 0.0; w.p = 1.0;
        }
        double fr[4], fs[4];  // contravariant fluxes along r and s
        contravariant_flux(U, w, ta, tb, tc, td, fr, fs);
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int j = 0; j < NP; ++j) acc[m][j] = fma(T.drw[k][j], fr[m], fma(T.dsw[k][j], fs[m], acc[m][j]));
      }
    }

    // ------------------------------------------------------------ surface
    if constexpr (MODE != kModeVolume) {
#if DGB_G1_SIDE_PREFETCH
      const int inf = inf0;
#else
      const int inf = __ldg(geo.info + e);
#endif
#pragma unroll kG1SideUnroll
      for (int q = 0; q < 3; ++q) {
#if DGB_G1_SIDE_PREFETCH
        const int nb = q == 0 ? nb3[0] : (q == 1 ? nb3[1] : nb3[2]);
        const int ed = q == 0 ? ed3[0] : (q == 1 ? ed3[1] : ed3[2]);
#else
        const int nb = __ldg(geo.nbr + q * ld + e);
        const int ed = __ldg(geo.eid + q * ld + e);
#endif
        const int snb = (inf >> (2 * q)) & 3;
        const bool left = (inf >> (6 + q)) & 1;
        const double nx = __ldg(geo.enx + ed), ny = __ldg(geo.eny + ed), h = __ldg(geo.eh + ed);
        const bool bnd = nb < 0;
        double un[K][4];
        double ut[4 * K];  // kTrG: this side's own traces [m][ko]
        if constexpr (kTrG) {
          if constexpr (kTrOwn) {
            const double2* ob = reinterpret_cast<const double2*>(a.tr_in + static_cast<long long>(e) * kTS + q * 4 * K);
#pragma unroll
            for (int i = 0; i < 2 * K; ++i) {
              const double2 v = __ldg(ob + i);
              ut[2 * i] = v.x;
              ut[2 * i + 1] = v.y;
            }
          }
          if (!bnd) {  // the neighbour's side block, its points reversed
            const double2* nbk =
                reinterpret_cast<const double2*>(a.tr_in + static_cast<long long>(nb) * kTS + (snb - 1) * 4 * K);
            double v4[4 * K];
#pragma unroll
            for (int i = 0; i < 2 * K; ++i) {
              const double2 v = __ldg(nbk + i);
              v4[2 * i] = v.x;
              v4[2 * i + 1] = v.y;
            }
#pragma unroll
            for (int ko = 0; ko < K; ++ko)
#pragma unroll
              for (int m = 0; m < 4; ++m) un[ko][m] = v4[m * K + (K - 1 - ko)];
          }
        } else if constexpr (PF) {
          cp_async_wait<3>();  // side q's neighbour column
          const double* col = pipe->base + (q + 1) * 4 * NP * pipe->stride;
          if (!bnd) {
            switch (snb) {
              case 1: neighbour_trace_s<P, 0>(T, col, pipe->stride, un); break;
              case 2: neighbour_trace_s<P, 1>(T, col, pipe->stride, un); break;
              default: neighbour_trace_s<P, 2>(T, col, pipe->stride, un); break;
            }
          }
          const int nbn = q == 0 ? pipe->nb_next[0] : (q == 1 ? pipe->nb_next[1] : pipe->nb_next[2]);
          g1_fetch_col<NP>(*pipe, q + 1, a.in, ld, nbn, pipe->e_next < a.e1 && nbn >= 0);
        } else if (!bnd) {
          switch (snb) {
            case 1: neighbour_trace<P, 0, 4>(T, a.in, ld, 0, nb, un); break;
            case 2: neighbour_trace<P, 1, 4>(T, a.in, ld, 0, nb, un); break;
            default: neighbour_trace<P, 2, 4>(T, a.in, ld, 0, nb, un); break;
          }
        }
        if (bnd) {
#pragma unroll
          for (int ko = 0; ko < K; ++ko)
#pragma unroll
            for (int m = 0; m < 4; ++m) un[ko][m] = 0.0;
        }
        if constexpr (MODE == kModeSurface) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int j = 0; j < NP; ++j) acc[m][j] = 0.0;
        }
        const double* __restrict__ phq = &T.phe[q][0][0];  // own side, uniform runtime offset
        constexpr bool kReload = P >= DGB_G1_RELOAD_MINP && !kTrOwn;
        // own trace of the side from a fresh (L1) read of the coefficients, so that they
        // need not stay in registers past the volume integral
        double uoa[K][4];
        if constexpr (kReload) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            const double cj = ld_nc(a.in + (static_cast<long long>(m) * NP + j) * ld + e);
            const double cj0 = phq[0] * cj;  // the mode-0 product, the same at every point
#pragma unroll
            for (int ko = 0; ko < K; ++ko) uoa[ko][m] = j == 0 ? cj0 : fma(phq[ko * NP + j], cj, uoa[ko][m]);
          }
        }
        double c0q[4];  // mode-0 products of the own trace, once per side (not kept across the loop)
#pragma unroll
        for (int m = 0; m < 4; ++m) c0q[m] = (kReload || !kHoist0 || kTrOwn) ? 0.0 : phq[0] * c[m][0];
#pragma unroll
        for (int ko = 0; ko < K; ++ko) {
          double uo[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            if constexpr (kTrOwn) {
              uo[m] = ut[m * K + ko];
            } else if constexpr (kReload) {
              uo[m] = uoa[ko][m];
            } else {
              double s = kHoist0 ? c0q[m] : phq[ko * NP] * c[m][0];
#pragma unroll
              for (int j = 1; j < NP; ++j) s = fma(phq[ko * NP + j], c[m][j], s);
              uo[m] = s;
            }
          }
          double UN[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) UN[m] = un[ko][m];
          const int kc = left ? ko : K - 1 - ko;
          if (BND && bnd) ghost_state<K>(uo, nb, ed, kc, nx, ny, tstage, geo, UN);  // boundary: the element is left
          const Prim wo = primitives(uo, g1), wn = primitives(UN, g1);
          const double wl_ = h * pick_weight<K>(T.we, kc);
          double cf[4];
          if (admissible(uo, wo) && admissible(UN, wn)) {
            num_flux_own<FLUX>(uo, wo, UN, wn, nx, ny, gamma, wl_, left, cf);
          } else {
            record_error(sc, err_key(a.seq, kPassSurface, ed, kc));
#pragma unroll
            for (int m = 0; m < 4; ++m) cf[m] = 0.0;
          }
#pragma unroll
          for (int m = 0; m < 4; ++m) {
#pragma unroll
            for (int j = 0; j < NP; ++j) acc[m][j] = fma(cf[m], phq[ko * NP + j], acc[m][j]);
          }
        }
        if constexpr (MODE == kModeSurface) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int j = 0; j < NP; ++j)
              a.out[((static_cast<long long>(q) * 4 + m) * NP + j) * ld + e] = acc[m][j];
        }
      }
    }

    // ------------------------------------------------------------ outputs
    if constexpr (MODE == kModeVolume) {
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int j = 0; j < NP; ++j) a.out[(static_cast<long long>(m) * NP + j) * ld + e] = acc[m][j];
    } else if constexpr (MODE == kModeRhs) {
      const double idet = __ldg(geo.inv_det + e);
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int j = 0; j < NP; ++j) a.out[(static_cast<long long>(m) * NP + j) * ld + e] = acc[m][j] * idet;
    } else if constexpr (MODE == kModeStage) {
      const double idet = __ldg(geo.inv_det + e);
      const double gdt = a.gcoef * dt;
      const double dt6 = dt / 6.0;
      const bool need_u = a.alpha != 0.0 || a.want_resid || kmode == 3;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const long long idx = (static_cast<long long>(m) * NP + j) * ld + e;
          const double d = acc[m][j] * idet;
          const double uu = need_u ? __ldg(a.u + idx) : 0.0;
          double o;
          if (kmode == 3) {
            o = fma(dt6, __ldg(a.kacc + idx) + d, uu);
          } else {
            const double cmj = (P >= DGB_G1_RELOAD_MINP) ? ld_nc(a.in + idx) : c[m][j];
            const double base = (a.alpha != 0.0) ? fma(a.alpha, uu, a.beta * cmj) : a.beta * cmj;
            o = fma(gdt, d, base);
            if (kmode == 1) a.kacc[idx] = d;
            if (kmode == 2) a.kacc[idx] = fma(2.0, d, a.kacc[idx]);
          }
          a.out[idx] = o;
          if (a.want_resid) res_max = std_max(res_max, fabs(uu - o));
          acc[m][j] = o;
        }
      }
      if constexpr (DGB_TRACE_P(P) && !PF) {
        if (a.tr_out) {
          // traces of the new stage for the next stage's kVarTrace instance: the own-trace chain of
          // the surface (mode-0 product, then the modes in order), side by side, one contiguous
          // 4K block per side
          double2* tb = reinterpret_cast<double2*>(a.tr_out + static_cast<long long>(e) * kTS);
#pragma unroll kG1SideUnroll
          for (int q = 0; q < 3; ++q) {
            const double* __restrict__ phq = &T.phe[q][0][0];
            double v4[4 * K];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double t0 = phq[0] * acc[m][0];
#pragma unroll
              for (int ko = 0; ko < K; ++ko) {
                double s = t0;
#pragma unroll
                for (int j = 1; j < NP; ++j) s = fma(phq[ko * NP + j], acc[m][j], s);
                v4[m * K + ko] = s;
              }
            }
#pragma unroll
            for (int i = 0; i < 2 * K; ++i) tb[q * 2 * K + i] = make_double2(v4[2 * i], v4[2 * i + 1]);
          }
        }
      }
      if (a.means) {  // the limiter's neighbour means as one 32-byte sector per element
        double2* mp = reinterpret_cast<double2*>(a.means + 4 * static_cast<long long>(e));
        mp[0] = make_double2(acc[0][0], acc[1][0]);
        mp[1] = make_double2(acc[2][0], acc[3][0]);
      }
      if (want_lambda) {
        double lam = 0.0;
        double a0[4];  // mode-0 products of the midpoint states (the same at the three midpoints)
#pragma unroll
        for (int m = 0; m < 4; ++m) a0[m] = T.phm[0][0] * acc[m][0];
#pragma unroll 1
        for (int q = 0; q < 3; ++q) {
          double U[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            double s = a0[m];
#pragma unroll
            for (int j = 1; j < NP; ++j) s = fma(T.phm[q][j], acc[m][j], s);
            U[m] = s;
          }
          const int ed = __ldg(geo.eid + q * ld + e);
          bool ok;
          const double ws = wave_speed_ieee(U, __ldg(geo.enx + ed), __ldg(geo.eny + ed), gamma, ok);
          if (ok) {
            lam = std_max(lam, ws);
          } else {
            record_error(sc, err_key(a.seq_next, kPassDt, __ldg(geo.ref_id + e), q + 1));
          }
        }
        lam_min = std_min(lam_min, 2.0 * __ldg(geo.inradius + e) / ((2.0 * P + 1.0) * lam));
      }
    }
  }
}

template <int P, int MODE, int FLUX, int VAR>
__device__ __forceinline__ void element_body_g1(const Tab<P>& T, const Geo& geo, const StageArgs& a) {
  const int stride = gridDim.x * blockDim.x;
  Scalars* sc = a.sc;
  constexpr bool LAM = VAR & kVarLambda;
  const bool want_lambda = LAM && a.want_lambda;

  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  __syncthreads();
  if (s_stop) return;

  double t0 = a.t_host, dt = 0.0;
  if constexpr (MODE == kModeStage) {
    if (!stage_prologue(a, sc, t0, dt)) return;
  }
  const double tstage = (MODE == kModeStage) ? fma(a.tcoef, dt, t0) : t0;

  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;

  if constexpr (G1Prefetch<P, MODE>::value) {
    // cross-element pipeline (G1Pipe): the first element's columns, then one element ahead
    extern __shared__ double pfbuf[];
    G1Pipe pp;
    pp.base = pfbuf + threadIdx.x;
    pp.stride = blockDim.x;
    const long long ld = geo.ld;
    constexpr int NP = Dim<P>::NP;
    int e = a.e0 + blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = e < a.e1;
    int nb[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) nb[q] = ok ? __ldg(geo.nbr + q * ld + e) : -1;
    g1_fetch_col<NP>(pp, 0, a.in, ld, e, ok);
#pragma unroll
    for (int q = 0; q < 3; ++q) g1_fetch_col<NP>(pp, q + 1, a.in, ld, nb[q], ok && nb[q] >= 0);
    for (; e < a.e1; e += stride) {
      pp.e_next = e + stride;
#pragma unroll
      for (int q = 0; q < 3; ++q) pp.nb_next[q] = pp.e_next < a.e1 ? __ldg(geo.nbr + q * ld + pp.e_next) : -1;
      g1_element<P, MODE, FLUX, VAR, true>(T, geo, a, e, dt, tstage, lam_min, res_max, &pp);
    }
    cp_async_wait<0>();
  } else {
    for (int e = a.e0 + blockIdx.x * blockDim.x + threadIdx.x; e < a.e1; e += stride)
      g1_element<P, MODE, FLUX, VAR>(T, geo, a, e, dt, tstage, lam_min, res_max);
  }

  if constexpr (MODE == kModeStage) {
    const int par = a.step & 1;
    if (want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
    if (a.want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
  }
}

// stable_dt (solver.cpp:427-461) for a standalone call / the first step.
template <int P>
__device__ __forceinline__ void dt_body(const Tab<P>& T, const Geo& geo, const double* __restrict__ c, Scalars* sc,
                                        int slot, unsigned long long seq) {
  constexpr int NP = Dim<P>::NP;
  const long long ld = geo.ld;
  const double gamma = geo.gamma;
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
      const int ed = __ldg(geo.eid + q * ld + e);
      bool ok;
      const double ws = wave_speed_ieee(U, __ldg(geo.enx + ed), __ldg(geo.eny + ed), gamma, ok);
      if (!ok) {
        record_error(sc, err_key(seq, kPassDt, __ldg(geo.ref_id + e), q + 1));
        continue;
      }
      lam = std_max(lam, ws);
    }
    lam_min = std_min(lam_min, 2.0 * __ldg(geo.inradius + e) / ((2.0 * P + 1.0) * lam));
  }
  block_reduce_atomic<true>(lam_min, &sc->dtmin[slot]);
}

}  // namespace dgbk
