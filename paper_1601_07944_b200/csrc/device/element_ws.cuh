// Warp-specialised DMMA element kernel (p >= DGB_WS_MINP, modes RHS and stage).
//
// Warps come in groups of three working on the same 8-element tile: a TENSOR warp (role 0)
// issues every contraction (interpolation, projections, traces — DMMA) and the epilogue; two
// FLUX warps (roles 1, 2: the first and second point of each lane's pair) evaluate every
// pointwise nonlinear term (volume fluxes, ghost states, numerical fluxes).  In the single-warp kernel (element_mma.cuh) each warp alternates DMMA bursts with
// long dependent FP64 chains, so the tensor pipe idles whenever all resident warps are in
// their flux phase; here the tensor warp keeps the pipe busy with the next contraction while
// its partner evaluates the fluxes of the previous one.
//
// The two warps exchange items through lane-private shared-memory slots: lane (g, t) of both
// warps handles element g at points 2t, 2t+1 (the DMMA accumulator layout, which is also the A
// fragment of the following projection), so an item is written and read by the same lane
// index — no bank conflicts, no transposition.  Items are double-buffered and handed over with
// mbarriers (32 arrivals = one warp).  Per tile the tensor warp produces, in order,
//   X: U0 U1 T0 U2 T1 T2 ...   (interpolated states at point tiles / side traces)
// and consumes the flux warp's answers Y_k for X_k, never more than two items ahead:
//   produce X0, X1; then for k >= 2: consume Y_{k-2}, produce X_k; finally consume the rest.
#pragma once

#include "element_mma.cuh"

namespace dgbk {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  unsigned long long st;
  asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(b)) : "memory");
  (void)st;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}

template <int P>
struct WsDim {
  using D = MmaDim<P>;
  static constexpr int FR = 4 * D::KS * 32;
  static constexpr int kItem = 16 * 32;  // doubles of one exchange item (largest: traces / fr+fs)
  // per pair: own + neighbour staging, X[2] and Y[2] exchange buffers, 4 mbarriers (as doubles)
  static constexpr int kPairBuf = 2 * FR + 4 * kItem + 4;
  static constexpr int kNX = D::NTD + 3;  // items per tile
};

// Schedule of the X items of a tile: for k in [0, kNX), is it a volume point tile (and
// which) or a side (and which)?  Order: U0, U1, T0, U2, T1, T2, ... (sides interleaved after
// the first two point tiles so each side's neighbour column has time to land).
template <int NTD>
__device__ __forceinline__ void ws_item(int k, bool& vol, int& idx) {
  // positions of the sides: 2, 4, 5 for NTD = 3; generically: sides at 2, 4, 6.. until the
  // point tiles run out, then the rest
  int nu = 0, ns = 0;
  for (int i = 0; i <= k; ++i) {
    const bool side_slot = (i >= 2) && ((i % 2 == 0) || nu >= NTD) && ns < 3;
    const bool is_vol = !side_slot && nu < NTD;
    if (i == k) {
      vol = is_vol;
      idx = is_vol ? nu : ns;
      return;
    }
    if (is_vol) ++nu; else ++ns;
  }
}

template <int P, int MODE>
__device__ __forceinline__ void element_body_ws(const Tab<P>& T, const Geo& geo, const StageArgs& a,
                                                double* __restrict__ smem) {
  using D = MmaDim<P>;
  using W = WsDim<P>;
  constexpr int NP = D::NP, NQ = D::NQ, K = D::K, KS = D::KS, NT = D::NT, JT = D::JT, NTD = D::NTD;
  constexpr int FR = W::FR, IT = W::kItem, NX = W::kNX;
  const long long ld = geo.ld;
  const double gamma = geo.gamma, g1 = gamma - 1.0;
  Scalars* sc = a.sc;

  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  for (int i = threadIdx.x; i < D::kSize; i += blockDim.x) smem[i] = __ldg(geo.mma_tab + i);
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wib = threadIdx.x >> 5;
  // groups of three warps per tile: role 0 tensor warp, roles 1 and 2 flux warps (point
  // 2t + role - 1 of each lane's pair, so each flux warp has half the dependent chains)
  const int pair = wib / 3, role = wib - 3 * (wib / 3);
  double* __restrict__ pbuf = smem + D::kSize + pair * W::kPairBuf;
  double* __restrict__ w_own = pbuf;
  double* __restrict__ w_nbr = pbuf + FR;
  double* __restrict__ xb = pbuf + 2 * FR;        // [2][IT]
  double* __restrict__ yb = xb + 2 * IT;          // [2][IT]
  unsigned long long* mb = reinterpret_cast<unsigned long long*>(yb + 2 * IT);  // mf[2], fm[2]
  if (role == 0 && lane == 0) {
    mbar_init(mb + 0, 32);  // X ready: the tensor warp's 32 lanes
    mbar_init(mb + 1, 32);
    mbar_init(mb + 2, 64);  // Y ready: both flux warps
    mbar_init(mb + 3, 64);
  }
  __syncthreads();
  if (s_stop) return;

  double t0 = a.t_host, dt = 0.0;
  if constexpr (MODE == kModeStage) {
    if (!mma_prologue(a, sc, t0, dt)) return;
  }
  const double tstage = (MODE == kModeStage) ? fma(a.tcoef, dt, t0) : t0;

  const int npairs = gridDim.x * (blockDim.x / 96);
  const int pg = blockIdx.x * (blockDim.x / 96) + pair;
  const int ntiles = (a.e1 - a.e0 + 7) >> 3;
  auto elem_of = [&](int tile, bool& ok) {
    int e = a.e0 + tile * 8 + g;
    ok = tile < ntiles && e < a.e1;
    return ok ? e : a.e1 - 1;
  };
  auto nbr_of = [&](int e, int q) { return __ldg(geo.nbr + q * ld + e); };

  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;
  unsigned nx_prod = 0, nx_cons = 0;  // X / Y item counters (each warp uses the pair it owns)

  if (role == 0) {
    // =================================================================== tensor warp
    int nbq[3] = {-4, -4, -4};
    {
      bool ok;
      const int e = elem_of(pg, ok);
      fetch_frag<NP, KS>(w_own, a.in, ld, e, ok, lane, t);
#pragma unroll
      for (int q = 0; q < 3; ++q) nbq[q] = nbr_of(e, q);
      fetch_frag<NP, KS>(w_nbr, a.in, ld, nbq[0], ok && nbq[0] >= 0, lane, t);
      cp_async_commit();
    }
    for (int tile = pg; tile < ntiles; tile += npairs) {
      bool valid;
      const int e = elem_of(tile, valid);
      bool nvalid;
      const int e_next = elem_of(tile + npairs, nvalid);
      int nbn[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) nbn[q] = nbr_of(e_next, q);
      const int inf = __ldg(geo.info + e);
      cp_async_wait<0>();
      __syncwarp();
      double R[4][JT][2];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int jt = 0; jt < JT; ++jt) R[m][jt][0] = R[m][jt][1] = 0.0;

      int side_done = 0;  // sides whose neighbour column has been consumed
      auto produce = [&](int k) {
        bool vol;
        int idx;
        ws_item<NTD>(k, vol, idx);
        const int b = nx_prod & 1;
        double* __restrict__ x = xb + b * IT;
        if (vol) {
          double u[4][2];
#pragma unroll
          for (int m = 0; m < 4; ++m) u[m][0] = u[m][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const double bb = smem[D::kPhi + (ks * NT + idx) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(u[m], w_own[(m * KS + ks) * 32 + lane], bb);
          }
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int i = 0; i < 2; ++i) x[(m * 2 + i) * 32 + lane] = u[m][i];
        } else {
          const int q = idx;
          if (q > 0) cp_async_wait<0>();  // this side's neighbour column
          double tw[4][2], tn[4][2];
#pragma unroll
          for (int m = 0; m < 4; ++m) tw[m][0] = tw[m][1] = tn[m][0] = tn[m][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const double bb = smem[D::kPhe + (q * KS + ks) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(tw[m], w_own[(m * KS + ks) * 32 + lane], bb);
          }
          const int snb = nbq[q] < 0 ? 0 : ((inf >> (2 * q)) & 3);
          unsigned todo = __reduce_or_sync(0xffffffffu, snb ? (1u << snb) : 0u);
          while (todo) {
            const int s = __ffs(todo) - 1;
            todo &= todo - 1;
            const bool mine = snb == s;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              const double bb = smem[D::kPheR + ((s - 1) * KS + ks) * 32 + lane];
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                const double an = w_nbr[(m * KS + ks) * 32 + lane];
                dmma(tn[m], mine ? an : 0.0, bb);
              }
            }
          }
          __syncwarp();
          // the neighbour buffer is consumed: next side (after side 2: the next tile's
          // side 0 and, the own buffer being free too, its own coefficients)
          if (q < 2) {
            const int nn = q == 0 ? nbq[1] : nbq[2];
            fetch_frag<NP, KS>(w_nbr, a.in, ld, nn, valid && nn >= 0, lane, t);
          } else {
            fetch_frag<NP, KS>(w_nbr, a.in, ld, nbn[0], nvalid && nbn[0] >= 0, lane, t);
          }
          cp_async_commit();
          ++side_done;
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              x[(m * 2 + i) * 32 + lane] = tw[m][i];
              x[((4 + m) * 2 + i) * 32 + lane] = tn[m][i];
            }
        }
        mbar_arrive(mb + b);  // mf[b]
        ++nx_prod;
      };
      auto consume = [&](int k) {
        bool vol;
        int idx;
        ws_item<NTD>(k, vol, idx);
        const int b = nx_cons & 1;
        mbar_wait(mb + 2 + b, (nx_cons >> 1) & 1);  // fm[b]
        const double* __restrict__ y = yb + b * IT;
        if (vol) {
          const int nt = idx;
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) {
              const double br = smem[D::kDr + ((nt * 2 + i) * JT + jt) * 32 + lane];
#pragma unroll
              for (int m = 0; m < 4; ++m) dmma(R[m][jt], y[(m * 2 + i) * 32 + lane], br);
            }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) {
              const double bs = smem[D::kDs + ((nt * 2 + i) * JT + jt) * 32 + lane];
#pragma unroll
              for (int m = 0; m < 4; ++m) dmma(R[m][jt], y[((4 + m) * 2 + i) * 32 + lane], bs);
            }
        } else {
          const int q = idx;
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) {
              const double bb = smem[D::kPheP + ((q * 2 + i) * JT + jt) * 32 + lane];
#pragma unroll
              for (int m = 0; m < 4; ++m) dmma(R[m][jt], y[(m * 2 + i) * 32 + lane], bb);
            }
        }
        ++nx_cons;
      };
      // the pipeline (at most two items ahead of the flux warp)
      produce(0);
      produce(1);
#pragma unroll 1
      for (int k = 2; k < NX; ++k) {
        consume(k - 2);
        produce(k);
      }
      consume(NX - 2);
      consume(NX - 1);
      (void)side_done;
      if constexpr (D::kTail1) {
        // the last interior point (NQ % 8 == 1): DFMAs by the tensor warp (see element_mma.cuh)
        constexpr int k = NQ - 1;
        const double ta = __ldg(geo.tau + e), tb = __ldg(geo.tau + ld + e);
        const double tc = __ldg(geo.tau + 2 * ld + e), td = __ldg(geo.tau + 3 * ld + e);
        double v[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          double sum = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) sum = fma(w_own[(m * KS + ks) * 32 + lane], smem[D::kTail + ks * 4 + t], sum);
          sum += __shfl_xor_sync(0xffffffffu, sum, 1);
          sum += __shfl_xor_sync(0xffffffffu, sum, 2);
          v[m] = sum;
        }
        Prim w = primitives(v, g1);
        if (!admissible(v, w)) {
          if (valid && t == 0) record_error(sc, err_key(a.seq, kPassVolume, __ldg(geo.ref_id + e), k));
          v[0] = 1.0; v[1] = 0.0; v[2] = 0.0; v[3] = 2.5;  // placeholder (solver.cpp:129-132)
          w.inv = 1.0; w.vx = 0.0; w.vy = 0.0; w.p = 1.0;
        }
        double fr[4], fs[4];
        contravariant_flux(v, w, ta, tb, tc, td, fr, fs);
#pragma unroll
        for (int jt = 0; jt < JT; ++jt)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int jj = 8 * jt + 2 * t + ii;
            const double dr = smem[D::kTail + KS * 4 + jj], ds = smem[D::kTail + KS * 4 + JT * 8 + jj];
#pragma unroll
            for (int m = 0; m < 4; ++m) R[m][jt][ii] = fma(dr, fr[m], fma(ds, fs[m], R[m][jt][ii]));
          }
      }
      // own buffer free (last use above): stage the next tile's coefficients
      __syncwarp();
      fetch_frag<NP, KS>(w_own, a.in, ld, e_next, nvalid, lane, t);
      cp_async_commit();
#pragma unroll
      for (int q = 0; q < 3; ++q) nbq[q] = nbn[q];

    // ------------------------------------------------------------ outputs (lane: element g, modes 8jt+2t+ii)
    if constexpr (MODE == kModeVolume || MODE == kModeRhs) {
      const double sc_ = (MODE == kModeRhs) ? __ldg(geo.inv_det + e) : 1.0;
      if (valid) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int jt = 0; jt < JT; ++jt)
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              const int j = 8 * jt + 2 * t + ii;
              if (j < NP) a.out[(static_cast<long long>(m) * NP + j) * ld + e] = R[m][jt][ii] * sc_;
            }
      }
    } else if constexpr (MODE == kModeStage) {
      const double idet = __ldg(geo.inv_det + e);
      const double gdt = a.gcoef * dt;
      const double dt6 = dt / 6.0;
      const bool need_u = a.alpha != 0.0 || a.want_resid || a.kmode == 3;
      const bool need_c = a.kmode != 3 && a.beta != 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        // this variable's u^n, stage input and RK4 accumulator: every load issued
        // before any store, so one memory latency per variable
        double uv[JT][2], cv[JT][2], kv[JT][2];
#pragma unroll
        for (int jt = 0; jt < JT; ++jt)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int j = 8 * jt + 2 * t + ii;
            const long long idx = (static_cast<long long>(m) * NP + j) * ld + e;
            uv[jt][ii] = (need_u && j < NP) ? __ldg(a.u + idx) : 0.0;
            cv[jt][ii] = (need_c && j < NP) ? __ldg(a.in + idx) : 0.0;
            kv[jt][ii] = ((a.kmode == 2 || a.kmode == 3) && j < NP) ? a.kacc[idx] : 0.0;
          }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int j = 8 * jt + 2 * t + ii;
            if (j < NP) {
              const long long idx = (static_cast<long long>(m) * NP + j) * ld + e;
              const double d = R[m][jt][ii] * idet;
              const double uu = uv[jt][ii], cj = cv[jt][ii];
              double o;
              if (a.kmode == 3) {
                o = fma(dt6, kv[jt][ii] + d, uu);
              } else {
                const double base = (a.alpha != 0.0) ? fma(a.alpha, uu, a.beta * cj) : a.beta * cj;
                o = fma(gdt, d, base);
                if (a.kmode == 1 && valid) a.kacc[idx] = d;
                if (a.kmode == 2 && valid) a.kacc[idx] = fma(2.0, d, kv[jt][ii]);
              }
              if (valid) {
                a.out[idx] = o;
                if (a.want_resid) res_max = fmax(res_max, fabs(uu - o));
              }
              R[m][jt][ii] = o;  // keep the new stage for the CFL epilogue / halo push
            } else {
              R[m][jt][ii] = 0.0;
            }
          }
      }
      if (a.push && valid && e >= geo.send_begin) {
        const int s0 = __ldg(geo.send_ptr + (e - geo.send_begin));
        const int s1 = __ldg(geo.send_ptr + (e - geo.send_begin) + 1);
        for (int sidx = s0; sidx < s1; ++sidx) {
          const int2 ent = __ldg(geo.send_ent + sidx);
          double* __restrict__ dst = a.peers->buf[ent.x][a.out_buf];
          const long long pld = a.peers->ld[ent.x];
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int jt = 0; jt < JT; ++jt)
#pragma unroll
              for (int ii = 0; ii < 2; ++ii) {
                const int j = 8 * jt + 2 * t + ii;
                if (j < NP) dst[(static_cast<long long>(m) * NP + j) * pld + ent.y] = R[m][jt][ii];
              }
        }
      }
      if (a.want_lambda) {
        // states at the 3 side midpoints: partial sums over this lane's modes, then
        // reduced over the 4 lanes of the element
        double v[3][4];
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            double s = 0.0;
#pragma unroll
            for (int jt = 0; jt < JT; ++jt)
#pragma unroll
              for (int ii = 0; ii < 2; ++ii) s = fma(smem[D::kPhm + q * JT * 8 + 8 * jt + 2 * t + ii], R[m][jt][ii], s);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            v[q][m] = s;
          }
        // lane t < 3 evaluates the wave speed at midpoint t
        double U[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) U[m] = t == 0 ? v[0][m] : (t == 1 ? v[1][m] : v[2][m]);
        const int qq = t < 3 ? t : 2;
        const int edq = __ldg(geo.eid + qq * ld + e);
        const Prim w = primitives(U, g1);
        double lam = 0.0;
        if (admissible(U, w)) {
          lam = fabs(w.vx * __ldg(geo.enx + edq) + w.vy * __ldg(geo.eny + edq)) + sqrt(gamma * w.p * w.inv);
        } else if (valid && t < 3) {
          record_error(sc, err_key(a.seq_next, kPassDt, __ldg(geo.ref_id + e), t + 1));
        }
        if (t == 3) lam = 0.0;
        lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, 1));
        lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, 2));
        if (valid && t == 0) lam_min = fmin(lam_min, 2.0 * __ldg(geo.inradius + e) / ((2.0 * P + 1.0) * lam));
      }
    }
    }  // tile loop (tensor warp)
  } else {
    // =================================================================== flux warp
    unsigned kk = 0;
    for (int tile = pg; tile < ntiles; tile += npairs) {
      bool valid;
      const int e = elem_of(tile, valid);
      const double ta = __ldg(geo.tau + e), tb = __ldg(geo.tau + ld + e);
      const double tc = __ldg(geo.tau + 2 * ld + e), td = __ldg(geo.tau + 3 * ld + e);
      const int inf = __ldg(geo.info + e);
      int nbs[3], eds[3];
      double enx[3], eny[3], eh[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        nbs[q] = nbr_of(e, q);
        eds[q] = __ldg(geo.eid + q * ld + e);
        enx[q] = __ldg(geo.enx + eds[q]);
        eny[q] = __ldg(geo.eny + eds[q]);
        eh[q] = __ldg(geo.eh + eds[q]);
      }
#pragma unroll 1
      for (int k = 0; k < NX; ++k) {
        bool vol;
        int idx;
        ws_item<NTD>(k, vol, idx);
        const int b = kk & 1;
        mbar_wait(mb + b, (kk >> 1) & 1);  // mf[b]: X_k is ready
        const double* __restrict__ x = xb + b * IT;
        double* __restrict__ y = yb + b * IT;
        if (vol) {
          const int nt = idx;
          {
            const int i = role - 1;
            const int kq = 8 * nt + 2 * t + i;
            double v[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) v[m] = x[(m * 2 + i) * 32 + lane];
            Prim w = primitives(v, g1);
            const bool bad = !admissible(v, w);
            if (bad && valid && kq < NQ) record_error(sc, err_key(a.seq, kPassVolume, __ldg(geo.ref_id + e), kq));
            if (bad) {  // placeholder (solver.cpp:129-132)
              v[0] = 1.0; v[1] = 0.0; v[2] = 0.0; v[3] = 2.5;
              w.inv = 1.0; w.vx = 0.0; w.vy = 0.0; w.p = 1.0;
            }
            double r_[4], s_[4];
            contravariant_flux(v, w, ta, tb, tc, td, r_, s_);
            const bool live = kq < NQ;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              y[(m * 2 + i) * 32 + lane] = live ? r_[m] : 0.0;
              y[((4 + m) * 2 + i) * 32 + lane] = live ? s_[m] : 0.0;
            }
          }
        } else {
          const int q = idx;
          const int nb = q == 0 ? nbs[0] : (q == 1 ? nbs[1] : nbs[2]);
          const int ed = q == 0 ? eds[0] : (q == 1 ? eds[1] : eds[2]);
          const double nx = q == 0 ? enx[0] : (q == 1 ? enx[1] : enx[2]);
          const double ny = q == 0 ? eny[0] : (q == 1 ? eny[1] : eny[2]);
          const double h = q == 0 ? eh[0] : (q == 1 ? eh[1] : eh[2]);
          const bool left = (inf >> (6 + q)) & 1;
          const bool bnd = nb < 0;
          {
            const int i = role - 1;
            const int ko = 2 * t + i;
            double UL[4], UR[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double tw = x[(m * 2 + i) * 32 + lane], tn = x[((4 + m) * 2 + i) * 32 + lane];
              UL[m] = left ? tw : tn;
              UR[m] = left ? tn : tw;
            }
            const int kc = left ? ko : K - 1 - ko;  // canonical (left-element) point index
            const bool live = ko < K;
            if (bnd && live) ghost_state<K>(UL, nb, ed, kc, nx, ny, tstage, geo, UR);
            const Prim wl = primitives(UL, g1), wr = primitives(UR, g1);
            double f[4];
            if (admissible(UL, wl) && admissible(UR, wr)) {
              num_flux(geo.flux, UL, wl, UR, wr, nx, ny, gamma, f);
            } else {
              if (valid && live) record_error(sc, err_key(a.seq, kPassSurface, ed, kc));
#pragma unroll
              for (int m = 0; m < 4; ++m) f[m] = 0.0;
            }
            const double wh = live ? h * smem[D::kWe + (kc < 8 ? kc : 0)] : 0.0;
#pragma unroll
            for (int m = 0; m < 4; ++m) y[(m * 2 + i) * 32 + lane] = left ? -(wh * f[m]) : (wh * f[m]);
          }
        }
        mbar_arrive(mb + 2 + b);  // fm[b]: Y_k is ready (and X_k consumed)
        ++kk;
      }
    }
  }
  cp_async_wait<0>();

  if constexpr (MODE == kModeStage) {
    const int par = a.step & 1;
    if (a.want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
    if (a.want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
    if (a.push) __threadfence_system();
  }
}

}  // namespace dgbk
