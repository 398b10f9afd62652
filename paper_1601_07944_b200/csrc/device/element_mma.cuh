// FP64 tensor-core (DMMA) variant of the fused element kernel, used for p >= 3.
//
// Every contraction of the modal-DG stage is a small GEMM over a tile of 8
// elements (one warp):
//
//   interior interpolation   U_m[e][k]  = sum_j C_m[e][j] phi[k][j]          (8 x Q  <- 8 x Np . Np x Q)
//   volume projection        R_m[e][j] += sum_k Fr_m[e][k] w dphi/dr[k][j]   (8 x Np <- 8 x Q  . Q  x Np)
//                                        + Fs_m[e][k] w dphi/ds[k][j]
//   own / neighbour traces   T_m[e][k]  = sum_j C_m[e][j] phi_q[k][j]        (8 x K  <- 8 x Np . Np x K)
//   surface projection       R_m[e][j] -= sum_k Fn_m[e][k] phi_q[k][j]       (8 x Np <- 8 x K  . K  x Np)
//
// issued as mma.sync.m8n8k4 f64 (DMMA.8x8x4 on sm_100a: 256 FMAs per warp
// instruction, the same FP64 pipe as DFMA but an eighth of the issue slots and
// no register dependency chains).  Rows are the 8 elements of the warp, one
// accumulator set per conserved variable.  Lane (g, t) = (lane / 4, lane % 4)
// holds A[g][t], B[t][g] and D[g][2t], D[g][2t+1], so after an interpolation
// the lane owns element g at points 2t, 2t+1 of every 8-point tile — exactly
// what it needs to evaluate the nonlinear flux, and exactly the A fragment of
// the following projection once the k index of that projection is permuted
// (k-step (tile n, i) takes point 8n + 2t + i in slot t).  So no data moves
// between the contractions and the pointwise physics: the basis tables are
// stored in shared memory in that permuted fragment order (one LDS per DMMA).
//
// Both sides of an edge still evaluate the same numerical flux from bit-identical
// traces: the neighbour's trace is the same DMMA (same A row = the neighbour's
// coefficients, same B column = its side's basis row, same k order) as the one
// the neighbour performs for its own trace, and the flux is evaluated in the
// edge's canonical left -> right orientation.
#pragma once

#include "element_impl.cuh"

namespace dgbk {

#ifndef DGB_MMA_VOL_PIPE
#define DGB_MMA_VOL_PIPE(P) 1  // interpolate the next point tile while this tile's fluxes run
#endif
#ifndef DGB_MMA_SIDE_UNROLL
#define DGB_MMA_SIDE_UNROLL 1  // per-side surface loop (p = 5): runtime loop, 1.84 vs 1.91 ms unrolled
#endif
constexpr int kMmaSideUnroll = DGB_MMA_SIDE_UNROLL;
#ifndef DGB_MMA_PACK_UNROLL
#define DGB_MMA_PACK_UNROLL 2  // packed surface tile loop (p = 3, 4)
#endif
constexpr int kMmaPackUnroll = DGB_MMA_PACK_UNROLL;
#ifndef DGB_MMA_C_SMEM_MINP
// degrees >= this read the stage input for the RK epilogue from the own fragment buffer
// (measured per stage: p=5 1.739 vs 1.846 ms, p=4 1.089 vs 1.108, p=3 0.870 vs 0.866; after
// the kernel-instance split p=3 0.730 vs 0.771)
#define DGB_MMA_C_SMEM_MINP 3
#endif
#ifndef DGB_MMA_U_AHEAD
#define DGB_MMA_U_AHEAD 1
#endif
#ifndef DGB_MMA_TMA
#define DGB_MMA_TMA(P) 1  // own coefficients of a tile by one TMA box (0: per-lane cp.async)
#endif
#ifndef DGB_MMA_SPLIT_J
#define DGB_MMA_SPLIT_J 1
#endif
#ifndef DGB_MMA_SPLIT_JV
// p=5 volume projection of modes 16..20 by DFMAs (288 -> 240 DMMAs per tile): 1.632 vs 1.553 ms,
// the 20 partial sums push the 168-register kernel into more spills
#define DGB_MMA_SPLIT_JV 0
#endif
#ifndef DGB_MMA_EDGE_EARLY
// issue the edge-normal gathers before the volume integral instead of at the surface: p=3, 4
// unchanged (0.667 / 0.980 ms), p=5 1.598 vs 1.550 (nine more live doubles across the volume)
#define DGB_MMA_EDGE_EARLY(P) 0
#endif
#ifndef DGB_MMA_SPLIT_K
// the last mode k-step of interpolations and traces by DFMAs when <= 2 modes are live: p=3
// 0.687 vs 0.666 ms, p=5 1.549 vs 1.533 (fewer DMMAs, 120 -> 92 per tile at p=3, but the
// lane-indexed table loads and the dependent DFMA chains sit on the flux's critical path)
#define DGB_MMA_SPLIT_K 0
#endif
#ifndef DGB_MMA_PACK_MAXK
#define DGB_MMA_PACK_MAXK 5  // largest edge-point count K that uses the packed surface
#endif

template <int P>
struct MmaDim {
  static constexpr int NP = Dim<P>::NP, NQ = Dim<P>::NQ, K = Dim<P>::K;
  static constexpr int KS = (NP + 3) / 4;  // k-steps over modes
  static constexpr int NT = (NQ + 7) / 8;  // 8-point tiles of interior points
  static constexpr int JT = (NP + 7) / 8;  // 8-mode tiles of the projections' output
  // shared-memory table layout (doubles), fragment order, 32 values per fragment
  static constexpr int kPhi = 0;                            // [KS][NT][32]
  static constexpr int kDr = kPhi + KS * NT * 32;           // [NT][2][JT][32]
  static constexpr int kDs = kDr + NT * 2 * JT * 32;        // [NT][2][JT][32]
  static constexpr int kPhe = kDs + NT * 2 * JT * 32;       // [3][KS][32] own trace of side q
  static constexpr int kPheR = kPhe + 3 * KS * 32;          // [3][KS][32] reversed trace of side s
  static constexpr int kPheP = kPheR + 3 * KS * 32;         // [3][2][JT][32] surface projection
  static constexpr int kPhm = kPheP + 3 * 2 * JT * 32;      // [3][JT*8] midpoint rows (zero padded)
  static constexpr int kWe = kPhm + 3 * JT * 8;             // [8] edge weights (zero padded)
  // a single trailing interior point (NQ % 8 == 1, p = 5) is done with DFMAs instead of a
  // whole padded DMMA tile: its basis row (mode 4ks+t at [ks][t]) and weighted gradient rows
  static constexpr bool kTail1 = (NQ % 8) == 1;
  static constexpr int NTD = kTail1 ? NQ / 8 : NT;  // point tiles done with DMMA
  static constexpr int kTail = kWe + 8;                     // [KS*4] phi, [JT*8] w dr, [JT*8] w ds
  // Packed surface (K <= 5, i.e. p = 3, 4): the 3K edge points of the three sides share
  // NSP = ceil(3K/8) column tiles instead of one padded tile per side, so fewer flux
  // evaluations, own-trace and projection DMMAs.  Column c of tile s is point 8s + c =
  // (side (8s+c) / K, point (8s+c) % K).
  static constexpr int NSP = (3 * K + 7) / 8;
  static constexpr bool kPacked = NSP < 3 && K <= DGB_MMA_PACK_MAXK;
  static constexpr int kPkOwn = kTail + (kTail1 ? KS * 4 + 2 * JT * 8 : 0);  // [NSP][KS][32]
  static constexpr int kPkNb = kPkOwn + (kPacked ? NSP * KS * 32 : 0);      // [NSP][3 sides][3 classes][KS][32]
  static constexpr int kPkProj = kPkNb + (kPacked ? NSP * 9 * KS * 32 : 0);  // [NSP][2][JT][32]
  static constexpr int kSize = kPkProj + (kPacked ? NSP * 2 * JT * 32 : 0);
  // the per-warp buffers start 128-byte aligned (TMA destination)
  static constexpr int kBufOff = (kSize + 15) / 16 * 16;
  // per-warp staging after the tables: own [4 KS][32] + neighbour [4 KS][32] (two
  // neighbour buffers when the surface is packed: a tile spans two sides)
  // one fragment buffer: 4 KS k-steps of 32 lanes, at least a tile's staged trace blocks in the
  // trace-buffer degrees (8 elements x (12K + 2) doubles, packed; a side is smaller), rounded to 16
  static constexpr int kFR = (DGB_TRACE_P(P) && kPacked && 8 * (12 * K + 2) > 4 * KS * 32)
                                 ? (8 * (12 * K + 2) + 15) / 16 * 16
                                 : 4 * KS * 32;
  static constexpr int kWarpBuf = (kPacked ? 3 : 2) * kFR;
};

// volatile: a non-volatile asm may be duplicated into both arms of a per-lane
// select (e.g. `a = cond ? load : 0`), giving two predicated DMMAs that the
// warp executes divergently — which deadlocks the .aligned warp-wide MMA.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}


// A-fragment copy of one element column (4 variables x Np modes) into a lane-private
// slot array [4 * KS][32] of shared memory.  The lane's source walks the column by uniform
// strides (4 ld within a variable, (NP - 4 (KS - 1)) ld to the next) and the zero-fill size is
// formed once (the last k-step masks modes >= NP): three instructions per copy instead of the
// ten a per-copy 64-bit index product and predicate cost (measured in the SASS).
#ifndef DGB_MMA_FETCH_WALK
// measured per stage (interleaved A/B): p=5 1.544 vs 1.580 ms, p=4 equal, p=3 0.717 vs 0.704 (kept off)
#define DGB_MMA_FETCH_WALK(NP) ((NP) > 10)
#endif
template <int NP, int KS>
__device__ __forceinline__ void fetch_frag(double* __restrict__ slot, const double* __restrict__ base, long long ld,
                                           int col, bool ok, int lane, int t) {
  if constexpr (!DGB_MMA_FETCH_WALK(NP)) {  // per-copy index and predicate
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int j = 4 * ks + t;
        const bool p = ok && j < NP;
        cp_async8(slot + (m * KS + ks) * 32 + lane, p ? base + (static_cast<long long>(m) * NP + j) * ld + col : base, p);
      }
    return;
  }
  const double* src = base + (ok ? static_cast<long long>(t) * ld + col : 0);
  const int sz = ok ? 8 : 0;
  const int sz_last = (ok && 4 * (KS - 1) + t < NP) ? 8 : 0;
  const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(slot + lane));
#pragma unroll
  for (int m = 0; m < 4; ++m) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int s = (ks == KS - 1 && 4 * ks + 3 >= NP) ? sz_last : sz;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + (m * KS + ks) * 32 * 8), "l"(src),
                   "r"(s)
                   : "memory");
      src += (ks + 1 < KS) ? 4 * ld : (NP - 4 * (KS - 1)) * ld;
    }
  }
}

// Half-live last tiles (p = 3): compact the points before the flux (one flux evaluation per
// lane, DGB_HALF_* = 1) or after it (two per lane, the fluxes shuffled into the compacted
// k-step by half_operands).  Measured at p = 3 (1M box, interleaved): volume compacted before
// 0.681 vs 0.690 ms; the surface compacted before 0.709 ms (eight shuffled trace values and
// the boundary / neighbour selects per lane cost more than the flux evaluation saved).
#ifndef DGB_HALF_VOL
#define DGB_HALF_VOL 1
#endif
#ifndef DGB_HALF_SURF
#define DGB_HALF_SURF 0
#endif
// Projection k-step of a half-live 8-point tile from fluxes evaluated at both slots: slot
// t < 2 takes this lane's point i=0, slot t >= 2 the point i=1 of lane t-2 (one shuffle per
// value).  The B fragment of that slot is the existing table entry of k-step i=1 at lane-2, so
// the caller offsets its table index by the returned flag * (one k-step of fragments - 2).
__device__ __forceinline__ int half_operands(const double (&v)[4][2], double (&a)[4], int lane, int t) {
  const bool hi = t >= 2;
  const int src = (lane + 30) & 31;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const double o = __shfl_sync(0xffffffffu, v[m][1], src);
    a[m] = hi ? o : v[m][0];
  }
  return hi ? 1 : 0;
}

// 16-byte cp.async (L2 only), zero-filled when !pred
__device__ __forceinline__ void cp_async16(double* dst, const double* src, bool pred) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(src), "r"(pred ? 16 : 0) : "memory");
}

// ---- TMA load of a tile's own coefficients (one cp.async.bulk.tensor per tile, lane 0)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
// Box {8 elements, NP modes, 4 variables} of the [4][NP][ld] tensor at element column `col`, into
// dst[(m NP + j) 8 + g]; completes on `bar`, its transaction count armed with the box bytes.  (A
// box of 4 KS mode rows, the padding rows zero-filled outside the tensor, measured slower: p=3
// 0.725 vs 0.718 ms, p=4 0.996 vs 0.979.)  The fence orders the warp's earlier generic-proxy
// reads of dst before the async-proxy write.
template <int NP>
__device__ __forceinline__ void tma_own_tile(double* dst, const void* tm, int col, unsigned long long* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(NP * 4 * 8 * 8)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(col), "r"(0), "r"(0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  unsigned done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

template <int P, int MODE, int FLUX, int VAR>
__device__ __forceinline__ void element_body_mma(const Tab<P>& T, const Geo& geo, const StageArgs& a,
                                                 double* __restrict__ smem) {
  using D = MmaDim<P>;
  constexpr int NP = D::NP, NQ = D::NQ, K = D::K, KS = D::KS, NT = D::NT, JT = D::JT;
  constexpr int FR = D::kFR;  // doubles of one fragment buffer (spacing of the per-warp buffers)
  const long long ld = geo.ld;
  const double gamma = geo.gamma, g1 = gamma - 1.0;
  Scalars* sc = a.sc;
  // instance variant (kernels_tu.cuh): paths the launch knows are unused compile away
  constexpr bool RK4 = VAR & kVarRk4, LAM = VAR & kVarLambda, BND = VAR & kVarBoundary;
  const int kmode = RK4 ? a.kmode : 0;
  const bool want_lambda = LAM && a.want_lambda;

  __shared__ int s_stop;
  if (threadIdx.x == 0) s_stop = (sc->err_key != kNoError || sc->halt) ? 1 : 0;
  // basis tables -> shared memory (fragment order, prepared on the host)
  for (int i = threadIdx.x; i < D::kSize; i += blockDim.x) smem[i] = __ldg(geo.mma_tab + i);
  __syncthreads();
  if (s_stop) return;

  double t0 = a.t_host, dt = 0.0;
  if constexpr (MODE == kModeStage) {
    if (!stage_prologue(a, sc, t0, dt)) return;
  }
  const double tstage = (MODE == kModeStage) ? fma(a.tcoef, dt, t0) : t0;

  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wib = threadIdx.x >> 5;
  const int warp = blockIdx.x * (blockDim.x >> 5) + wib;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int ntiles = (a.e1 - a.e0 + 7) >> 3;
  // per-warp staging: own coefficients of the tile, neighbour coefficients of one side
  double* __restrict__ w_own = smem + D::kBufOff + wib * D::kWarpBuf;
  double* __restrict__ w_nbr = w_own + FR;
  // packed surface (p = 3, 4): a second neighbour buffer, side q lives in buffer q & 1
  constexpr bool kPk = D::kPacked && (MODE == kModeRhs || MODE == kModeStage);
  // last point tile / last packed surface tile with only slots t < 2 live (p = 3: Q = 12,
  // 3K = 12): one compacted projection k-step (DGB_HALF_VOL / DGB_HALF_SURF, half_operands)
  constexpr bool kHalfQ = NQ % 8 == 4 && !D::kTail1;
  constexpr bool kHalfS = kPk && (3 * K) % 8 == 4;
  // trace-buffer instance: the packed surface reads the own and neighbour traces of the stage
  // input from a.tr_in (staged into the two neighbour buffers by cp.async one tile ahead, own
  // traces in w_nbr, the neighbours' reversed traces in w_nbr2, both [4][3K][8 elements])
  // instead of interpolating them; the epilogue writes the traces of the new stage (a.tr_out)
  constexpr bool kTrIn = kPk && MODE == kModeStage && DGB_TRACE_P(P) && (VAR & kVarTrace) != 0;
  // the same for the per-side surface (p = 5): side q's own rows and its neighbour's reversed rows
  // staged into w_nbr one side ahead, [own | neighbour][4][K][8 elements]
  constexpr bool kTrInS = !kPk && MODE == kModeStage && DGB_TRACE_P(P) && (VAR & kVarTrace) != 0;
  constexpr int K3 = 3 * K;
  // trace layout (element-major, so a neighbour's side is one contiguous 4K-double block):
  // tr[e][side][var][point], kTS doubles per element; in shared memory kTSP (kTS padded so the 8
  // elements of a tile start in different banks), kSSP per element for one staged side
  constexpr int kTS = 4 * K3;
  constexpr int kTSP = kTS + 2;
  constexpr int kSSP = 8 * K + 2;
  static_assert(!DGB_TRACE_P(P) || (kPk ? 8 * kTSP : 8 * kSSP) <= FR, "staged trace blocks exceed a fragment buffer");
  // the last output tile of the projections when it holds at most two live modes (p = 3: modes
  // 8, 9 in 8 columns): the volume and packed-surface projections accumulate those modes with
  // DFMAs into X (each lane its own points' share), reduced over the element's four lanes
  // before the outputs, instead of DMMAs whose output tile is three quarters padding
  constexpr int kNJR = NP - 8 * (JT - 1);
  constexpr bool kSplitJ = DGB_MMA_SPLIT_J != 0 && JT > 1 && kNJR <= 2;
  constexpr int JTD = kSplitJ ? JT - 1 : JT;  // output tiles done with DMMA there
  // the volume projection alone split the same way when the last output tile holds up to five
  // live modes (p = 5: modes 16..20), X folded into R right after the volume integral
  constexpr bool kSplitJV = !kSplitJ && DGB_MMA_SPLIT_JV != 0 && JT > 1 && kNJR <= 5;
  constexpr bool kSplitJVol = kSplitJ || kSplitJV;
  constexpr int JTDV = kSplitJVol ? JT - 1 : JT;
  // the last mode k-step of the interpolations and traces when it holds at most two live modes
  // (p = 3: modes 8, 9 of 8..11; p = 5: mode 20): DFMAs on the lane's own output columns instead
  // of a half- or quarter-live DMMA.  Own and neighbour traces take the same path in the same
  // order, so the two sides of an edge still see bit-identical traces.
  constexpr bool kEdgeEarly = DGB_MMA_EDGE_EARLY(P) != 0;
  constexpr int kNKR = NP - 4 * (KS - 1);
  constexpr bool kSplitK = DGB_MMA_SPLIT_K != 0 && kNKR <= 2;
  constexpr int KSD = kSplitK ? KS - 1 : KS;  // k-steps done with DMMA
  // stage mode: the epilogue reads the stage input from the own fragment buffer (shared
  // memory) instead of global memory; the next tile's own prefetch waits until then
  constexpr bool kCSmem = P >= DGB_MMA_C_SMEM_MINP && MODE == kModeStage;
  constexpr bool kUAhead = DGB_MMA_U_AHEAD != 0;
  double* __restrict__ w_nbr2 = w_own + 2 * FR;
  // Own coefficients of a tile.  kTma builds: one cp.async.bulk.tensor box per tile (a.tm_in, the
  // launcher guarantees an even first column: 16-byte aligned boxes), issued by lane 0 into
  // w_own[(m NP + j) 8 + g] and completing on the warp's mbarrier.  Otherwise per-lane cp.async
  // into the fragment order w_own[(m KS + ks) 32 + lane].
  constexpr bool kTma = DGB_MMA_TMA(P) != 0;
  __shared__ unsigned long long s_own_bar[32];
  unsigned long long* own_bar = &s_own_bar[wib];
  unsigned own_phase = 0;
  if (kTma) {
    if (lane == 0) {
      mbar_init(own_bar);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  auto own_fetch = [&](int tl, int col, bool ok) {  // tile tl (element column col of lane group g)
    if constexpr (kTma) {
      if (lane == 0 && tl < ntiles) tma_own_tile<NP>(w_own, a.tm_in, a.e0 + tl * 8, own_bar);
    } else {
      fetch_frag<NP, KS>(w_own, a.in, ld, col, ok, lane, t);
    }
  };
  // A fragment (element g, mode 4 ks + t) of variable m from the own buffer
  auto own_a = [&](int m, int ks) -> double {
    if constexpr (kTma) {
      const int j = 4 * ks + t;
      return j < NP ? w_own[(m * NP + j) * 8 + g] : 0.0;
    } else {
      return w_own[(m * KS + ks) * 32 + lane];
    }
  };

  // coefficient j >= 4 (KS - 1) of element g from the own buffer / a neighbour fragment buffer
  auto own_c = [&](int m, int j) -> double {
    if constexpr (kTma) {
      return w_own[(m * NP + j) * 8 + g];
    } else {
      return w_own[(m * KS + KS - 1) * 32 + 4 * g + (j - 4 * (KS - 1))];
    }
  };
  // kSplitK: acc[m][ii] += sum_jj c(m, jj) B[jj][2t + ii] over the live modes of the last
  // k-step, B the k-step's fragment (B[t'][g'] at 4 g' + t')
  auto ktail = [&](double(&acc)[4][2], const double* __restrict__ frag, auto cval) {
    double ph[2][2];
#pragma unroll
    for (int ii = 0; ii < 2; ++ii)
#pragma unroll
      for (int jj = 0; jj < kNKR; ++jj) ph[ii][jj] = frag[4 * (2 * t + ii) + jj];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int jj = 0; jj < kNKR; ++jj) {
        const double c = cval(m, jj);
#pragma unroll
        for (int ii = 0; ii < 2; ++ii) acc[m][ii] = fma(c, ph[ii][jj], acc[m][ii]);
      }
  };

  double lam_min = __longlong_as_double(0x7ff0000000000000ll);
  double res_max = 0.0;

  auto elem_of = [&](int tile, bool& ok) {
    int e = a.e0 + tile * 8 + g;
    ok = tile < ntiles && e < a.e1;
    return ok ? e : a.e1 - 1;
  };
  auto nbr_of = [&](int e, int q) { return __ldg(geo.nbr + q * ld + e); };
  // kTrIn: traces of element column col (lane group g) and of its neighbours nb[] (side labels in
  // inf_) into the neighbour buffers; lane t copies rows t, t + 4, ... of the 4 * 3K rows
  auto fetch_side_traces = [&](int col, bool ok, int q, int nbc, int inf_) {
    if constexpr (kTrInS) {
      // element g's side q block and its neighbour's side block (4K doubles each) into
      // w_nbr[g kSSP + (own | 4K + neighbour)], 16 bytes per copy, lane t every fourth chunk
      const int sl = (inf_ >> (2 * q)) & 3;
      const bool okn = ok && nbc >= 0 && sl != 0;
      const double* so = a.tr_in + static_cast<long long>(col) * kTS + q * 4 * K;
      const double* sn = a.tr_in + static_cast<long long>(okn ? nbc : 0) * kTS + (okn ? sl - 1 : 0) * 4 * K;
#pragma unroll
      for (int i = 0; i < K; ++i) {  // 4K chunks of 16 bytes: K per lane
        const int c = 4 * i + t;      // chunk < 4K: own (c < 2K) or neighbour
        const bool own = c < 2 * K;
        const int cc = own ? c : c - 2 * K;
        cp_async16(w_nbr + g * kSSP + (own ? 0 : 4 * K) + 2 * cc, (own ? so : sn) + 2 * cc, own ? ok : okn);
      }
    }
  };
  auto fetch_traces = [&](int col, bool ok, const int (&nb)[3], int inf_) {
    if constexpr (kTrIn) {
      // element g's whole block into w_nbr[g kTSP], its neighbours' side blocks (4K doubles each,
      // side q's neighbour at q 4K) into w_nbr2[g kTSP]; 16 bytes per copy
      const double* so = a.tr_in + static_cast<long long>(col) * kTS;
#pragma unroll
      for (int i = 0; i < (kTS / 2 + 3) / 4; ++i) {
        const int c = 4 * i + t;
        if (c < kTS / 2) cp_async16(w_nbr + g * kTSP + 2 * c, so + 2 * c, ok);
      }
#pragma unroll
      for (int i = 0; i < (kTS / 2 + 3) / 4; ++i) {
        const int c = 4 * i + t;
        if (c < kTS / 2) {
          const int q = c / (2 * K), cc = c - q * 2 * K;
          const int nbc = q == 0 ? nb[0] : (q == 1 ? nb[1] : nb[2]);
          const int sl = (inf_ >> (2 * q)) & 3;
          const bool okn = ok && nbc >= 0 && sl != 0;
          const double* sn = a.tr_in + static_cast<long long>(okn ? nbc : 0) * kTS + (okn ? sl - 1 : 0) * 4 * K;
          cp_async16(w_nbr2 + g * kTSP + q * 4 * K + 2 * cc, sn + 2 * cc, okn);
        }
      }
    }
  };

  // pipeline prologue: own coefficients and side-0 neighbours of the first tile
  int nbq[3] = {-4, -4, -4};  // neighbour columns of the current tile's element
  {
    bool ok;
    const int e = elem_of(warp, ok);
    own_fetch(warp, e, ok);
    cp_async_commit();
    if constexpr (MODE != kModeVolume) {
#pragma unroll
      for (int q = 0; q < 3; ++q) nbq[q] = nbr_of(e, q);
      if constexpr (kTrIn) {
        fetch_traces(e, ok, nbq, __ldg(geo.info + e));
      } else if constexpr (kTrInS) {
        fetch_side_traces(e, ok, 0, nbq[0], __ldg(geo.info + e));
      } else {
        fetch_frag<NP, KS>(w_nbr, a.in, ld, nbq[0], ok && nbq[0] >= 0, lane, t);
        if constexpr (kPk) fetch_frag<NP, KS>(w_nbr2, a.in, ld, nbq[1], ok && nbq[1] >= 0, lane, t);
      }
    }
    cp_async_commit();
  }

  for (int tile = warp; tile < ntiles; tile += nwarps) {
    bool valid;
    const int e = elem_of(tile, valid);
    bool nvalid;
    const int e_next = elem_of(tile + nwarps, nvalid);
    // side data of this tile and the next tile's neighbour columns, issued early so
    // they land during the volume integral
    int nbn[3] = {-4, -4, -4}, edq[3] = {0, 0, 0}, inf = 0, inf_next = 0;
    if constexpr (MODE != kModeVolume) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        nbn[q] = nbr_of(e_next, q);
        edq[q] = __ldg(geo.eid + q * ld + e);
      }
      inf = __ldg(geo.info + e);
      if constexpr (kTrIn || kTrInS) inf_next = __ldg(geo.info + e_next);
    }
    cp_async_wait<0>();  // own coefficients and side-0 neighbours of this tile
    if constexpr (kTma) {
      mbar_wait(own_bar, own_phase);
      own_phase ^= 1u;
    }
    __syncwarp();
    // edge normals and lengths of the tile's three sides (gathered by edge id)
    double enx[3], eny[3], eh[3];
    auto load_edges = [&]() {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        enx[q] = __ldg(geo.enx + edq[q]);
        eny[q] = __ldg(geo.eny + edq[q]);
        eh[q] = __ldg(geo.eh + edq[q]);
      }
    };
    if constexpr (kEdgeEarly && MODE != kModeVolume) load_edges();  // in flight during the volume integral

    double R[4][JT][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int jt = 0; jt < JT; ++jt) R[m][jt][0] = R[m][jt][1] = 0.0;
    double X[4][kNJR] = {};  // kSplitJ / kSplitJV: this lane's share of modes 8 (JT - 1) + gg
    // the four lanes' shares of X summed in the same order on every lane; lane t holds output
    // columns 8 (JT - 1) + 2t + ii (the columns >= NP are padding)
    auto fold_x = [&]() {
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int gg = 0; gg < kNJR; ++gg) {
          double x = X[m][gg];
          x += __shfl_xor_sync(0xffffffffu, x, 1);
          x += __shfl_xor_sync(0xffffffffu, x, 2);
          R[m][JT - 1][gg & 1] += (gg >> 1) == t ? x : 0.0;
        }
    };

    // ------------------------------------------------------------ volume
    if constexpr (MODE != kModeSurface) {
      const double ta = __ldg(geo.tau + e), tb = __ldg(geo.tau + ld + e);
      const double tc = __ldg(geo.tau + 2 * ld + e), td = __ldg(geo.tau + 3 * ld + e);
      double U[2][4][2];
      auto interp = [&](double(&u)[4][2], int nt) {
#pragma unroll
        for (int m = 0; m < 4; ++m) u[m][0] = u[m][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KSD; ++ks) {
          const double b = smem[D::kPhi + (ks * NT + nt) * 32 + lane];
#pragma unroll
          for (int m = 0; m < 4; ++m) dmma(u[m], own_a(m, ks), b);
        }
        if constexpr (kSplitK)
          ktail(u, smem + D::kPhi + ((KS - 1) * NT + nt) * 32, [&](int m, int jj) { return own_c(m, 4 * (KS - 1) + jj); });
      };
      constexpr int NTD = D::NTD;
      if (DGB_MMA_VOL_PIPE(P)) interp(U[0], 0);
#pragma unroll
      for (int nt = 0; nt < NTD; ++nt) {
        // software pipeline: the next tile of points is interpolated while this
        // tile's fluxes are evaluated
        if (DGB_MMA_VOL_PIPE(P)) {
          if (nt + 1 < NTD) interp(U[(nt + 1) & 1], nt + 1);
        } else {
          interp(U[nt & 1], nt);
        }
        // contravariant flux at interior point k from its interpolated state v
        auto vol_point = [&](double(&v)[4], int k, double(&r_)[4], double(&s_)[4]) {
          Prim w = primitives(v, g1);
          const bool bad = !admissible(v, w);
          if (bad && valid && k < NQ) record_error(sc, err_key(a.seq, kPassVolume, __ldg(geo.ref_id + e), k));
          if (bad) {  // placeholder (solver.cpp:129-132)
            v[0] = 1.0; v[1] = 0.0; v[2] = 0.0; v[3] = 2.5;
            w.inv = 1.0; w.vx = 0.0; w.vy = 0.0; w.p = 1.0;
          }
          contravariant_flux(v, w, ta, tb, tc, td, r_, s_);
        };
        if (DGB_HALF_VOL && kHalfQ && nt == NTD - 1) {
          // half-live last tile (p = 3: points 8..11, live in slots t < 2): slots t >= 2 take the
          // second point of lane t - 2 before the flux, so every lane evaluates one live point
          // and its fluxes are already the operands of one compacted projection k-step
          const bool hi = t >= 2;
          const int src = (lane + 30) & 31;
          double v[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const double o = __shfl_sync(0xffffffffu, U[nt & 1][m][1], src);
            v[m] = hi ? o : U[nt & 1][m][0];
          }
          double ar[4], as[4];
          vol_point(v, 8 * nt + (hi ? 2 * t - 3 : 2 * t), ar, as);
          __syncwarp();
          const int boff = hi ? JT * 32 - 2 : 0;  // the B fragment of k-step i=1 at lane - 2
#pragma unroll
          for (int jt = 0; jt < JTDV; ++jt) {
            const double br = smem[D::kDr + (nt * 2 * JT + jt) * 32 + lane + boff];
            const double bs = smem[D::kDs + (nt * 2 * JT + jt) * 32 + lane + boff];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], ar[m], br);
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], as[m], bs);
          }
          if constexpr (kSplitJVol) {
#pragma unroll
            for (int gg = 0; gg < kNJR; ++gg) {
              const double dr = smem[D::kDr + (nt * 2 * JT + JT - 1) * 32 + 4 * gg + t + boff];
              const double ds = smem[D::kDs + (nt * 2 * JT + JT - 1) * 32 + 4 * gg + t + boff];
#pragma unroll
              for (int m = 0; m < 4; ++m) X[m][gg] = fma(dr, ar[m], fma(ds, as[m], X[m][gg]));
            }
          }
          continue;
        }
        double fr[4][2], fs[4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int k = 8 * nt + 2 * t + i;
          double v[4] = {U[nt & 1][0][i], U[nt & 1][1][i], U[nt & 1][2][i], U[nt & 1][3][i]};
          double r_[4], s_[4];
          vol_point(v, k, r_, s_);
          const bool live = k < NQ;  // padded points contribute nothing
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            fr[m][i] = live ? r_[m] : 0.0;  // contravariant flux along r
            fs[m][i] = live ? s_[m] : 0.0;  // along s
          }
        }
        __syncwarp();
        if (!DGB_HALF_VOL && kHalfQ && nt == NTD - 1) {
          double ar[4], as[4];
          const int boff = half_operands(fr, ar, lane, t) * (JT * 32 - 2);
          half_operands(fs, as, lane, t);
#pragma unroll
          for (int jt = 0; jt < JTDV; ++jt) {
            const double br = smem[D::kDr + (nt * 2 * JT + jt) * 32 + lane + boff];
            const double bs = smem[D::kDs + (nt * 2 * JT + jt) * 32 + lane + boff];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], ar[m], br);
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], as[m], bs);
          }
          if constexpr (kSplitJVol) {
#pragma unroll
            for (int gg = 0; gg < kNJR; ++gg) {
              const double dr = smem[D::kDr + (nt * 2 * JT + JT - 1) * 32 + 4 * gg + t + boff];
              const double ds = smem[D::kDs + (nt * 2 * JT + JT - 1) * 32 + 4 * gg + t + boff];
#pragma unroll
              for (int m = 0; m < 4; ++m) X[m][gg] = fma(dr, ar[m], fma(ds, as[m], X[m][gg]));
            }
          }
          continue;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jt = 0; jt < JTDV; ++jt) {
            const double br = smem[D::kDr + ((nt * 2 + i) * JT + jt) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], fr[m][i], br);
          }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jt = 0; jt < JTDV; ++jt) {
            const double bs = smem[D::kDs + ((nt * 2 + i) * JT + jt) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], fs[m][i], bs);
          }
        if constexpr (kSplitJVol) {
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int gg = 0; gg < kNJR; ++gg) {
              const double dr = smem[D::kDr + ((nt * 2 + i) * JT + JT - 1) * 32 + 4 * gg + t];
              const double ds = smem[D::kDs + ((nt * 2 + i) * JT + JT - 1) * 32 + 4 * gg + t];
#pragma unroll
              for (int m = 0; m < 4; ++m) X[m][gg] = fma(dr, fr[m][i], fma(ds, fs[m][i], X[m][gg]));
            }
        }
      }
      if constexpr (D::kTail1) {
        // the last interior point: the 4 lanes of an element reduce their modes' share
        // of the interpolation, all 4 evaluate the flux, each projects onto its own modes
        constexpr int k = NQ - 1;
        double v[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          double sum = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) sum = fma(own_a(m, ks), smem[D::kTail + ks * 4 + t], sum);
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
        __syncwarp();
      }
      if constexpr (kSplitJV) fold_x();
    }

    // ------------------------------------------------------------ surface
    if constexpr (kPk) {
      if constexpr (!kEdgeEarly) load_edges();
      auto sel3 = [](int q, auto x0, auto x1, auto x2) { return q == 0 ? x0 : (q == 1 ? x1 : x2); };
#pragma unroll kMmaPackUnroll
      for (int sp = 0; sp < D::NSP; ++sp) {
        if (!kTrIn && sp > 0) cp_async_wait<0>();  // side 2's neighbour column (prefetched during tile 0)
        // own trace of the packed tile
        double Tw[4][2], Tn[4][2];
#pragma unroll
        for (int m = 0; m < 4; ++m) Tw[m][0] = Tw[m][1] = Tn[m][0] = Tn[m][1] = 0.0;
        if constexpr (kTrIn) {  // from the staged trace rows (waited for at the tile start)
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              const int pt = 8 * sp + 2 * t + ii;
              const int q = pt < K3 ? pt / K : 0, ko = pt - q * K;
              Tw[m][ii] = pt < K3 ? w_nbr[g * kTSP + (q * 4 + m) * K + ko] : 0.0;
              Tn[m][ii] = pt < K3 ? w_nbr2[g * kTSP + (q * 4 + m) * K + (K - 1 - ko)] : 0.0;
            }
        } else {
#pragma unroll
        for (int ks = 0; ks < KSD; ++ks) {
          const double b = smem[D::kPkOwn + (sp * KS + ks) * 32 + lane];
#pragma unroll
          for (int m = 0; m < 4; ++m) dmma(Tw[m], own_a(m, ks), b);
        }
        if constexpr (kSplitK)
          ktail(Tw, smem + D::kPkOwn + (sp * KS + KS - 1) * 32, [&](int m, int jj) { return own_c(m, 4 * (KS - 1) + jj); });
        // neighbour traces of the sides present in this tile (their columns only)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          if (q * K >= 8 * (sp + 1) || (q + 1) * K <= 8 * sp) continue;  // side q not in tile sp
          const double* __restrict__ nbuf = (q & 1) ? w_nbr2 : w_nbr;
          const int snb_q = nbq[q] < 0 ? 0 : ((inf >> (2 * q)) & 3);
          unsigned todo = __reduce_or_sync(0xffffffffu, snb_q ? (1u << snb_q) : 0u);
          while (todo) {
            const int cls = __ffs(todo) - 1;
            todo &= todo - 1;
            const bool mine = snb_q == cls;
#pragma unroll
            for (int ks = 0; ks < KSD; ++ks) {
              const double b = smem[D::kPkNb + (((sp * 3 + q) * 3 + (cls - 1)) * KS + ks) * 32 + lane];
#pragma unroll
              for (int m = 0; m < 4; ++m) {
                const double an = nbuf[(m * KS + ks) * 32 + lane];
                dmma(Tn[m], mine ? an : 0.0, b);
              }
            }
            if constexpr (kSplitK)
              ktail(Tn, smem + D::kPkNb + (((sp * 3 + q) * 3 + (cls - 1)) * KS + KS - 1) * 32, [&](int m, int jj) {
                return mine ? nbuf[(m * KS + KS - 1) * 32 + 4 * g + jj] : 0.0;
              });
          }
        }
        }  // !kTrIn
        __syncwarp();
        // buffers consumed: tile 0 frees side 0's buffer (side 2 goes there); the last
        // tile frees everything (the next tile's sides 0, 1 and own coefficients)
        if constexpr (kTrIn) {
          if (sp + 1 == D::NSP) {
            fetch_traces(e_next, nvalid, nbn, inf_next);
            if (!kCSmem) own_fetch(tile + nwarps, e_next, nvalid);
          }
        } else if (sp + 1 < D::NSP) {
          fetch_frag<NP, KS>(w_nbr, a.in, ld, nbq[2], valid && nbq[2] >= 0, lane, t);
        } else {
          fetch_frag<NP, KS>(w_nbr, a.in, ld, nbn[0], nvalid && nbn[0] >= 0, lane, t);
          fetch_frag<NP, KS>(w_nbr2, a.in, ld, nbn[1], nvalid && nbn[1] >= 0, lane, t);
          if (!kCSmem) own_fetch(tile + nwarps, e_next, nvalid);
        }
        cp_async_commit();
        // numerical flux at packed point pt (side pt / K), canonical orientation
        auto surf_point = [&](double(&UO)[4], double(&UN)[4], int pt, double(&f)[4]) {
          const bool live = pt < 3 * K;
          const int q = live ? pt / K : 0, ko = live ? pt % K : 0;
          const int nb = sel3(q, nbq[0], nbq[1], nbq[2]);
          const int ed = sel3(q, edq[0], edq[1], edq[2]);
          const double nx = sel3(q, enx[0], enx[1], enx[2]), ny = sel3(q, eny[0], eny[1], eny[2]);
          const double h = sel3(q, eh[0], eh[1], eh[2]);
          const bool left = (inf >> (6 + q)) & 1;
          const bool bnd = nb < 0;
          const int kc = left ? ko : K - 1 - ko;  // canonical (left-element) point index
          if (BND && bnd && live) ghost_state<K>(UO, nb, ed, kc, nx, ny, tstage, geo, UN);  // boundary: left
          const Prim wo = primitives(UO, g1), wn = primitives(UN, g1);
          const double wh = live ? h * smem[D::kWe + kc] : 0.0;
          if (admissible(UO, wo) && admissible(UN, wn)) {
            num_flux_own<FLUX>(UO, wo, UN, wn, nx, ny, gamma, wh, left, f);
          } else {
            if (valid && live) record_error(sc, err_key(a.seq, kPassSurface, ed, kc));
#pragma unroll
            for (int m = 0; m < 4; ++m) f[m] = 0.0;
          }
        };
        if (DGB_HALF_SURF && kHalfS && sp == D::NSP - 1) {
          // half-live last packed tile (p = 3: points 8..11, live in slots t < 2): compacted
          // before the flux as in the volume's last tile, one projection k-step
          const bool hi = t >= 2;
          const int src = (lane + 30) & 31;
          double UO[4], UN[4], an[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const double oo = __shfl_sync(0xffffffffu, Tw[m][1], src);
            const double on = __shfl_sync(0xffffffffu, Tn[m][1], src);
            UO[m] = hi ? oo : Tw[m][0];
            UN[m] = hi ? on : Tn[m][0];
          }
          surf_point(UO, UN, 8 * sp + (hi ? 2 * t - 3 : 2 * t), an);
          __syncwarp();
          const int boff = hi ? JT * 32 - 2 : 0;
#pragma unroll
          for (int jt = 0; jt < JTD; ++jt) {
            const double b = smem[D::kPkProj + (sp * 2 * JT + jt) * 32 + lane + boff];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], an[m], b);
          }
          if constexpr (kSplitJ) {
#pragma unroll
            for (int gg = 0; gg < kNJR; ++gg) {
              const double b = smem[D::kPkProj + (sp * 2 * JT + JT - 1) * 32 + 4 * gg + t + boff];
#pragma unroll
              for (int m = 0; m < 4; ++m) X[m][gg] = fma(b, an[m], X[m][gg]);
            }
          }
          continue;
        }
        double fn[4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          double UO[4], UN[4], f[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            UO[m] = Tw[m][i];
            UN[m] = Tn[m][i];
          }
          surf_point(UO, UN, 8 * sp + 2 * t + i, f);
#pragma unroll
          for (int m = 0; m < 4; ++m) fn[m][i] = f[m];
        }
        __syncwarp();
        if (!DGB_HALF_SURF && kHalfS && sp == D::NSP - 1) {
          double an[4];
          const int boff = half_operands(fn, an, lane, t) * (JT * 32 - 2);
#pragma unroll
          for (int jt = 0; jt < JTD; ++jt) {
            const double b = smem[D::kPkProj + (sp * 2 * JT + jt) * 32 + lane + boff];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], an[m], b);
          }
          if constexpr (kSplitJ) {
#pragma unroll
            for (int gg = 0; gg < kNJR; ++gg) {
              const double b = smem[D::kPkProj + (sp * 2 * JT + JT - 1) * 32 + 4 * gg + t + boff];
#pragma unroll
              for (int m = 0; m < 4; ++m) X[m][gg] = fma(b, an[m], X[m][gg]);
            }
          }
          continue;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jt = 0; jt < JTD; ++jt) {
            const double b = smem[D::kPkProj + ((sp * 2 + i) * JT + jt) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], fn[m][i], b);
          }
        if constexpr (kSplitJ) {
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int gg = 0; gg < kNJR; ++gg) {
              const double b = smem[D::kPkProj + ((sp * 2 + i) * JT + JT - 1) * 32 + 4 * gg + t];
#pragma unroll
              for (int m = 0; m < 4; ++m) X[m][gg] = fma(b, fn[m][i], X[m][gg]);
            }
        }
      }
    } else if constexpr (MODE != kModeVolume) {
      if constexpr (!kEdgeEarly) load_edges();
#pragma unroll kMmaSideUnroll
      for (int q = 0; q < 3; ++q) {
        const int nb = nbq[q];
        const int ed = edq[q];
        const bool left = (inf >> (6 + q)) & 1;
        const bool bnd = nb < 0;
        const int snb = bnd ? 0 : ((inf >> (2 * q)) & 3);
        const double nx = enx[q], ny = eny[q], h = eh[q];
        if (q > 0) {
          cp_async_wait<0>();  // this side's neighbour column / traces (prefetched during the previous side)
          // the trace blocks are copied by other lanes than the ones reading them (each lane's wait
          // covers only its own copies); the coefficient fragments are read by their own copier
          if constexpr (kTrInS) __syncwarp();
        }
        if constexpr (MODE == kModeSurface) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int jt = 0; jt < JT; ++jt) R[m][jt][0] = R[m][jt][1] = 0.0;
        }
        // own trace of side q
        double Tw[4][2], Tn[4][2];
#pragma unroll
        for (int m = 0; m < 4; ++m) Tw[m][0] = Tw[m][1] = Tn[m][0] = Tn[m][1] = 0.0;
        if constexpr (kTrInS) {
#pragma unroll
          for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              const int ko = 2 * t + ii;
              Tw[m][ii] = ko < K ? w_nbr[g * kSSP + m * K + ko] : 0.0;
              Tn[m][ii] = ko < K ? w_nbr[g * kSSP + 4 * K + m * K + (K - 1 - ko)] : 0.0;
            }
        } else {
#pragma unroll
        for (int ks = 0; ks < KSD; ++ks) {
          const double b = smem[D::kPhe + (q * KS + ks) * 32 + lane];
#pragma unroll
          for (int m = 0; m < 4; ++m) dmma(Tw[m], own_a(m, ks), b);
        }
        if constexpr (kSplitK)
          ktail(Tw, smem + D::kPhe + (q * KS + KS - 1) * 32, [&](int m, int jj) { return own_c(m, 4 * (KS - 1) + jj); });
        // neighbour trace (reversed points) — one pass per neighbour side label
        // present in the warp (class renumbering makes that one pass almost always)
        unsigned todo = __reduce_or_sync(0xffffffffu, snb ? (1u << snb) : 0u);
        while (todo) {
          const int s = __ffs(todo) - 1;
          todo &= todo - 1;
          const bool mine = snb == s;
#pragma unroll
          for (int ks = 0; ks < KSD; ++ks) {
            const double b = smem[D::kPheR + ((s - 1) * KS + ks) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const double an = w_nbr[(m * KS + ks) * 32 + lane];
              dmma(Tn[m], mine ? an : 0.0, b);  // a select, not an FP64 multiply
            }
          }
          if constexpr (kSplitK)
            ktail(Tn, smem + D::kPheR + ((s - 1) * KS + KS - 1) * 32, [&](int m, int jj) {
              return mine ? w_nbr[(m * KS + KS - 1) * 32 + 4 * g + jj] : 0.0;
            });
        }
        }  // !kTrInS
        __syncwarp();
        // the neighbour buffer is consumed: prefetch the next side (after side 2: the
        // next tile's side 0 and, the own buffer being free too, its own coefficients)
        if constexpr (kTrInS) {
          if (q < 2) {
            fetch_side_traces(e, valid, q + 1, q == 0 ? nbq[1] : nbq[2], inf);
          } else {
            fetch_side_traces(e_next, nvalid, 0, nbn[0], inf_next);
            if (!kCSmem) own_fetch(tile + nwarps, e_next, nvalid);
          }
        } else if (q < 2) {
          fetch_frag<NP, KS>(w_nbr, a.in, ld, nbq[q + 1], valid && nbq[q + 1] >= 0, lane, t);
        } else {
          fetch_frag<NP, KS>(w_nbr, a.in, ld, nbn[0], nvalid && nbn[0] >= 0, lane, t);
          if (!kCSmem) own_fetch(tile + nwarps, e_next, nvalid);
        }
        cp_async_commit();
        // numerical flux at points ko = 2t + i, canonical orientation
        double fn[4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int ko = 2 * t + i;
          double UO[4], UN[4];
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            UO[m] = Tw[m][i];
            UN[m] = Tn[m][i];
          }
          const int kc = left ? ko : K - 1 - ko;  // canonical (left-element) point index
          const bool live = ko < K;
          if (BND && bnd && live) ghost_state<K>(UO, nb, ed, kc, nx, ny, tstage, geo, UN);  // boundary: left
          const Prim wo = primitives(UO, g1), wn = primitives(UN, g1);
          const double wh = live ? h * smem[D::kWe + (kc < 8 ? kc : 0)] : 0.0;
          double f[4];
          if (admissible(UO, wo) && admissible(UN, wn)) {
            num_flux_own<FLUX>(UO, wo, UN, wn, nx, ny, gamma, wh, left, f);
          } else {
            if (valid && live) record_error(sc, err_key(a.seq, kPassSurface, ed, kc));
#pragma unroll
            for (int m = 0; m < 4; ++m) f[m] = 0.0;
          }
#pragma unroll
          for (int m = 0; m < 4; ++m) fn[m][i] = f[m];
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) {
            const double b = smem[D::kPheP + ((q * 2 + i) * JT + jt) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(R[m][jt], fn[m][i], b);
          }
        if constexpr (MODE == kModeSurface) {
          if (valid) {
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
              for (int jt = 0; jt < JT; ++jt)
#pragma unroll
                for (int ii = 0; ii < 2; ++ii) {
                  const int j = 8 * jt + 2 * t + ii;
                  if (j < NP) a.out[((static_cast<long long>(q) * 4 + m) * NP + j) * ld + e] = R[m][jt][ii];
                }
          }
        }
      }
    } else {
      // volume-only: own prefetch for the next tile
      __syncwarp();
      own_fetch(tile + nwarps, e_next, nvalid);
      cp_async_commit();
    }

    if constexpr (kSplitJ && MODE != kModeSurface) fold_x();

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
      const bool need_u = a.alpha != 0.0 || a.want_resid || kmode == 3;
      const bool need_c = kmode != 3 && a.beta != 0.0;
      // u^n is loaded one variable ahead of the stores (the stores may alias for all the
      // compiler knows, so it cannot hoist the loads itself)
      auto load_u = [&](double(&dst)[JT][2], int m) {
#pragma unroll
        for (int jt = 0; jt < JT; ++jt)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int j = 8 * jt + 2 * t + ii;
            dst[jt][ii] = (need_u && j < NP) ? __ldg(a.u + (static_cast<long long>(m) * NP + j) * ld + e) : 0.0;
          }
      };
      double uv_next[JT][2];
      if (kUAhead) load_u(uv_next, 0);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        // this variable's u^n, stage input and RK4 accumulator: every load issued
        // before any store, so one memory latency per variable
        double uv[JT][2], cv[JT][2], kv[JT][2];
        if (kUAhead) {
#pragma unroll
          for (int jt = 0; jt < JT; ++jt) uv[jt][0] = uv_next[jt][0], uv[jt][1] = uv_next[jt][1];
          if (m + 1 < 4) load_u(uv_next, m + 1);
        }
#pragma unroll
        for (int jt = 0; jt < JT; ++jt)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) {
            const int j = 8 * jt + 2 * t + ii;
            const long long idx = (static_cast<long long>(m) * NP + j) * ld + e;
            if (!kUAhead) uv[jt][ii] = (need_u && j < NP) ? __ldg(a.u + idx) : 0.0;
            if constexpr (kCSmem) {  // element g's mode j from the tile's own fragment buffer
              cv[jt][ii] = (need_c && j < NP) ? (kTma ? w_own[(m * NP + j) * 8 + g]
                                                      : w_own[(m * KS + (j >> 2)) * 32 + (g << 2) + (j & 3)])
                                              : 0.0;
            } else {
              cv[jt][ii] = (need_c && j < NP) ? __ldg(a.in + idx) : 0.0;
            }
            kv[jt][ii] = ((kmode == 2 || kmode == 3) && j < NP) ? a.kacc[idx] : 0.0;
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
              if (kmode == 3) {
                o = fma(dt6, kv[jt][ii] + d, uu);
              } else {
                const double base = (a.alpha != 0.0) ? fma(a.alpha, uu, a.beta * cj) : a.beta * cj;
                o = fma(gdt, d, base);
                if (kmode == 1 && valid) a.kacc[idx] = d;
                if (kmode == 2 && valid) a.kacc[idx] = fma(2.0, d, kv[jt][ii]);
              }
              if (valid) {
                a.out[idx] = o;
                if (a.want_resid) res_max = std_max(res_max, fabs(uu - o));
              }
              R[m][jt][ii] = o;  // keep the new stage for the CFL epilogue
            } else {
              R[m][jt][ii] = 0.0;
            }
          }
      }
      if (want_lambda) {
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
        double lam = 0.0;
        bool ok;
        const double ws = wave_speed_ieee(U, __ldg(geo.enx + edq), __ldg(geo.eny + edq), gamma, ok);
        if (ok) {
          lam = ws;
        } else if (valid && t < 3) {
          record_error(sc, err_key(a.seq_next, kPassDt, __ldg(geo.ref_id + e), t + 1));
        }
        if (t == 3) lam = 0.0;
        lam = std_max(lam, __shfl_xor_sync(0xffffffffu, lam, 1));
        lam = std_max(lam, __shfl_xor_sync(0xffffffffu, lam, 2));
        if (valid && t == 0) lam_min = std_min(lam_min, 2.0 * __ldg(geo.inradius + e) / ((2.0 * P + 1.0) * lam));
      }
    }
    if constexpr (MODE == kModeStage && DGB_TRACE_P(P)) {
      if (a.tr_out) {
        // traces of the new stage for the next stage's kVarTrace instance: the new coefficients
        // go through the own buffer into the A-fragment order, then the surface's packed
        // own-trace contraction (same tables, same order: the values the next stage would
        // interpolate itself, for this element and as the neighbour of its neighbours)
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int jt = 0; jt < JT; ++jt)
#pragma unroll
            for (int ii = 0; ii < 2; ++ii) {
              const int j = 8 * jt + 2 * t + ii;
              if (j < NP) w_own[kTma ? (m * NP + j) * 8 + g : (m * KS + (j >> 2)) * 32 + (g << 2) + (j & 3)] = R[m][jt][ii];
            }
        __syncwarp();
        if constexpr (D::kPacked) {
#pragma unroll
        for (int sp = 0; sp < D::NSP; ++sp) {
          double Tw[4][2];
#pragma unroll
          for (int m = 0; m < 4; ++m) Tw[m][0] = Tw[m][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < KSD; ++ks) {
            const double b = smem[D::kPkOwn + (sp * KS + ks) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(Tw[m], own_a(m, ks), b);
          }
          if constexpr (kSplitK)
            ktail(Tw, smem + D::kPkOwn + (sp * KS + KS - 1) * 32, [&](int m, int jj) { return own_c(m, 4 * (KS - 1) + jj); });
          if (valid) {
            if constexpr (K % 2 == 0) {  // the lane's two points are adjacent in one side: one 16-byte store
              const int pt = 8 * sp + 2 * t;
              if (pt < K3) {
#pragma unroll
                for (int m = 0; m < 4; ++m)
                  *reinterpret_cast<double2*>(a.tr_out + static_cast<long long>(e) * kTS + ((pt / K) * 4 + m) * K + pt % K) =
                      make_double2(Tw[m][0], Tw[m][1]);
              }
            } else {
#pragma unroll
              for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int ii = 0; ii < 2; ++ii) {
                  const int pt = 8 * sp + 2 * t + ii;
                  if (pt < K3) a.tr_out[static_cast<long long>(e) * kTS + ((pt / K) * 4 + m) * K + pt % K] = Tw[m][ii];
                }
            }
          }
        }
        } else {  // per-side surface: side q's own-trace contraction (kPhe)
#pragma unroll kMmaSideUnroll
        for (int q = 0; q < 3; ++q) {
          double Tw[4][2];
#pragma unroll
          for (int m = 0; m < 4; ++m) Tw[m][0] = Tw[m][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < KSD; ++ks) {
            const double b = smem[D::kPhe + (q * KS + ks) * 32 + lane];
#pragma unroll
            for (int m = 0; m < 4; ++m) dmma(Tw[m], own_a(m, ks), b);
          }
          if constexpr (kSplitK)
            ktail(Tw, smem + D::kPhe + (q * KS + KS - 1) * 32, [&](int m, int jj) { return own_c(m, 4 * (KS - 1) + jj); });
          if (valid) {
            if constexpr (K % 2 == 0) {
              if (2 * t < K) {
#pragma unroll
                for (int m = 0; m < 4; ++m)
                  *reinterpret_cast<double2*>(a.tr_out + static_cast<long long>(e) * kTS + (q * 4 + m) * K + 2 * t) =
                      make_double2(Tw[m][0], Tw[m][1]);
              }
            } else {
#pragma unroll
              for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int ii = 0; ii < 2; ++ii) {
                  const int ko = 2 * t + ii;
                  if (ko < K) a.tr_out[static_cast<long long>(e) * kTS + (q * 4 + m) * K + ko] = Tw[m][ii];
                }
            }
          }
        }
        }
      }
    }
    if constexpr (kCSmem) {  // the own buffer is free only now
      __syncwarp();
      own_fetch(tile + nwarps, e_next, nvalid);
      cp_async_commit();
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) nbq[q] = nbn[q];
  }
  cp_async_wait<0>();

  if constexpr (MODE == kModeStage) {
    const int par = a.step & 1;
    if (want_lambda) block_reduce_atomic<true>(lam_min, &sc->dtmin[par ^ 1]);
    if (a.want_resid) block_reduce_atomic<false>(res_max, &sc->resid[par]);
  }
}

// Host-side preparation of the fragment-ordered tables (see MmaDim for the layout).
template <int P>
inline void fill_mma_tab(const Tab<P>& T, double* out) {
  using D = MmaDim<P>;
  constexpr int NP = D::NP, NQ = D::NQ, K = D::K, KS = D::KS, NT = D::NT, JT = D::JT;
  for (int i = 0; i < D::kSize; ++i) out[i] = 0.0;
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;  // B fragment: row t, column g
    for (int ks = 0; ks < KS; ++ks)
      for (int nt = 0; nt < NT; ++nt) {
        const int j = 4 * ks + t, k = 8 * nt + g;
        out[D::kPhi + (ks * NT + nt) * 32 + lane] = (j < NP && k < NQ) ? T.phi[k][j] : 0.0;
      }
    for (int nt = 0; nt < NT; ++nt)
      for (int i = 0; i < 2; ++i)
        for (int jt = 0; jt < JT; ++jt) {
          const int k = 8 * nt + 2 * t + i, j = 8 * jt + g;
          const bool ok = k < NQ && j < NP;
          out[D::kDr + ((nt * 2 + i) * JT + jt) * 32 + lane] = ok ? T.drw[k][j] : 0.0;
          out[D::kDs + ((nt * 2 + i) * JT + jt) * 32 + lane] = ok ? T.dsw[k][j] : 0.0;
        }
    for (int q = 0; q < 3; ++q)
      for (int ks = 0; ks < KS; ++ks) {
        const int j = 4 * ks + t, ko = g;
        const bool ok = j < NP && ko < K;
        out[D::kPhe + (q * KS + ks) * 32 + lane] = ok ? T.phe[q][ko][j] : 0.0;
        out[D::kPheR + (q * KS + ks) * 32 + lane] = ok ? T.phe[q][K - 1 - ko][j] : 0.0;
      }
    for (int q = 0; q < 3; ++q)
      for (int i = 0; i < 2; ++i)
        for (int jt = 0; jt < JT; ++jt) {
          const int ko = 2 * t + i, j = 8 * jt + g;
          out[D::kPheP + ((q * 2 + i) * JT + jt) * 32 + lane] = (ko < K && j < NP) ? T.phe[q][ko][j] : 0.0;
        }
  }
  for (int q = 0; q < 3; ++q)
    for (int j = 0; j < NP; ++j) out[D::kPhm + q * JT * 8 + j] = T.phm[q][j];
  for (int k = 0; k < K; ++k) out[D::kWe + k] = T.we[k];
  if (D::kPacked) {
    for (int sp = 0; sp < D::NSP; ++sp)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        for (int ks = 0; ks < KS; ++ks) {
          const int j = 4 * ks + t, pt = 8 * sp + g;  // B[row t = mode][col g = packed point]
          const bool okc = j < NP && pt < 3 * K;
          const int q = okc ? pt / K : 0, ko = okc ? pt % K : 0;
          out[D::kPkOwn + (sp * KS + ks) * 32 + lane] = okc ? T.phe[q][ko][j] : 0.0;
          for (int qq = 0; qq < 3; ++qq)
            for (int cls = 0; cls < 3; ++cls)  // neighbour side label cls+1, reversed points
              out[D::kPkNb + (((sp * 3 + qq) * 3 + cls) * KS + ks) * 32 + lane] =
                  (okc && q == qq) ? T.phe[cls][K - 1 - ko][j] : 0.0;
        }
        for (int i = 0; i < 2; ++i)
          for (int jt = 0; jt < JT; ++jt) {
            const int pt = 8 * sp + 2 * t + i, j = 8 * jt + g;  // B[row t = k slot][col g = mode]
            const bool ok = pt < 3 * K && j < NP;
            out[D::kPkProj + ((sp * 2 + i) * JT + jt) * 32 + lane] = ok ? T.phe[pt / K][pt % K][j] : 0.0;
          }
      }
  }
  if (D::kTail1) {
    const int k = NQ - 1;
    for (int j = 0; j < NP; ++j) {
      out[D::kTail + j] = T.phi[k][j];  // mode j = 4ks + t sits at ks*4 + t
      out[D::kTail + KS * 4 + j] = T.drw[k][j];
      out[D::kTail + KS * 4 + JT * 8 + j] = T.dsw[k][j];
    }
  }
}

}  // namespace dgbk
