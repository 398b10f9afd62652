// sm_100a kernels for the modal-DG Euler right-hand side and RK stage.
//
// One fused element-centric kernel replaces the reference's three passes
// (proj/src/solver.cpp: eval_volume_pass :99-158, eval_surface_pass :160-251,
// eval_rhs_pass :253-277) plus the stage axpy / rk4_combine (:483-504), the
// residual (:672-678) and the per-element CFL bound (:427-461):
//
//   * G lanes per element (template), each lane owns 4/G conserved variables;
//     full states at a point are assembled with warp shuffles.
//   * all basis tables live in __constant__ banks; every contraction is a
//     fully unrolled DFMA chain with a constant-bank operand.
//   * each element evaluates the numerical flux of its three edges itself, in
//     the edge's canonical left->right orientation with identical operands on
//     both sides, so the two sides of an edge receive bit-identical fluxes and
//     conservation is exact (no edge buffer, no atomics, no second pass).
//   * the neighbour's side label is warp-uniform after the host's class
//     renumbering, so the neighbour-trace switch does not diverge.
//
// Coefficients are SoA [4][n_p][ld] in device element order (ld = padded N),
// coalesced across elements exactly as the reference's CoefficientArray.
#pragma once

#include <cstdint>

namespace dgbk {

template <int P>
struct Dim {
  static constexpr int NP = (P + 1) * (P + 2) / 2;
  static constexpr int NQ = P == 1 ? 3 : P == 2 ? 6 : P == 3 ? 12 : P == 4 ? 16 : 25;
  static constexpr int K = P + 1;
};

// Basis tables of one degree (basis.hpp:48-82), volume gradients pre-scaled by
// the interior weights.
template <int P>
struct Tab {
  double phi[Dim<P>::NQ][Dim<P>::NP];
  double drw[Dim<P>::NQ][Dim<P>::NP];  // w_k * dphi/dr
  double dsw[Dim<P>::NQ][Dim<P>::NP];  // w_k * dphi/ds
  double phe[3][Dim<P>::K][Dim<P>::NP];
  double we[Dim<P>::K];
  double phm[3][Dim<P>::NP];
};

// Limiter evaluation points for p = 1 (solver.cpp:296-322).
struct LimTab {
  double phi1[64], phi2[64];
  double max_phi1, max_phi2;
  int n_pts, edge_begin, n_edge;
};

// Boundary codes (euler.hpp:80-86).
enum : int { kReflecting = -1, kCurved = -2, kInflow = -3, kOutflow = -4, kShock = -5 };

// Passes recorded in an error key (lower wins at equal sequence number).
enum : int { kPassDt = 0, kPassVolume = 1, kPassSurface = 2 };

constexpr unsigned long long kNoError = ~0ull;

// Device-resident per-run scalars; parity-indexed slots let a whole batch of
// steps run without host round trips ("device step loop").
struct Scalars {
  unsigned long long err_key;  // min over (seq, pass, id, point); kNoError = none
  int halt;                    // set when a driver stop rule fired
  int halt_step;               // relative step index at which it fired
  double t[2];                 // time at the start of step s lives in t[s & 1]
  unsigned long long dtmin[2]; // bits of min_i 2 r_i / ((2p+1) lambda_i) for step s in [s & 1]
  unsigned long long resid[2]; // bits of max |u_new - u| of step s in [s & 1]
  double dt_used[2];           // dt of step s in [s & 1]
};

// Peer-memory halo exchange (multi-GPU).  One entry per
// rank of the job; the local rank's entry is unused.
constexpr int kMaxRanks = 8;
struct PeerTab {
  double* buf[kMaxRanks][4];            // the peer's rotating coefficient buffers (state0/1, stage0/1)
  long long ld[kMaxRanks];              // the peer's leading dimension
  unsigned long long* flag[kMaxRanks];  // the peer's flag array [kMaxRanks] (we write our slot)
  unsigned long long* scal[kMaxRanks];  // the peer's scalar exchange [2][kMaxRanks][4]
};

struct Geo {
  int N, ld;                           // N = owned elements (device columns [0, N)); halo columns follow
  const double* __restrict__ tau;      // [4][ld]
  const double* __restrict__ inv_det;  // [ld]
  const double* __restrict__ inradius; // [ld]
  const int* __restrict__ nbr;         // [3][ld] device id of the neighbour or the BC code
  const int* __restrict__ eid;         // [3][ld] edge id (reference numbering)
  const int* __restrict__ info;        // [ld] bits 2q..2q+1: neighbour side label (0 = boundary); bit 6+q: left
  const int* __restrict__ ref_id;      // [ld] reference element id
  const double* __restrict__ enx;      // [n_edges]
  const double* __restrict__ eny;
  const double* __restrict__ eh;
  const double* __restrict__ bstate;   // [n_bnd][K][4] Dirichlet states
  const double* __restrict__ bwn;      // [n_bnd][K][2] exact wall normals
  const double* __restrict__ bx;       // [n_bnd][K][2] boundary Gauss points
  int has_dir, has_wn, has_shock;
  int has_bnd;                         // some owned element has a physical-boundary side
  double inflow[4];
  double sh_x0, sh_cos, sh_sin, sh_speed;
  double sh_post[4], sh_pre[4];
  double gamma;
  // basis tables in DMMA fragment order (element_mma.cuh), p >= 3
  const double* __restrict__ mma_tab;
  int flux;  // numerical flux: 0 local Lax-Friedrichs (euler.hpp:59-71), 1 Roe
  // launch forms (kernels_tu.cuh, kernels_p1.cu): launches of at most this many elements take
  // the four-lane latency form of the p <= 2 stage kernel / the limiter; -1 = the built-in size
  int lat_stage_n, lat_limit_n;
};

// Modes of the fused element kernel.
enum : int { kModeVolume = 0, kModeSurface = 1, kModeRhs = 2, kModeStage = 3 };

// Instance variants of the element kernel (bit set): the RK4 derivative accumulator is in
// use, the CFL wave speeds are wanted (last stage of a step), the partition has elements
// on the physical boundary.  Each unused path is compiled out of its instance, which
// frees registers in the common case (SSP / midpoint stages, periodic meshes).
enum : int { kVarRk4 = 1, kVarLambda = 2, kVarBoundary = 4, kVarTrace = 8 };
// kVarTrace (stage mode, packed-surface degrees p = 3, 4): the own and neighbour edge traces of
// the stage input are read from the trace buffer its producing stage wrote (StageArgs::tr_in)
// instead of being interpolated from the coefficient columns.

struct StageArgs {
  const double* __restrict__ in;  // stage input coefficients
  // TMA tensor map (CUtensorMap in global memory) of `in` viewed as [4][n_p][ld] doubles, box
  // 8 elements x n_p modes x 4 variables: the DMMA kernel (p >= 3) loads each tile's own
  // coefficients with one cp.async.bulk.tensor; null = per-lane cp.async
  const void* tm_in;
  const double* __restrict__ u;   // u^n (for alpha, residual, rk4 combine)
  double* __restrict__ out;       // output (volume / slots / deriv / next stage)
  double* __restrict__ kacc;      // RK4 derivative accumulator
  double* __restrict__ means;     // p <= 2 with a limiter kernel next: the new cell means, [ld][4] (null: none)
  // edge traces, element-major [ld][3 sides][4 variables][K points] (the element's own orientation):
  // tr_in those of `in` (kVarTrace instances), tr_out those of `out` (written when non-null)
  const double* __restrict__ tr_in;
  double* __restrict__ tr_out;
  double alpha, beta, gcoef;      // out = alpha u + beta in + (gcoef dt) L(in)
  double tcoef;                   // stage time = t + tcoef dt
  int kmode;                      // 0 none, 1 kacc = L, 2 kacc += 2L, 3 out = u + dt/6 (kacc + L)
  int dt_mode;                    // 0: dt_host, 1: cfl * dtmin[parity] (clipped to t_end if clip)
  double dt_host, cfl, t_end;
  int clip_t_end;                 // run_to_time: clip the last step
  int stop_at_t_end;              // run_to_time: halt when t >= t_end at step start
  int stop_steady;                // run_to_steady: halt when resid of previous step <= tol
  double tol;
  int step;                       // relative step index (parity = step & 1)
  int first, last;                // first / last stage of the step
  int want_lambda, want_resid;    // fused epilogues (off when a final limiter follows)
  double t_host;                  // time for pass-level calls (dt_mode irrelevant)
  int use_t_host;
  unsigned long long seq;         // error sequence number of this launch
  unsigned long long seq_next;    // sequence number of the next step's CFL pass
  Scalars* sc;
  double* hist;                   // optional residual history (on_step)
  int e0, e1;                     // device element range of this launch
};

// Fused stage + limiter launch (p = 1 with limiting, kernels_p1.cu k_stage_limit).  Work unit:
// a tile of 32 elements (one warp).  Warp w of W (a cooperative launch: every warp resident)
// runs tiles w, w + W, ...: the stage of tile i, published by adding 1 to the counter of its
// chunk (kFuseChunk tiles), then the limiter of tile i - lag once every chunk holding a
// neighbour of that tile has published this launch.  Counters only grow: a chunk of s tiles is
// complete for launch `epoch` (1, 2, ... since the run started) at epoch * s.
constexpr int kFuseTile = 32;   // elements per tile (one warp)
constexpr int kFuseChunk = 32;  // tiles per chunk counter
struct FuseArgs {
  unsigned long long* count;  // [n_chunks] publications so far (reset at the start of each run)
  const int2* range;          // [n_tiles] (first, last) chunk holding a neighbour of the tile (own included)
  int n_tiles, lag;
  unsigned long long epoch;   // launches of this run so far, this one included
};

struct LimArgs {
  double* __restrict__ c;         // limited in place
  const double* __restrict__ means;  // the stage kernel's compact copy of c's mode 0, [ld][4] (null: read c)
  const double* __restrict__ u;   // for the residual (final limit)
  int step, want_lambda, want_resid;
  unsigned long long seq;         // error key for the CFL epilogue (next step)
  Scalars* sc;
  int e0, e1;                     // device element range of this launch
};

}  // namespace dgbk
