// Device context and C ABI of the solver half (include/dg2d_b200/dg2d_b200.h).
//
// Owns the device-resident mesh (SoA, class-renumbered element order), the
// coefficient slots, the per-run scalars and the step drivers that replace the
// reference's rk_step_ws / run_* loops (proj/src/solver.cpp:506-613) with a
// device step loop: dt, stop rules and residuals stay on the GPU and the host
// synchronises once per batch of steps.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/dg2d_b200/dg2d_b200.h"
#include "../host/capi_common.hpp"
#include "dg_kernels.cuh"
#include "launch.hpp"

using dgbk::Geo;
using dgbk::LimArgs;
using dgbk::Scalars;
using dgbk::StageArgs;

namespace {

constexpr int kWindow = 256;  // renumbering window (elements), multiple of 32
constexpr int kBatch = 64;    // steps per host synchronisation in open-ended drivers
constexpr int kFuseMaxN = 400000;  // fused stage + limiter launch by default up to this many elements (crossover measured between 184K and 737K)

struct Fail {
  int code;
  std::string msg;
};

#ifndef DGB_TRACE_BUF_DEFAULT
#define DGB_TRACE_BUF_DEFAULT 1  // trace-buffer stage instances (the degrees of DGB_TRACE_P) by default
#endif
#define CU(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) throw Fail{DGB_ERR_CUDA, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #call}; \
  } while (0)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count) CU(cudaMalloc(&p, count * sizeof(T)));
  }
  // alloc, then zero on `s` (coefficient buffers: the DMMA kernel's TMA boxes read the padding
  // columns past N, never using them; zeroed they hold defined values)
  void alloc_zero(size_t count, cudaStream_t s) {
    alloc(count);
    if (count) CU(cudaMemsetAsync(p, 0, count * sizeof(T), s));
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) CU(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// ------------------------------------------------------------------ small kernels
// Reference (host) layout <-> device layout.  Host arrays are [rows][n_host] in
// "compact" order: the reference order for a whole-mesh context, and for a
// partition the owned elements (ascending reference id) followed by the halo
// elements (ascending reference id).  cmp[d] = compact index of device column d.
__global__ void k_permute_in(double* __restrict__ dst, const double* __restrict__ src, const int* __restrict__ cmp,
                             int n_cols, int n_host, int ld, int rows) {
  const long long total = static_cast<long long>(rows) * ld;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(t / ld), d = static_cast<int>(t % ld);
    dst[t] = d < n_cols ? src[static_cast<long long>(r) * n_host + cmp[d]] : 0.0;
  }
}

__global__ void k_permute_out(double* __restrict__ dst, const double* __restrict__ src, const int* __restrict__ cmp,
                              int n_cols, int n_host, int ld, int rows) {
  const long long total = static_cast<long long>(rows) * ld;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(t / ld), d = static_cast<int>(t % ld);
    if (d < n_cols) dst[static_cast<long long>(r) * n_host + cmp[d]] = src[t];
  }
}

// ------------------------------------------------------------------ halo exchange
// Error key of an exchange timeout (sorts before every solver error).
constexpr unsigned long long kTimeoutKey = (7ull << 35);

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Halo push: copy the new coefficient columns of the send elements into the halo columns of
// every peer that needs them, over NVLink peer memory (plain global stores into the peers'
// IPC-mapped buffers).  Entry i = (own column, peer rank, peer column); thread k covers row
// k / n of entry k % n, so a warp stores one row of consecutive entries, which the host sorted
// by (peer, peer column).  Kept out of the stage and limiter kernels: the push code there cost
// the whole-mesh instances registers and issue slots.
__global__ void k_push(const dgbk::PeerTab* __restrict__ pt, int buf, const double* __restrict__ src, long long ld,
                       const int4* __restrict__ ent, int n, int rows, int tblock) {
  // rows [0, rows): coefficient rows (column e of row r at r ld + e); then (trace mode) the
  // element-major trace blocks after them (tblock doubles per element at rows ld + e tblock)
  const long long total = static_cast<long long>(n) * (rows + tblock);
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(k / n), i = static_cast<int>(k - static_cast<long long>(r) * n);
    const int4 e = __ldg(ent + i);
    const long long pld = pt->ld[e.y];
    double* dst = pt->buf[e.y][buf];
    if (r < rows) {
      dst[static_cast<long long>(r) * pld + e.z] = src[static_cast<long long>(r) * ld + e.x];
    } else {
      const int o = r - rows;
      dst[static_cast<long long>(rows) * pld + static_cast<long long>(e.z) * tblock + o] =
          src[static_cast<long long>(rows) * ld + static_cast<long long>(e.x) * tblock + o];
    }
  }
  __threadfence_system();  // visible at the peers before the signal kernel's flag
}

// One warp: publish (optionally) this rank's step scalars into every peer of
// `mask`, then raise our flag there to `epoch`.  The push kernel before it fenced
// the halo values (system scope) before it completed.
__global__ void k_signal(const dgbk::PeerTab* __restrict__ pt, unsigned mask, int me, unsigned long long epoch,
                         const dgbk::Scalars* __restrict__ sc, int publish, int slot, int dt_idx, int res_idx) {
  const int r = threadIdx.x;
  unsigned long long v0 = 0, v1 = 0, v2 = 0;
  if (publish) {
    v0 = sc->dtmin[dt_idx];
    v1 = sc->resid[res_idx];
    v2 = sc->err_key;
  }
  __threadfence_system();
  if (r < dgbk::kMaxRanks && ((mask >> r) & 1u)) {
    if (publish) {
      unsigned long long* dst = pt->scal[r] + (static_cast<long long>(slot) * dgbk::kMaxRanks + me) * 4;
      dst[0] = v0;
      dst[1] = v1;
      dst[2] = v2;
      __threadfence_system();
    }
    st_release_sys(pt->flag[r] + me, epoch);
  }
}

// One warp: wait until every rank of `mask` raised its flag in our memory to
// at least `epoch` (bounded by a timeout that turns into an error key), then
// optionally merge the published scalars: min dt bound, max residual, min error.
__global__ void k_wait(const unsigned long long* __restrict__ flags, const unsigned long long* __restrict__ scal,
                       unsigned mask, unsigned long long epoch, dgbk::Scalars* sc, int merge, int slot, int dt_idx,
                       int res_idx, unsigned long long timeout_ns) {
  const int r = threadIdx.x;
  bool ok = true;
  if (r < dgbk::kMaxRanks && ((mask >> r) & 1u)) {
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(flags + r) < epoch) {
      if (global_ns() - t0 > timeout_ns) {
        ok = false;
        break;
      }
      __nanosleep(64);
    }
  }
  ok = __all_sync(0xffffffffu, ok);
  if (r != 0) return;
  if (!ok) {
    atomicMin(&sc->err_key, kTimeoutKey);
    return;
  }
  if (!merge) return;
  __threadfence_system();
  for (int k = 0; k < dgbk::kMaxRanks; ++k) {
    if (!((mask >> k) & 1u)) continue;
    const unsigned long long* v = scal + (static_cast<long long>(slot) * dgbk::kMaxRanks + k) * 4;
    const unsigned long long v0 = ld_acquire_sys(v), v1 = ld_acquire_sys(v + 1), v2 = ld_acquire_sys(v + 2);
    if (v0 < sc->dtmin[dt_idx]) sc->dtmin[dt_idx] = v0;  // non-negative doubles order like their bits
    if (v1 > sc->resid[res_idx]) sc->resid[res_idx] = v1;
    if (v2 < sc->err_key) sc->err_key = v2;
  }
}

// eval_rhs_pass (solver.cpp:253-277): (volume + slot_0 + slot_1 + slot_2) * (1/det)
__global__ void k_gather(double* __restrict__ deriv, const double* __restrict__ vol, const double* __restrict__ slots,
                         const double* __restrict__ inv_det, int n, int ld, int rows) {
  const long long total = static_cast<long long>(rows) * ld;
  const long long qs = static_cast<long long>(rows) * ld;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int d = static_cast<int>(t % ld);
    if (d >= n) continue;
    double acc = vol[t];
    acc += slots[t];
    acc += slots[qs + t];
    acc += slots[2 * qs + t];
    deriv[t] = acc * inv_det[d];
  }
}

// compute_l2_error (runner.cpp:127-150), per-element partials: det_i * sum_k w_k (rho_h - rho_ex)^2.
// exact[(local i) * nq + k] holds the exact density at interior point k of owned element i (reference
// order); part[local i] receives the partial (the host adds them in element order).
__global__ void k_l2_partial(const double* __restrict__ c, const double* __restrict__ exact,
                             const double* __restrict__ tab /* phi[nq][np], w[nq] */, const int* __restrict__ cmp,
                             const double* __restrict__ inv_det, int n, int ld, int np, int nq, double* part) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const int i = cmp[d];
    double acc = 0.0;
    for (int k = 0; k < nq; ++k) {
      double rho = 0.0;
      for (int j = 0; j < np; ++j) rho += c[static_cast<long long>(j) * ld + d] * tab[k * np + j];
      const double diff = rho - exact[static_cast<long long>(i) * nq + k];
      acc += tab[nq * np + k] * diff * diff;
    }
    part[i] = acc / inv_det[d];
  }
}

// project_initial (solver.cpp:74-97) on the device: coefficient (m, j) of element i is
// sum_k w_k phi[k][j] u_k[m] (orthonormal basis: the mass matrix is detJ I, which cancels
// against the detJ of the quadrature); ps[(i * nq + k) * 4 + m] in reference order.
__global__ void k_project(const double* __restrict__ ps, const double* __restrict__ tab /* phi[nq][np], w[nq] */,
                          const int* __restrict__ cmp, int n, int ld, int np, int nq, double* __restrict__ c,
                          double gamma, unsigned long long* bad) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const long long i = cmp[d];
    for (int m = 0; m < 4; ++m)
      for (int j = 0; j < np; ++j) {
        double s = 0.0;
        for (int k = 0; k < nq; ++k) s += tab[nq * np + k] * tab[k * np + j] * ps[(i * nq + k) * 4 + m];
        c[(static_cast<long long>(m) * np + j) * ld + d] = s;
      }
    for (int k = 0; k < nq; ++k) {  // admissibility, lowest (element, point) wins as on the host
      const double* u = ps + (i * nq + k) * 4;
      const double pr = (gamma - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
      if (!(u[0] > 0.0 && pr > 0.0)) atomicMin(bad, static_cast<unsigned long long>(i) * 64 + k);
    }
  }
}

// Output extraction (output.cpp:10-20, 30-65): the state at the three corners of every
// owned element, out[(i * 3 + c) * 4 + m] (reference order), same j order as corner_state.
__global__ void k_corner_states(const double* __restrict__ c, const double* __restrict__ phic /* [3][np] */,
                                const int* __restrict__ cmp, int n, int ld, int np, double* __restrict__ out) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const long long i = cmp[d];
    for (int cc = 0; cc < 3; ++cc)
      for (int m = 0; m < 4; ++m) {
        double s = 0.0;
        for (int j = 0; j < np; ++j) s = fma(c[(static_cast<long long>(m) * np + j) * ld + d], phic[cc * np + j], s);
        out[(i * 3 + cc) * 4 + m] = s;
      }
  }
}

__global__ void k_max_abs_diff(const double* __restrict__ a, const double* __restrict__ b, int n, int ld, int rows,
                               unsigned long long* out) {
  const long long total = static_cast<long long>(rows) * ld;
  double m = 0.0;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (static_cast<int>(t % ld) < n) m = fmax(m, fabs(a[t] - b[t]));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// FP64 FMA-pipe peak probe: 8 independent DFMA chains per thread, all SMs.
__global__ void k_fp64_peak(double* out, int iters) {
  double a[8];
  const double m = 1.0000001, c = 1e-9;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int small_grid(long long work) {
  long long g = (work + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

double pressure_ref(const double* u, double gamma) {
  return (gamma - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
}

struct StageSpec {
  double alpha, beta, gcoef, tcoef;
  int kmode;
};

bool scheme_stages(int scheme, std::vector<StageSpec>& st) {
  switch (scheme) {
    case DGB_RK2_MIDPOINT:  // solver.cpp:513-519
      st = {{0.0, 1.0, 0.5, 0.0, 0}, {1.0, 0.0, 1.0, 0.5, 0}};
      return true;
    case DGB_RK4_CLASSIC:  // solver.cpp:520-531
      st = {{0.0, 1.0, 0.5, 0.0, 1}, {1.0, 0.0, 0.5, 0.5, 2}, {1.0, 0.0, 1.0, 0.5, 2}, {0.0, 0.0, 0.0, 1.0, 3}};
      return true;
    case DGB_SSP_RK2:  // Heun / SSP(2,2)
      st = {{0.0, 1.0, 1.0, 0.0, 0}, {0.5, 0.5, 0.5, 1.0, 0}};
      return true;
    case DGB_SSP_RK3:  // Shu-Osher SSP(3,3)
      st = {{0.0, 1.0, 1.0, 0.0, 0}, {0.75, 0.25, 0.25, 1.0, 0}, {1.0 / 3.0, 2.0 / 3.0, 2.0 / 3.0, 0.5, 0}};
      return true;
    default:
      return false;
  }
}

}  // namespace

// ------------------------------------------------------------------ context
struct dgb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // asynchronous host copies (dgb_upload_async / dgb_download_async): one copy stream per
  // direction and a staging buffer each, so a result's device->host copy overlaps the
  // next input's host->device copy (PCIe is full duplex)
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d = nullptr, ev_in_free = nullptr, ev_perm_out = nullptr, ev_out_free = nullptr;
  bool staged = false;  // an input is (being) copied into staging_in and not yet committed
  int p = 1, np = 3, nq = 3, K = 2;
  int N = 0, ld = 0, n_edges = 0, n_bnd = 0;
  double gamma = 1.4;

  // host copies needed for diagnostics and reference-layout conversions
  std::vector<double> vx, vy, det;
  std::vector<int32_t> elem_v, elem_edge, eleft, eright, esl, esr, ev0, ev1;
  std::vector<double> enx, eny;
  std::vector<double> bc_dir, bc_wn;
  dgb_bc_view bc{};
  std::vector<double> t_phi, t_phe, t_phm, t_xi, t_w;
  std::vector<int> ref_of;   // device column -> reference element id (owned, then halo)
  std::vector<int> col_of;   // reference element id -> device column (-1 when not local)
  std::vector<int> halo_gid; // reference ids of the halo columns [N, N + n_halo)

  // partition (multi-GPU); a whole-mesh context is rank 0 of 1
  int rank = 0, world = 1, lo = 0, hi = 0, n_global = 0, n_int = 0, n_halo = 0;
  bool partitioned = false, finalized = true;
  unsigned nb_mask = 0;                       // ranks owning our halo elements (we wait on them)
  unsigned send_mask = 0;                     // ranks fed from our send elements (we signal them)
  std::vector<std::vector<std::pair<int, int>>> sends;  // per peer: (reference id, peer column)
  dgbk::PeerTab h_peers{};
  dgbk::PeerTab* d_peers = nullptr;
  unsigned long long* d_xch = nullptr;        // flags[kMaxRanks] + scalar slots [2][kMaxRanks][4]
  std::vector<void*> ipc_opened;
  DevBuf<int> d_cmp;
  DevBuf<int4> d_push;                        // halo push entries (own column, peer, peer column)
  int n_push = 0;
  unsigned long long epoch = 0;               // signals sent so far (same sequence on every rank)
  unsigned long long pub_epoch = 0;           // epoch of the last scalar publish
  int64_t n_pub = 0;                          // publishes so far (slot = n_pub & 1)
  double timeout_s = 60.0;
  std::string bc_error;  // deferred boundary-condition failure (reference throws in the surface pass)

  // device geometry
  DevBuf<double> d_tau, d_inv_det, d_inradius, d_enx, d_eny, d_eh, d_bstate, d_bwn, d_bx, d_mma;
  // Dirichlet tables at the stage times of the next step (time-dependent boundary data,
  // dgb_set_dirichlet_stages): stage k of a step reads table min(k, n_dir_stages - 1)
  DevBuf<double> d_bstage;
  int n_dir_stages = 0;
  DevBuf<int> d_nbr, d_eid, d_info, d_ref_id;  // d_ref_id: reference id of each device column
  Geo geo = [] {
    Geo g{};
    g.lat_stage_n = g.lat_limit_n = -1;  // built-in latency-form sizes
    return g;
  }();

  // coefficient buffers (device order [4][np][ld])
  DevBuf<double> state[2], input, volume, deriv, stage[2], kacc, slots, staging, hist, staging_in, staging_out;
  DevBuf<double> means;  // [ld][4] cell means of the last stage output (two-kernel limiter path)
  int k3 = 0;               // 3K when the degree has trace-buffer stage instances, else 0
  int trace_mode = -1;      // 1 on, 0 off, -1 default (env DGB_TRACE_BUF, else on)
  int cur = 0;
  Scalars* d_sc = nullptr;
  Scalars* h_sc = nullptr;  // pinned mirror
  unsigned long long* d_red = nullptr;
  unsigned long long* h_red = nullptr;

  double t = 0.0;
  int64_t step_count = 0;
  dgb_abort_info last_abort{};

  // timers
  bool timing = false;
  dgb_pass_timers timers{};
  struct Pending {
    int cat;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  int64_t launches = 0;
  double stage_ms = 0.0;
  int64_t stage_launches = 0;
  std::vector<double> samples[6];  // per-launch device ms of each timer category since the last reset

  // TMA tensor maps of the coefficient buffers the DMMA kernel reads (p >= 3): host cache
  // keyed by the buffer address, the maps themselves in device memory (kMaxMaps slots)
  std::vector<const double*> tm_keys;
  DevBuf<CUtensorMap> tm_dev;

  // fused stage + limiter (p = 1, whole mesh; kernels_p1.cu k_stage_limit)
  int fuse_limit = -1;  // 1 fused stage + limiter launch, 0 two kernels, -1 by mesh size (kFuseMaxN)
  std::vector<int2> fz_range_h;  // per 32-element tile: first and last chunk holding a neighbour
  int fz_maxreach = 0;           // max over tiles of (last tile waited for - tile)
  DevBuf<unsigned long long> fz_count;
  DevBuf<int2> fz_range;
  int fz_grid = 0, fz_lag = 0;
  unsigned long long fz_epoch = 0;  // fused launches of the current run

  dgbk::Tab<1> tab1;
  dgbk::Tab<2> tab2;
  dgbk::Tab<3> tab3;
  dgbk::Tab<4> tab4;
  dgbk::Tab<5> tab5;
  dgbk::LimTab lim{};

  size_t coeff_count() const { return static_cast<size_t>(4) * np * ld; }
  // rotating buffers (state0/1, stage0/1): the coefficients, then at the degrees with
  // trace-buffer stage instances the edge traces [4][3K][ld] of those coefficients (trace mode,
  // DESIGN.md section 3.1); one allocation, so a peer's mapping of a buffer covers both
  size_t rot_count() const { return coeff_count() + static_cast<size_t>(4) * k3 * ld; }
};

namespace {

// Contents of each degree's constant bank, per (device, degree): a context uploads its
// tables only when the bank holds different bytes (contexts built from the same tables
// share the bank, so partitions driven from several host threads never rewrite it under
// each other's kernels).  When the content does change, the device is drained first so no
// kernel of another context still reads the old tables.  Guarded by g_bank_mutex: contexts
// may run from several host threads (dist.run_group).
std::mutex g_bank_mutex;
std::map<std::pair<int, int>, std::vector<char>> g_bank_content;

template <class T>
bool bank_claim(int device, int key, const T& tab) {  // caller holds g_bank_mutex
  std::vector<char>& cur = g_bank_content[std::make_pair(device, key)];
  const char* b = reinterpret_cast<const char*>(&tab);
  if (cur.size() == sizeof(T) && std::memcmp(cur.data(), b, sizeof(T)) == 0) return false;
  if (!cur.empty()) CU(cudaDeviceSynchronize());
  cur.assign(b, b + sizeof(T));
  return true;
}

void set_device(dgb_ctx* c) { CU(cudaSetDevice(c->device)); }

cudaEvent_t take_event(dgb_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CU(cudaEventCreate(&e));
  return e;
}

// category: 0 volume, 1 surface, 2 rhs, 3 limiter, 4 other, 5 stage
struct Timed {
  dgb_ctx* c;
  int cat;
  cudaEvent_t a = nullptr, b = nullptr;
  Timed(dgb_ctx* ctx, int category) : c(ctx), cat(category) {
    if (c->timing) {
      a = take_event(c);
      b = take_event(c);
      CU(cudaEventRecord(a, c->stream));
    }
  }
  ~Timed() {
    if (c->timing && a) {
      cudaEventRecord(b, c->stream);
      c->pending.push_back({cat, a, b});
    }
  }
};

void settle_timers(dgb_ctx* c) {
  for (auto& pd : c->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pd.a, pd.b) == cudaSuccess) {
      const double s = ms * 1e-3;
      if (pd.cat >= 0 && pd.cat < 6) c->samples[pd.cat].push_back(ms);
      switch (pd.cat) {
        case 0: c->timers.volume += s; break;
        case 1: c->timers.surface += s; break;
        case 2: c->timers.rhs += s; break;
        case 3: c->timers.limiter += s; break;
        case 4: c->timers.other += s; break;
        default:
          c->timers.stage += s;
          c->stage_ms += ms;
          break;
      }
    }
    c->event_pool.push_back(pd.a);
    c->event_pool.push_back(pd.b);
  }
  c->pending.clear();
}

void sync(dgb_ctx* c) {
  CU(cudaStreamSynchronize(c->stream));
  settle_timers(c);
}

template <int P>
void upload_tab(dgb_ctx* c, dgbk::Tab<P>& tab) {
  if (bank_claim(c->device, P, tab)) {
    CU(dgbk::Launch<P>::upload(tab, c->stream));
    CU(cudaStreamSynchronize(c->stream));  // the bank is in place before any other stream launches
  }
  if (!c->d_mma.p) {  // DMMA fragment-ordered copy (global memory, staged to smem per block)
    const int n = dgbk::Launch<P>::mma_table(tab, nullptr);
    if (n > 0) {
      std::vector<double> h(n);
      dgbk::Launch<P>::mma_table(tab, h.data());
      c->d_mma.upload(h.data(), n, c->stream);
      CU(cudaStreamSynchronize(c->stream));
    } else {
      c->d_mma.alloc(1);
    }
    c->geo.mma_tab = c->d_mma.p;
  }
}

void ensure_tables(dgb_ctx* c) {
  std::lock_guard<std::mutex> lock(g_bank_mutex);
  switch (c->p) {
    case 1:
      upload_tab<1>(c, c->tab1);
      if (bank_claim(c->device, 100, c->lim)) {
        CU(dgbk::upload_limtab(c->lim, c->stream));
        CU(cudaStreamSynchronize(c->stream));
      }
      break;
    case 2: upload_tab<2>(c, c->tab2); break;
    case 3: upload_tab<3>(c, c->tab3); break;
    case 4: upload_tab<4>(c, c->tab4); break;
    default: upload_tab<5>(c, c->tab5); break;
  }
}

template <int P>
void fill_tab(dgbk::Tab<P>& T, const dgb_tables_view* t) {
  constexpr int NP = dgbk::Dim<P>::NP, NQ = dgbk::Dim<P>::NQ, K = dgbk::Dim<P>::K;
  for (int k = 0; k < NQ; ++k)
    for (int j = 0; j < NP; ++j) {
      T.phi[k][j] = t->phi_interior[k * NP + j];
      T.drw[k][j] = t->w_interior[k] * t->dphi_dr_interior[k * NP + j];
      T.dsw[k][j] = t->w_interior[k] * t->dphi_ds_interior[k * NP + j];
    }
  for (int q = 0; q < 3; ++q)
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < NP; ++j) T.phe[q][k][j] = t->phi_edge[(q * K + k) * NP + j];
  for (int k = 0; k < K; ++k) T.we[k] = t->w_edge[k];
  for (int q = 0; q < 3; ++q)
    for (int j = 0; j < NP; ++j) T.phm[q][j] = t->phi_edge_mid[q * NP + j];
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

constexpr int kMaxMaps = 16;

// The device address of the tensor map of coefficient buffer `buf` ([4][np][ld] doubles, box
// {8 elements, np modes, 4 variables}), encoded and uploaded on first use.  Columns past ld (a
// tail tile) are zero-filled by the TMA unit.
const void* tensor_map_of(dgb_ctx* c, const double* buf) {
  if (!buf) return nullptr;
  for (size_t i = 0; i < c->tm_keys.size(); ++i)
    if (c->tm_keys[i] == buf) return c->tm_dev.p + i;
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) throw Fail{DGB_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable"};
  if (!c->tm_dev.p) c->tm_dev.alloc(kMaxMaps);
  if (c->tm_keys.size() == static_cast<size_t>(kMaxMaps)) {  // buffers were reallocated: start over
    CU(cudaStreamSynchronize(c->stream));
    c->tm_keys.clear();
  }
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(c->ld), static_cast<cuuint64_t>(c->np), 4};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(c->ld) * 8, static_cast<cuuint64_t>(c->np) * c->ld * 8};
  const cuuint32_t box[3] = {8, static_cast<cuuint32_t>(c->np), 4};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(buf), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Fail{DGB_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")"};
  const size_t i = c->tm_keys.size();
  c->tm_keys.push_back(buf);
  CU(cudaMemcpyAsync(c->tm_dev.p + i, &m, sizeof(m), cudaMemcpyHostToDevice, c->stream));
  return c->tm_dev.p + i;
}

cudaError_t launch_element(dgb_ctx* c, int mode, const StageArgs& a_in) {
  StageArgs a = a_in;
  // the DMMA kernel's own-tile TMA boxes start at column e0 + 8 k: 16-byte aligned for an even e0
  // (run_steps splits partitions at an even column; every other launch starts at 0)
  if (c->p >= 3 && (a.e0 & 1)) throw Fail{DGB_ERR_ARG, "DMMA stage launch at an odd first column"};
  a.tm_in = c->p >= 3 ? tensor_map_of(c, a.in) : nullptr;
  switch (c->p) {
    case 1: return dgbk::Launch<1>::element(mode, 0, c->geo, a, c->stream);
    case 2: return dgbk::Launch<2>::element(mode, 0, c->geo, a, c->stream);
    case 3: return dgbk::Launch<3>::element(mode, 0, c->geo, a, c->stream);
    case 4: return dgbk::Launch<4>::element(mode, 0, c->geo, a, c->stream);
    default: return dgbk::Launch<5>::element(mode, 0, c->geo, a, c->stream);
  }
}

cudaError_t launch_dt(dgb_ctx* c, const double* coeffs, int slot, unsigned long long seq) {
  switch (c->p) {
    case 1: return dgbk::Launch<1>::dt(0, c->geo, coeffs, c->d_sc, slot, seq, c->stream);
    case 2: return dgbk::Launch<2>::dt(0, c->geo, coeffs, c->d_sc, slot, seq, c->stream);
    case 3: return dgbk::Launch<3>::dt(0, c->geo, coeffs, c->d_sc, slot, seq, c->stream);
    case 4: return dgbk::Launch<4>::dt(0, c->geo, coeffs, c->d_sc, slot, seq, c->stream);
    default: return dgbk::Launch<5>::dt(0, c->geo, coeffs, c->d_sc, slot, seq, c->stream);
  }
}

double* slot_ptr(dgb_ctx* c, int slot) {
  switch (slot) {
    case DGB_SLOT_STATE: return c->state[c->cur].p;
    case DGB_SLOT_INPUT:
      if (!c->input.p) {
        c->input.alloc_zero(c->coeff_count(), c->stream);
        CU(cudaMemsetAsync(c->input.p, 0, c->coeff_count() * 8, c->stream));
      }
      return c->input.p;
    case DGB_SLOT_VOLUME:
      if (!c->volume.p) {
        c->volume.alloc_zero(c->coeff_count(), c->stream);
        CU(cudaMemsetAsync(c->volume.p, 0, c->coeff_count() * 8, c->stream));
      }
      return c->volume.p;
    case DGB_SLOT_DERIV:
      if (!c->deriv.p) {
        c->deriv.alloc_zero(c->coeff_count(), c->stream);
        CU(cudaMemsetAsync(c->deriv.p, 0, c->coeff_count() * 8, c->stream));
      }
      return c->deriv.p;
    default:
      throw Fail{DGB_ERR_ARG, "unknown coefficient slot " + std::to_string(slot)};
  }
}

void reset_scalars(dgb_ctx* c, double t0) {
  Scalars& s = *c->h_sc;
  s.err_key = dgbk::kNoError;
  s.halt = 0;
  s.halt_step = 0;
  s.t[0] = t0;
  s.t[1] = t0;
  s.dtmin[0] = s.dtmin[1] = 0x7ff0000000000000ull;
  s.resid[0] = s.resid[1] = 0ull;
  s.dt_used[0] = s.dt_used[1] = 0.0;
  CU(cudaMemcpyAsync(c->d_sc, c->h_sc, sizeof(Scalars), cudaMemcpyHostToDevice, c->stream));
}

void read_scalars(dgb_ctx* c) {
  CU(cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
}

// Device -> host: the owned columns, [rows][N] in compact order.
void download_dev(dgb_ctx* c, const double* dev, int rows, double* host) {
  const size_t n = static_cast<size_t>(rows) * c->N;
  if (c->staging.n < n) c->staging.alloc(n);
  k_permute_out<<<small_grid(static_cast<long long>(rows) * c->ld), 256, 0, c->stream>>>(
      c->staging.p, dev, c->d_cmp.p, c->N, c->N, c->ld, rows);
  CU(cudaGetLastError());
  ++c->launches;
  CU(cudaMemcpyAsync(host, c->staging.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
  sync(c);
}

// Host -> device: owned + halo columns from [rows][N + n_halo] in compact order.
void upload_dev(dgb_ctx* c, double* dev, int rows, const double* host) {
  const int nl = c->N + c->n_halo;
  const size_t n = static_cast<size_t>(rows) * nl;
  if (c->staging.n < n) c->staging.alloc(n);
  CU(cudaMemcpyAsync(c->staging.p, host, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
  k_permute_in<<<small_grid(static_cast<long long>(rows) * c->ld), 256, 0, c->stream>>>(
      dev, c->staging.p, c->d_cmp.p, nl, nl, c->ld, rows);
  CU(cudaGetLastError());
  ++c->launches;
}

// Host recomputation of the failing state for the SolverAbort message
// (solver.cpp:57-62); only runs after a device error.  Ghost states follow
// euler.hpp:118-140.
void ghost_host(const dgb_ctx* c, const double* ul, int code, int e, int k, double t, double* ur) {
  auto reflect = [&](double nx, double ny) {
    const double mn = 2.0 * (ul[1] * nx + ul[2] * ny);
    ur[0] = ul[0];
    ur[1] = ul[1] - mn * nx;
    ur[2] = ul[2] - mn * ny;
    ur[3] = ul[3];
  };
  const size_t pk = static_cast<size_t>(e) * c->K + k;
  switch (code) {
    case -1: reflect(c->enx[e], c->eny[e]); break;
    case -2: reflect(c->bc_wn[2 * pk], c->bc_wn[2 * pk + 1]); break;
    case -3:
      std::memcpy(ur, c->bc_dir.empty() ? c->bc.inflow_state : &c->bc_dir[4 * pk], 4 * sizeof(double));
      break;
    case -5: {
      const double xi = c->t_xi[k];
      const double wa = 0.5 * (1.0 - xi), wb = 0.5 * (1.0 + xi);
      const double x = wa * c->vx[c->ev0[e]] + wb * c->vx[c->ev1[e]];
      const double y = wa * c->vy[c->ev0[e]] + wb * c->vy[c->ev1[e]];
      const double front = c->geo.sh_x0 + (y * c->geo.sh_cos + c->geo.sh_speed * t) / c->geo.sh_sin;
      std::memcpy(ur, x < front ? c->bc.shock_post : c->bc.shock_pre, 4 * sizeof(double));
      break;
    }
    default: std::memcpy(ur, ul, 4 * sizeof(double)); break;
  }
}

std::string failure_message(dgb_ctx* c, unsigned long long key, const double* dev_in, double t_stage) {
  const int pass = static_cast<int>((key >> 35) & 7);
  const long long id = static_cast<long long>((key >> 5) & 0x3fffffff);
  const int point = static_cast<int>(key & 31);
  if (pass == 7)
    return (key & 31) == 1 ? "fused stage + limiter launch: a tile wait timed out"
                            : "halo exchange timed out (a peer rank stopped signalling)";
  std::vector<double> h(static_cast<size_t>(4) * c->np * c->N);
  download_dev(c, dev_in, 4 * c->np, h.data());
  // the download holds the owned elements only (compact index = reference id - lo)
  bool have = true;
  auto coef = [&](int m, int j, int i) {
    if (i < c->lo || i >= c->hi) {
      have = false;
      return 0.0;
    }
    return h[(static_cast<size_t>(m) * c->np + j) * c->N + (i - c->lo)];
  };
  double u[4] = {0, 0, 0, 0};
  const char* where = "eval_volume";
  if (pass == dgbk::kPassVolume) {
    for (int m = 0; m < 4; ++m) {
      double s = 0.0;
      for (int j = 0; j < c->np; ++j) s += coef(m, j, static_cast<int>(id)) * c->t_phi[point * c->np + j];
      u[m] = s;
    }
  } else if (pass == dgbk::kPassDt) {
    where = "stable_dt";
    for (int m = 0; m < 4; ++m) {
      double s = 0.0;
      for (int j = 0; j < c->np; ++j) s += coef(m, j, static_cast<int>(id)) * c->t_phm[(point - 1) * c->np + j];
      u[m] = s;
    }
  } else {
    where = "eval_surface";
    const int e = static_cast<int>(id);
    const int L = c->eleft[e], R = c->eright[e];
    double ul[4], ur[4];
    for (int m = 0; m < 4; ++m) {
      double s = 0.0;
      for (int j = 0; j < c->np; ++j) s += coef(m, j, L) * c->t_phe[((c->esl[e] - 1) * c->K + point) * c->np + j];
      ul[m] = s;
    }
    if (R >= 0) {
      for (int m = 0; m < 4; ++m) {
        double s = 0.0;
        for (int j = 0; j < c->np; ++j)
          s += coef(m, j, R) * c->t_phe[((c->esr[e] - 1) * c->K + (c->K - 1 - point)) * c->np + j];
        ur[m] = s;
      }
    } else {
      ghost_host(c, ul, R, e, point, t_stage, ur);
    }
    const bool okl = ul[0] > 0.0 && pressure_ref(ul, c->gamma) > 0.0;
    std::memcpy(u, okl ? ur : ul, sizeof u);
  }
  if (!have) u[0] = u[3] = std::nan("");  // failing element lives on another rank
  const double pr = pressure_ref(u, c->gamma);
  std::snprintf(c->last_abort.where, sizeof c->last_abort.where, "%s", where);
  c->last_abort.id = id;
  c->last_abort.point = point;
  c->last_abort.rho = u[0];
  c->last_abort.p = pr;
  return std::string(where) + ": inadmissible state at id " + std::to_string(id) + ", point " +
         std::to_string(point) + " (rho=" + std::to_string(u[0]) + ", p=" + std::to_string(pr) + ")";
}

void check_bc(dgb_ctx* c) {
  if (!c->bc_error.empty()) throw Fail{DGB_ERR_BC, "eval_surface: " + c->bc_error};
}

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Fail& e) {
    dgb::set_message(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    dgb::set_message("out of host memory");
    return DGB_ERR_ARG;
  } catch (const std::exception& e) {
    dgb::set_message(e.what());
    return DGB_ERR_ARG;
  }
}

// Pass-level launch with an immediate error check.
void run_pass(dgb_ctx* c, int mode, const double* in, double* out, double t, int cat) {
  ensure_tables(c);
  reset_scalars(c, t);
  StageArgs a{};
  a.in = in;
  a.u = in;
  a.out = out;
  a.kacc = nullptr;
  a.t_host = t;
  a.use_t_host = 1;
  a.seq = 1;
  a.seq_next = 2;
  a.sc = c->d_sc;
  a.e0 = 0;
  a.e1 = c->N;
  {
    Timed tm(c, cat);
    CU(launch_element(c, mode, a));
    ++c->launches;
  }
  read_scalars(c);
  if (c->h_sc->err_key != dgbk::kNoError) throw Fail{DGB_ERR_INADMISSIBLE, failure_message(c, c->h_sc->err_key, in, t)};
}

// ------------------------------------------------------------------ the device step loop
struct RunSpec {
  int scheme;
  int dt_mode;  // 0 host dt, 1 stable dt
  double dt_host = 0.0, cfl = 0.3;
  bool limiting = false;
  int64_t max_steps = 1;
  bool clip = false, stop_t = false, stop_steady = false;
  double t_end = 0.0, tol = 0.0;
  double* hist = nullptr;  // host history
  int64_t hist_cap = 0;
};

struct RunOut {
  int64_t steps = 0;
  double residual = 0.0;
  bool halted = false;
};

int trace_points(int p) {
  switch (p) {
    case 1: return dgbk::Launch<1>::trace_points();
    case 2: return dgbk::Launch<2>::trace_points();
    case 3: return dgbk::Launch<3>::trace_points();
    case 4: return dgbk::Launch<4>::trace_points();
    case 5: return dgbk::Launch<5>::trace_points();
    default: return 0;
  }
}

bool trace_wanted(const dgb_ctx* c) {
  switch (c->p) {
    case 1: return dgbk::Launch<1>::trace_wanted(c->N, c->geo);
    case 2: return dgbk::Launch<2>::trace_wanted(c->N, c->geo);
    case 3: return dgbk::Launch<3>::trace_wanted(c->N, c->geo);
    case 4: return dgbk::Launch<4>::trace_wanted(c->N, c->geo);
    default: return dgbk::Launch<5>::trace_wanted(c->N, c->geo);
  }
}

int buf_id(const dgb_ctx* c, const double* p) {
  if (p == c->state[0].p) return 0;
  if (p == c->state[1].p) return 1;
  if (p == c->stage[0].p) return 2;
  if (p == c->stage[1].p) return 3;
  return -1;
}

bool exchanging(const dgb_ctx* c) { return c->partitioned && c->world > 1; }

unsigned all_peers(const dgb_ctx* c) { return ((1u << c->world) - 1u) & ~(1u << c->rank); }

// Push the send elements' columns of `p` (one of the rotating buffers) to the peers.
void xch_push(dgb_ctx* c, const double* p, bool traces) {
  if (c->n_push == 0) return;
  const int buf = buf_id(c, p);
  if (buf < 0) throw Fail{DGB_ERR_ARG, "halo push from a buffer the peers do not map"};
  // the coefficient rows, then (trace mode) the element-major trace blocks that follow them
  const int rows = 4 * c->np, tblock = traces ? 4 * c->k3 : 0;
  const long long total = static_cast<long long>(c->n_push) * (rows + tblock);
  const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 8));
  k_push<<<grid, 256, 0, c->stream>>>(c->d_peers, buf, p, c->ld, c->d_push.p, c->n_push, rows, tblock);
  CU(cudaGetLastError());
  ++c->launches;
}

// Raise our flag at the peers in `mask` (publishing the step scalars to every
// rank when `publish`).  Returns the epoch of this signal.
unsigned long long xch_signal(dgb_ctx* c, unsigned mask, bool publish, int dt_idx, int res_idx) {
  const unsigned long long ep = ++c->epoch;
  const int slot = static_cast<int>(c->n_pub & 1);
  k_signal<<<1, 32, 0, c->stream>>>(c->d_peers, mask, c->rank, ep, c->d_sc, publish ? 1 : 0, slot, dt_idx, res_idx);
  CU(cudaGetLastError());
  ++c->launches;
  if (publish) {
    c->pub_epoch = ep;
    ++c->n_pub;
  }
  return ep;
}

void xch_wait(dgb_ctx* c, unsigned mask, unsigned long long ep, bool merge, int dt_idx, int res_idx) {
  const int slot = static_cast<int>((c->n_pub - 1) & 1);
  k_wait<<<1, 32, 0, c->stream>>>(c->d_xch, c->d_xch + dgbk::kMaxRanks, mask, ep, c->d_sc, merge ? 1 : 0, slot, dt_idx,
                                  res_idx, static_cast<unsigned long long>(c->timeout_s * 1e9));
  CU(cudaGetLastError());
  ++c->launches;
}

RunOut run_steps(dgb_ctx* c, const RunSpec& r) {
  std::vector<StageSpec> st;
  if (!scheme_stages(r.scheme, st)) throw Fail{DGB_ERR_ARG, "rk_order must be 2 or 4"};
  if (r.limiting && c->p != 1) throw Fail{DGB_ERR_ARG, "slope limiting is only supported for p = 1"};
  if (!c->finalized) throw Fail{DGB_ERR_ARG, "partitioned context used before dgb_part_finalize"};
  check_bc(c);
  ensure_tables(c);
  const int S = static_cast<int>(st.size());
  if (!c->stage[0].p) c->stage[0].alloc_zero(c->rot_count(), c->stream);
  if (!c->stage[1].p) c->stage[1].alloc_zero(c->rot_count(), c->stream);
  if (r.scheme == DGB_RK4_CLASSIC && !c->kacc.p) c->kacc.alloc_zero(c->coeff_count(), c->stream);
  if (!c->state[1 - c->cur].p) c->state[1 - c->cur].alloc_zero(c->rot_count(), c->stream);
  double* d_hist = nullptr;
  if (r.hist && r.hist_cap > 0) {
    if (c->hist.n < static_cast<size_t>(r.hist_cap)) c->hist.alloc(r.hist_cap);
    d_hist = c->hist.p;
  }
  const bool X = exchanging(c);
  const unsigned ALL = X ? all_peers(c) : 0u;
  // the fused stage + limiter launch (whole-mesh contexts; a partition keeps the two-kernel
  // path, whose halo rounds it needs)
  const bool fused = r.limiting && !c->partitioned && c->p == 1 &&
                     (c->fuse_limit < 0 ? c->N <= kFuseMaxN : c->fuse_limit != 0);
  if (fused) {
    const int nt = static_cast<int>(c->fz_range_h.size());
    const int nch = (nt + dgbk::kFuseChunk - 1) / dgbk::kFuseChunk;
    if (!c->fz_range.p) {
      c->fz_range.upload(c->fz_range_h.data(), nt, c->stream);
      c->fz_count.alloc(nch);
      // one warp per tile, every warp resident (cooperative launch): no more warps than tiles
      const int warps_per_block = dgbk::kBlock / 32;
      c->fz_grid = std::min(dgbk::stage_limit_grid(), (nt + warps_per_block - 1) / warps_per_block);
      if (const char* g = std::getenv("DGB_FUSE_GRID")) c->fz_grid = std::max(1, std::min(c->fz_grid, std::atoi(g)));
      c->fz_lag = c->fz_maxreach + c->fz_grid * warps_per_block;
    }
    // chunk counters count this run's publications: zero them, restart the epochs
    CU(cudaMemsetAsync(c->fz_count.p, 0, nch * sizeof(unsigned long long), c->stream));
    c->fz_epoch = 0;
  }
  // two-kernel limiting on a whole mesh: the stage kernel also writes the new cell means as one
  // 32-byte record per element, the limiter gathers its neighbours' means from it (one sector
  // per neighbour instead of four); a partition keeps reading the coefficient columns (its halo
  // columns arrive through the coefficient push)
  double* means_buf = nullptr;
  if (r.limiting && !fused && !c->partitioned) {
    if (c->means.n < static_cast<size_t>(4) * c->ld) c->means.alloc(static_cast<size_t>(4) * c->ld);
    means_buf = c->means.p;
  }
  // interior elements [0, n_int) never read a halo column; boundary elements
  // [n_int, N) do, and only they feed the peers.  The split point is rounded down to an even
  // column (an interior element computed after the halo wait is harmless): the DMMA kernel's
  // TMA boxes start at e0 + 8 k and must be 16-byte aligned.
  const int n_int = X ? (c->n_int & ~1) : c->N;
  // trace mode (p >= 2, no limiter, p = 2 above the latency-form size): each stage writes the edge traces of its output, the
  // next stage reads its own and its neighbours' traces instead of interpolating them (results
  // bit-identical).  A partition pushes the send elements' trace rows
  // with their coefficient rows, so the halo columns carry traces too.
  const bool use_tr = c->trace_mode != 0 && c->k3 > 0 && !r.limiting && !fused && trace_wanted(c);
  auto trace_of = [&](const double* p) -> double* {
    if (buf_id(c, p) < 0) throw Fail{DGB_ERR_ARG, "trace of a buffer outside the rotation"};
    return const_cast<double*>(p) + c->coeff_count();
  };

  const int cur0 = c->cur;
  reset_scalars(c, c->t);
  if (r.dt_mode == 1) {
    Timed tm(c, 4);
    CU(launch_dt(c, c->state[cur0].p, 0, 0));
    ++c->launches;
  }
  // the first step's dt bound is a global min over the ranks
  if (X) xch_signal(c, ALL, true, 0, 0);

  RunOut out;
  int64_t launched = 0;
  bool stop = false;
  while (!stop && launched < r.max_steps) {
    const int64_t batch = std::min<int64_t>(r.max_steps - launched,
                                             (r.stop_t || r.stop_steady) ? kBatch : r.max_steps);
    for (int64_t b = 0; b < batch; ++b) {
      const int64_t s = launched + b;
      const int par = static_cast<int>(s & 1);
      // max|u_new - u| (max_abs_diff, solver.cpp:536) is observable only through the stop rules, the
      // on_step history and the residual of the last step: a fixed-step run without a history
      // evaluates it on its last step alone (the limiter then skips reading u^n on every other step)
      const bool resid = r.stop_t || r.stop_steady || d_hist || s + 1 == r.max_steps;
      double* u = c->state[(cur0 + s) & 1].p;
      double* unext = c->state[(cur0 + s + 1) & 1].p;
      for (int k = 0; k < S; ++k) {
        const bool last = k == S - 1;
        if (c->n_dir_stages > 0)  // the boundary data at this stage's time (solver.cpp:198-211)
          c->geo.bstate = c->d_bstage.p + static_cast<size_t>(std::min(k, c->n_dir_stages - 1)) * 4 * c->n_bnd * c->K;
        StageArgs a{};
        a.in = k == 0 ? u : c->stage[(k - 1) & 1].p;
        a.u = u;
        a.out = last ? unext : c->stage[k & 1].p;
        a.kacc = c->kacc.p;
        a.means = means_buf;
        a.alpha = st[k].alpha;
        a.beta = st[k].beta;
        a.gcoef = st[k].gcoef;
        a.tcoef = st[k].tcoef;
        a.kmode = st[k].kmode;
        a.dt_mode = r.dt_mode;
        a.dt_host = r.dt_host;
        a.cfl = r.cfl;
        a.t_end = r.t_end;
        a.clip_t_end = r.clip;
        a.stop_at_t_end = r.stop_t;
        a.stop_steady = r.stop_steady;
        a.tol = r.tol;
        a.step = static_cast<int>(s);
        a.first = k == 0;
        a.last = last;
        a.want_lambda = last && !r.limiting && r.dt_mode == 1;
        a.want_resid = last && !r.limiting && resid;
        a.seq = static_cast<unsigned long long>(s) * 8 + k + 1;
        a.seq_next = static_cast<unsigned long long>(s + 1) * 8;
        a.sc = c->d_sc;
        a.hist = d_hist && s <= r.hist_cap ? d_hist : nullptr;
        if (use_tr) {  // the run's first stage interpolates; its last writes no traces
          a.tr_in = (s == 0 && k == 0) ? nullptr : trace_of(a.in);
          a.tr_out = (s + 1 == r.max_steps && last) ? nullptr : trace_of(a.out);
        }
        // step start: merge the previous step's scalars (dt bound, residual, error) from every rank
        if (X && k == 0) xch_wait(c, ALL, c->pub_epoch, true, par, par ^ 1);
        const unsigned long long prev = c->epoch;
        if (fused) {  // stage + limiter in one launch
          LimArgs la{};
          la.c = a.out;
          la.u = u;
          la.step = static_cast<int>(s);
          la.want_lambda = last && r.dt_mode == 1;
          la.want_resid = last && resid;
          la.seq = static_cast<unsigned long long>(s + 1) * 8;
          la.sc = c->d_sc;
          la.e0 = 0;
          la.e1 = c->N;
          a.e0 = 0;
          a.e1 = c->N;
          dgbk::FuseArgs f{c->fz_count.p, c->fz_range.p, static_cast<int>(c->fz_range_h.size()), c->fz_lag,
                           ++c->fz_epoch};
          Timed tm(c, 5);
          CU(dgbk::launch_stage_limit(c->fz_grid, c->geo, a, la, f, c->stream));
          ++c->launches;
          ++c->stage_launches;
          continue;
        }
        {
          Timed tm(c, 5);
          a.e0 = 0;
          a.e1 = n_int;
          CU(launch_element(c, dgbk::kModeStage, a));
          ++c->launches;
          ++c->stage_launches;
          if (X) {
            if (k > 0) xch_wait(c, c->nb_mask, prev, false, 0, 0);  // the peers' previous stage landed
            a.e0 = n_int;
            a.e1 = c->N;
            CU(launch_element(c, dgbk::kModeStage, a));
            ++c->launches;
            xch_push(c, a.out, a.tr_out != nullptr);
          }
        }
        if (X) {
          if (last && !r.limiting)
            xch_signal(c, ALL, true, par ^ 1, par);
          else
            xch_signal(c, c->send_mask, false, 0, 0);
        }
        if (r.limiting) {
          LimArgs la{};
          la.c = a.out;
          la.u = u;
          la.step = static_cast<int>(s);
          la.want_lambda = last && r.dt_mode == 1;
          la.want_resid = last && resid;
          la.means = means_buf;
          la.seq = static_cast<unsigned long long>(s + 1) * 8;
          la.sc = c->d_sc;
          const unsigned long long prev2 = c->epoch;
          Timed tm(c, 3);
          la.e0 = 0;
          la.e1 = n_int;
          CU(dgbk::launch_limit(0, c->geo, la, c->stream));
          ++c->launches;
          if (X) {
            // the limiter needs the neighbours' new means: wait for this stage's halo
            xch_wait(c, c->nb_mask, prev2, false, 0, 0);
            la.e0 = n_int;
            la.e1 = c->N;
            CU(dgbk::launch_limit(0, c->geo, la, c->stream));
            ++c->launches;
            xch_push(c, la.c, false);
            if (last)
              xch_signal(c, ALL, true, par ^ 1, par);
            else
              xch_signal(c, c->send_mask, false, 0, 0);
          }
        }
      }
    }
    launched += batch;
    if (X) xch_wait(c, ALL, c->pub_epoch, true, static_cast<int>(launched & 1), static_cast<int>((launched - 1) & 1));
    read_scalars(c);
    const Scalars& h = *c->h_sc;
    if (h.err_key != dgbk::kNoError) {
      const unsigned long long seq = h.err_key >> 38;
      if (((h.err_key >> 35) & 7) == 7 && seq == 0) throw Fail{DGB_ERR_CUDA, failure_message(c, h.err_key, nullptr, 0.0)};
      const int64_t s_fail = static_cast<int64_t>(seq >> 3);
      const int kst = static_cast<int>(seq & 7);
      const double* in = (kst <= 1) ? c->state[(cur0 + s_fail) & 1].p : c->stage[(kst - 2) & 1].p;
      // the failed step leaves the state untouched (rk_step_ws throws before the swap)
      c->cur = static_cast<int>((cur0 + s_fail) & 1);
      c->t = h.t[s_fail & 1];
      c->step_count += s_fail;
      if (d_hist && s_fail > 0) {
        const int64_t n = std::min<int64_t>(s_fail, r.hist_cap);
        CU(cudaMemcpyAsync(r.hist, d_hist, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
      }
      const double tst = h.t[s_fail & 1];
      throw Fail{DGB_ERR_INADMISSIBLE, failure_message(c, h.err_key, in, tst)};
    }
    if (h.halt) {
      stop = true;
      out.halted = true;
      out.steps = h.halt_step;
    }
  }
  if (!out.halted) out.steps = launched;
  const Scalars& h = *c->h_sc;
  if (out.steps > 0) out.residual = __builtin_bit_cast(double, h.resid[(out.steps - 1) & 1]);
  if (d_hist && out.steps > 0) {
    const int64_t n = std::min<int64_t>(out.steps, r.hist_cap);
    // the last step's residual is only in the scalars (hist[s-1] is written by step s)
    if (n > 1) CU(cudaMemcpyAsync(r.hist, d_hist, sizeof(double) * (n - 1), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (out.steps <= r.hist_cap) r.hist[out.steps - 1] = out.residual;
  }
  c->cur = static_cast<int>((cur0 + out.steps) & 1);
  c->t = h.t[out.steps & 1];
  c->step_count += out.steps;
  return out;
}

// Partition plan (host only): owned range, per owned element its neighbour ids /
// side labels / left bits / class, the interior-boundary split and the halo.
struct PartPlan {
  int lo = 0, hi = 0;
  std::vector<int> cls, nb_side, nb_id, left_bits;  // per owned element (index id - lo)
  std::vector<int> interior, boundary, halo;        // reference ids (ascending)
  unsigned nb_mask = 0;                             // owners of halo elements
};

int owner_of(int id, int n, int world) {
  int r = static_cast<int>((static_cast<long long>(id) * world) / n);
  r = std::min(world - 1, std::max(0, r));
  while (r > 0 && id < static_cast<int>(static_cast<long long>(n) * r / world)) --r;
  while (r < world - 1 && id >= static_cast<int>(static_cast<long long>(n) * (r + 1) / world)) ++r;
  return r;
}

void make_plan(const dgb_mesh_view* m, int rank, int world, PartPlan& P) {
  const int NG = m->n_elements;
  P.lo = static_cast<int>(static_cast<long long>(NG) * rank / world);
  P.hi = static_cast<int>(static_cast<long long>(NG) * (rank + 1) / world);
  const int lo = P.lo, hi = P.hi, N = hi - lo;
  auto owned = [&](int i) { return i >= lo && i < hi; };
  P.cls.assign(N, 0);
  P.nb_side.assign(3 * static_cast<size_t>(N), 0);
  P.nb_id.assign(3 * static_cast<size_t>(N), 0);
  P.left_bits.assign(N, 0);
  for (int l = 0; l < N; ++l) {
    const int i = lo + l;
    int key = 0;
    bool cut = false;
    for (int q = 0; q < 3; ++q) {
      const int e = m->elem_edge[3 * i + q];
      if (e < 0 || e >= m->n_edges) throw Fail{DGB_ERR_MESH, "element edge id out of range"};
      const bool left = m->edge_left[e] == i;
      int sd = 0, nb;
      if (m->edge_right[e] < 0) {
        nb = m->edge_right[e];
        if (!left) throw Fail{DGB_ERR_MESH, "boundary edge whose left element is not its owner"};
      } else {
        nb = left ? m->edge_right[e] : m->edge_left[e];
        sd = left ? m->edge_side_right[e] : m->edge_side_left[e];
        if (!owned(nb)) {
          cut = true;
          P.halo.push_back(nb);
        }
      }
      P.nb_side[3 * l + q] = sd;
      P.nb_id[3 * l + q] = nb;
      if (left) P.left_bits[l] |= 1 << q;
      key |= sd << (2 * q);
    }
    P.cls[l] = key;
    (cut ? P.boundary : P.interior).push_back(i);
  }
  std::sort(P.halo.begin(), P.halo.end());
  P.halo.erase(std::unique(P.halo.begin(), P.halo.end()), P.halo.end());
  for (int h : P.halo) P.nb_mask |= 1u << owner_of(h, NG, world);
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" {

int dgb_create(const dgb_mesh_view* m, const dgb_tables_view* t, const dgb_bc_view* bc, double gamma, int device,
               dgb_ctx** out) {
  return dgb_part_create(m, t, bc, gamma, device, 0, 1, out);
}

int dgb_part_create(const dgb_mesh_view* m, const dgb_tables_view* t, const dgb_bc_view* bc, double gamma, int device,
                    int rank, int world, dgb_ctx** out) {
  return guarded([&] {
    if (!m || !t || !out) throw Fail{DGB_ERR_ARG, "null argument"};
    if (t->p < 1 || t->p > 5) throw Fail{DGB_ERR_ARG, "polynomial degree must be in [1,5]"};
    if (world < 1 || world > dgbk::kMaxRanks || rank < 0 || rank >= world)
      throw Fail{DGB_ERR_ARG, "rank/world out of range (1 <= world <= 8)"};
    const int np = (t->p + 1) * (t->p + 2) / 2;
    const int nq_expect[5] = {3, 6, 12, 16, 25};
    if (t->n_p != np || t->n_quad != nq_expect[t->p - 1] || t->n_edge_pts != t->p + 1)
      throw Fail{DGB_ERR_ARG, "tables do not match the expected sizes for p = " + std::to_string(t->p)};
    if (m->n_elements <= 0) throw Fail{DGB_ERR_ARG, "empty mesh"};
    const int NG = m->n_elements;
    if (NG < world) throw Fail{DGB_ERR_ARG, "fewer elements than ranks"};
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Fail{DGB_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)"};
    if (device < 0 || device >= ndev) throw Fail{DGB_ERR_ARG, "bad device ordinal"};
    std::unique_ptr<dgb_ctx> c(new dgb_ctx);
    c->device = device;
    set_device(c.get());
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    c->p = t->p;
    c->np = np;
    c->nq = t->n_quad;
    c->K = t->n_edge_pts;
    c->gamma = gamma;
    c->rank = rank;
    c->world = world;
    c->partitioned = world > 1;
    c->finalized = world == 1;
    c->n_global = NG;
    // contiguous ranges of reference ids ("identical partition indexing")
    const int lo = static_cast<int>(static_cast<long long>(NG) * rank / world);
    const int hi = static_cast<int>(static_cast<long long>(NG) * (rank + 1) / world);
    c->lo = lo;
    c->hi = hi;
    const int N = hi - lo;  // owned
    c->N = N;
    c->n_edges = m->n_edges;
    c->n_bnd = m->n_boundary_edges;

    c->vx.assign(m->vx, m->vx + m->n_vertices);
    c->vy.assign(m->vy, m->vy + m->n_vertices);
    c->det.assign(m->det_jac, m->det_jac + NG);
    c->elem_v.assign(m->elem_v, m->elem_v + 3 * static_cast<size_t>(NG));
    c->elem_edge.assign(m->elem_edge, m->elem_edge + 3 * static_cast<size_t>(NG));
    c->eleft.assign(m->edge_left, m->edge_left + m->n_edges);
    c->eright.assign(m->edge_right, m->edge_right + m->n_edges);
    c->esl.assign(m->edge_side_left, m->edge_side_left + m->n_edges);
    c->esr.assign(m->edge_side_right, m->edge_side_right + m->n_edges);
    c->ev0.assign(m->edge_v0, m->edge_v0 + m->n_edges);
    c->ev1.assign(m->edge_v1, m->edge_v1 + m->n_edges);
    c->enx.assign(m->edge_nx, m->edge_nx + m->n_edges);
    c->eny.assign(m->edge_ny, m->edge_ny + m->n_edges);
    c->t_phi.assign(t->phi_interior, t->phi_interior + c->nq * np);
    c->t_phe.assign(t->phi_edge, t->phi_edge + 3 * c->K * np);
    c->t_phm.assign(t->phi_edge_mid, t->phi_edge_mid + 3 * np);
    c->t_xi.assign(t->xi_edge, t->xi_edge + c->K);
    c->t_w.assign(t->w_interior, t->w_interior + c->nq);

    PartPlan P;
    make_plan(m, rank, world, P);
    std::vector<int>& cls = P.cls;
    std::vector<int>& nb_side = P.nb_side;
    std::vector<int>& nb_id = P.nb_id;
    std::vector<int>& left_bits = P.left_bits;
    std::vector<int>& interior = P.interior;
    std::vector<int>& boundary = P.boundary;
    std::vector<int>& halo = P.halo;
    c->nb_mask = P.nb_mask;
    c->n_int = static_cast<int>(interior.size());
    c->n_halo = static_cast<int>(halo.size());
    c->halo_gid = halo;
    c->ld = (N + c->n_halo + 31) / 32 * 32;
    const int ld = c->ld;

    // --- device order: interior, then boundary elements, each windowed-class
    // sorted so every warp sees one neighbour-side class (warp-uniform trace switch);
    // halo columns follow the owned ones
    auto window_sort = [&](std::vector<int>& v) {
      for (size_t w0 = 0; w0 < v.size(); w0 += kWindow) {
        const size_t w1 = std::min(v.size(), w0 + kWindow);
        std::stable_sort(v.begin() + w0, v.begin() + w1, [&](int a, int b) { return cls[a - lo] < cls[b - lo]; });
      }
    };
    window_sort(interior);
    window_sort(boundary);
    c->ref_of.clear();
    c->ref_of.insert(c->ref_of.end(), interior.begin(), interior.end());
    c->ref_of.insert(c->ref_of.end(), boundary.begin(), boundary.end());
    c->ref_of.insert(c->ref_of.end(), halo.begin(), halo.end());
    c->col_of.assign(NG, -1);
    for (size_t d = 0; d < c->ref_of.size(); ++d) c->col_of[c->ref_of[d]] = static_cast<int>(d);

    std::vector<double> tau(4 * static_cast<size_t>(ld), 0.0), inv_det(ld, 1.0), inr(ld, 1.0);
    std::vector<int> nbr(3 * static_cast<size_t>(ld), -4), eid(3 * static_cast<size_t>(ld), 0), info(ld, 0),
        ref_id(ld, 0), cmp(ld, 0);
    for (int d = 0; d < N; ++d) {
      const int i = c->ref_of[d];
      const int l = i - lo;
      for (int k = 0; k < 4; ++k) tau[static_cast<size_t>(k) * ld + d] = m->tau[4 * static_cast<size_t>(i) + k];
      inv_det[d] = 1.0 / m->det_jac[i];
      inr[d] = m->inradius[i];
      int bits = 0;
      for (int q = 0; q < 3; ++q) {
        const int nb = nb_id[3 * l + q];
        nbr[static_cast<size_t>(q) * ld + d] = nb >= 0 ? c->col_of[nb] : nb;
        eid[static_cast<size_t>(q) * ld + d] = m->elem_edge[3 * i + q];
        bits |= nb_side[3 * l + q] << (2 * q);
        if (left_bits[l] & (1 << q)) bits |= 1 << (6 + q);
      }
      info[d] = bits;
      ref_id[d] = i;
      cmp[d] = l;
    }
    for (int h = 0; h < c->n_halo; ++h) {
      ref_id[N + h] = halo[h];
      cmp[N + h] = N + h;
    }
    c->sends.assign(world, {});
    {  // neighbour chunk ranges for the fused stage + limiter launch (whole-mesh contexts)
      constexpr int TL = dgbk::kFuseTile, CH = dgbk::kFuseChunk;
      const int nt = (N + TL - 1) / TL;
      c->fz_range_h.assign(nt, make_int2(0, 0));
      c->fz_maxreach = 0;
      for (int t = 0; t < nt; ++t) {
        int lo_c = t / CH, hi_c = t / CH;
        for (int d = t * TL; d < std::min(N, (t + 1) * TL); ++d)
          for (int q = 0; q < 3; ++q) {
            const int nbd = nbr[static_cast<size_t>(q) * ld + d];
            if (nbd < 0 || nbd >= N) continue;
            lo_c = std::min(lo_c, nbd / TL / CH);
            hi_c = std::max(hi_c, nbd / TL / CH);
          }
        c->fz_range_h[t] = make_int2(lo_c, hi_c);
        // the last tile the limiter of t waits for
        c->fz_maxreach = std::max(c->fz_maxreach, std::min(nt - 1, (hi_c + 1) * CH - 1) - t);
      }
      const char* env = std::getenv("DGB_FUSED_LIMIT");
      c->fuse_limit = env ? (env[0] == '0' ? 0 : (env[0] == '1' ? 1 : -1)) : -1;
    }
    {
      const char* env = std::getenv("DGB_TRACE_BUF");
      c->trace_mode = env ? (env[0] == '0' ? 0 : 1) : DGB_TRACE_BUF_DEFAULT;
    }
    c->d_tau.upload(tau.data(), tau.size(), c->stream);
    c->d_inv_det.upload(inv_det.data(), ld, c->stream);
    c->d_inradius.upload(inr.data(), ld, c->stream);
    c->d_nbr.upload(nbr.data(), nbr.size(), c->stream);
    c->geo.has_bnd = 0;  // any owned element with a boundary code (padding columns hold -4 too)
    for (int q = 0; q < 3; ++q)
      for (int d = 0; d < N; ++d)
        if (nbr[static_cast<size_t>(q) * ld + d] < 0) c->geo.has_bnd = 1;
    c->d_eid.upload(eid.data(), eid.size(), c->stream);
    c->d_info.upload(info.data(), ld, c->stream);
    c->d_ref_id.upload(ref_id.data(), ld, c->stream);
    c->d_cmp.upload(cmp.data(), ld, c->stream);
    c->d_enx.upload(m->edge_nx, m->n_edges, c->stream);
    c->d_eny.upload(m->edge_ny, m->n_edges, c->stream);
    c->d_eh.upload(m->edge_half_length, m->n_edges, c->stream);

    // --- boundary data (closures evaluated by the caller at the Gauss points)
    const int K = c->K, nb = c->n_bnd;
    dgb_bc_view bcv{};
    if (bc) bcv = *bc;
    c->bc = bcv;
    std::vector<double> bx(2 * static_cast<size_t>(std::max(nb, 1)) * K, 0.0);
    for (int e = 0; e < nb; ++e) {
      const double ax = m->vx[m->edge_v0[e]], ay = m->vy[m->edge_v0[e]];
      const double bxx = m->vx[m->edge_v1[e]], byy = m->vy[m->edge_v1[e]];
      for (int k = 0; k < K; ++k) {
        const double xi = t->xi_edge[k];
        const double wa = 0.5 * (1.0 - xi), wb = 0.5 * (1.0 + xi);
        bx[2 * (static_cast<size_t>(e) * K + k)] = wa * ax + wb * bxx;
        bx[2 * (static_cast<size_t>(e) * K + k) + 1] = wa * ay + wb * byy;
      }
    }
    c->d_bx.upload(bx.data(), bx.size(), c->stream);
    bool has_curved = false, has_shock = false;
    for (int e = 0; e < nb; ++e) {
      const int code = m->edge_right[e];
      if (code == -2) has_curved = true;
      if (code == -5) has_shock = true;
      if (code < -5 && c->bc_error.empty()) c->bc_error = "unknown boundary code " + std::to_string(code);
    }
    if (bcv.dirichlet_state) {
      c->bc_dir.assign(bcv.dirichlet_state, bcv.dirichlet_state + 4 * static_cast<size_t>(nb) * K);
      c->d_bstate.upload(c->bc_dir.data(), c->bc_dir.size(), c->stream);
    } else {
      double z[4] = {0, 0, 0, 0};
      c->d_bstate.upload(z, 4, c->stream);
    }
    if (bcv.wall_normal) {
      c->bc_wn.assign(bcv.wall_normal, bcv.wall_normal + 2 * static_cast<size_t>(nb) * K);
      c->d_bwn.upload(c->bc_wn.data(), c->bc_wn.size(), c->stream);
    } else {
      double z[2] = {0, 0};
      c->d_bwn.upload(z, 2, c->stream);
      if (has_curved && c->bc_error.empty()) c->bc_error = "curved reflecting boundary needs a wall-normal function";
    }
    if (has_shock && !bcv.has_shock && c->bc_error.empty())
      c->bc_error = "moving-shock boundary needs shock parameters";

    Geo& g = c->geo;
    g.N = N;
    g.ld = ld;
    g.tau = c->d_tau.p;
    g.inv_det = c->d_inv_det.p;
    g.inradius = c->d_inradius.p;
    g.nbr = c->d_nbr.p;
    g.eid = c->d_eid.p;
    g.info = c->d_info.p;
    g.ref_id = c->d_ref_id.p;
    g.enx = c->d_enx.p;
    g.eny = c->d_eny.p;
    g.eh = c->d_eh.p;
    g.bstate = c->d_bstate.p;
    g.bwn = c->d_bwn.p;
    g.bx = c->d_bx.p;
    g.has_dir = bcv.dirichlet_state ? 1 : 0;
    g.has_wn = bcv.wall_normal ? 1 : 0;
    g.has_shock = bcv.has_shock;
    for (int k = 0; k < 4; ++k) {
      g.inflow[k] = bcv.inflow_state[k];
      g.sh_post[k] = bcv.shock_post[k];
      g.sh_pre[k] = bcv.shock_pre[k];
    }
    const double rad = bcv.shock_angle_deg * M_PI / 180.0;
    g.sh_x0 = bcv.shock_x0;
    g.sh_cos = std::cos(rad);
    g.sh_sin = std::sin(rad);
    g.sh_speed = bcv.shock_speed;
    g.gamma = gamma;

    // --- tables
    switch (c->p) {
      case 1: fill_tab<1>(c->tab1, t); break;
      case 2: fill_tab<2>(c->tab2, t); break;
      case 3: fill_tab<3>(c->tab3, t); break;
      case 4: fill_tab<4>(c->tab4, t); break;
      default: fill_tab<5>(c->tab5, t); break;
    }
    if (c->p == 1) {  // limiter evaluation points (solver.cpp:296-321)
      std::memset(&c->lim, 0, sizeof c->lim);  // the bank is compared bytewise (bank_claim)
      dgbk::LimTab& L = c->lim;
      int idx = 0;
      for (int k = 0; k < c->nq; ++k, ++idx) {
        L.phi1[idx] = t->phi_interior[k * np + 1];
        L.phi2[idx] = t->phi_interior[k * np + 2];
      }
      for (int q = 0; q < 3; ++q)
        for (int k = 0; k < K; ++k, ++idx) {
          L.phi1[idx] = t->phi_edge[(q * K + k) * np + 1];
          L.phi2[idx] = t->phi_edge[(q * K + k) * np + 2];
        }
      for (int q = 0; q < 3; ++q, ++idx) {
        L.phi1[idx] = t->phi_edge_mid[q * np + 1];
        L.phi2[idx] = t->phi_edge_mid[q * np + 2];
      }
      L.n_pts = idx;
      L.edge_begin = c->nq;
      L.n_edge = 3 * K;
      L.max_phi1 = 0.0;
      L.max_phi2 = 0.0;
      for (int k = 0; k < idx; ++k) {
        L.max_phi1 = std::max(L.max_phi1, std::abs(L.phi1[k]));
        L.max_phi2 = std::max(L.max_phi2, std::abs(L.phi2[k]));
      }
    }

    // --- scalars and state
    CU(cudaMalloc(&c->d_sc, sizeof(Scalars)));
    CU(cudaMallocHost(&c->h_sc, sizeof(Scalars)));
    CU(cudaMalloc(&c->d_red, sizeof(unsigned long long)));
    CU(cudaMallocHost(&c->h_red, sizeof(unsigned long long)));
    c->k3 = trace_points(c->p);
    c->state[0].alloc_zero(c->rot_count(), c->stream);
    if (c->partitioned) {
      // the peers address our rotating buffers directly, so they exist from the start
      c->state[1].alloc_zero(c->rot_count(), c->stream);
      c->stage[0].alloc_zero(c->rot_count(), c->stream);
      c->stage[1].alloc_zero(c->rot_count(), c->stream);
      const size_t nx = dgbk::kMaxRanks + 2 * dgbk::kMaxRanks * 4;
      CU(cudaMalloc(&c->d_xch, nx * sizeof(unsigned long long)));
      CU(cudaMemsetAsync(c->d_xch, 0, nx * sizeof(unsigned long long), c->stream));
      CU(cudaMalloc(&c->d_peers, sizeof(dgbk::PeerTab)));
      CU(cudaMemsetAsync(c->d_peers, 0, sizeof(dgbk::PeerTab), c->stream));
    }
    reset_scalars(c.get(), 0.0);
    // constant banks and the kernels' shared-memory opt-in for this device, now rather than
    // at the first launch (partitions may first launch from several host threads at once)
    ensure_tables(c.get());
    sync(c.get());
    *out = c.release();
    return DGB_OK;
  });
}

int dgb_destroy(dgb_ctx* c) {
  if (!c) return DGB_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& pd : c->pending) {
    cudaEventDestroy(pd.a);
    cudaEventDestroy(pd.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  for (cudaStream_t cs : {c->s_h2d, c->s_d2h})
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
    }
  for (cudaEvent_t ev : {c->ev_h2d, c->ev_in_free, c->ev_perm_out, c->ev_out_free})
    if (ev) cudaEventDestroy(ev);
  if (c->d_sc) cudaFree(c->d_sc);
  if (c->h_sc) cudaFreeHost(c->h_sc);
  if (c->d_red) cudaFree(c->d_red);
  if (c->h_red) cudaFreeHost(c->h_red);
  if (c->d_xch) cudaFree(c->d_xch);
  if (c->d_peers) cudaFree(c->d_peers);
  for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  const bool own = c->own_stream;
  cudaStream_t s = c->stream;
  delete c;
  if (own && s) cudaStreamDestroy(s);
  return DGB_OK;
}

int dgb_set_stream(dgb_ctx* c, void* stream) {
  return guarded([&] {
    set_device(c);
    sync(c);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
      c->own_stream = false;
    } else {
      CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    // constant banks are device state; nothing to re-upload
    return DGB_OK;
  });
}

int dgb_set_flux(dgb_ctx* c, int flux) {
  if (!c) return DGB_ERR_ARG;
  if (flux != DGB_FLUX_LLF && flux != DGB_FLUX_ROE) {
    dgb::set_message("unknown numerical flux " + std::to_string(flux));
    return DGB_ERR_ARG;
  }
  c->geo.flux = flux;
  return DGB_OK;
}

int dgb_set_fused_limiter(dgb_ctx* c, int enable) {
  if (!c || enable < -1 || enable > 1) return DGB_ERR_ARG;
  c->fuse_limit = enable;
  return DGB_OK;
}

int dgb_set_trace_buffers(dgb_ctx* c, int enable) {
  if (!c || enable < 0 || enable > 1) return DGB_ERR_ARG;
  c->trace_mode = enable;
  return DGB_OK;
}

int dgb_set_latency_forms(dgb_ctx* c, int stage_max_n, int limit_max_n) {
  if (!c || stage_max_n < -1 || limit_max_n < -1) return DGB_ERR_ARG;
  c->geo.lat_stage_n = stage_max_n;
  c->geo.lat_limit_n = limit_max_n;
  return DGB_OK;
}

int dgb_set_dirichlet(dgb_ctx* c, const double* states) {
  return guarded([&] {
    set_device(c);
    if (!states) throw Fail{DGB_ERR_ARG, "null Dirichlet table"};
    c->bc_dir.assign(states, states + 4 * static_cast<size_t>(c->n_bnd) * c->K);
    c->d_bstate.upload(c->bc_dir.data(), c->bc_dir.size(), c->stream);
    c->geo.bstate = c->d_bstate.p;
    c->geo.has_dir = 1;
    c->n_dir_stages = 0;
    sync(c);
    return DGB_OK;
  });
}

int dgb_set_dirichlet_stages(dgb_ctx* c, int n_tables, const double* tables) {
  return guarded([&] {
    set_device(c);
    if (n_tables < 1 || n_tables > 8 || !tables) throw Fail{DGB_ERR_ARG, "expected 1..8 Dirichlet stage tables"};
    const size_t per = 4 * static_cast<size_t>(c->n_bnd) * c->K;
    c->bc_dir.assign(tables, tables + per);  // stage 0 (host diagnostics of a failing ghost state)
    c->d_bstage.upload(tables, per * n_tables, c->stream);
    c->geo.bstate = c->d_bstage.p;
    c->geo.has_dir = 1;
    c->n_dir_stages = n_tables;
    sync(c);
    return DGB_OK;
  });
}

int dgb_scheme_stage_times(int scheme, double* tcoef, int* n_stages) {
  std::vector<StageSpec> st;
  if (!scheme_stages(scheme, st)) {
    dgb::set_message("rk_order must be 2 or 4");
    return DGB_ERR_ARG;
  }
  if (n_stages) *n_stages = static_cast<int>(st.size());
  if (tcoef)
    for (size_t k = 0; k < st.size(); ++k) tcoef[k] = st[k].tcoef;
  return DGB_OK;
}

int dgb_upload(dgb_ctx* c, int slot, const double* host) {
  return guarded([&] {
    set_device(c);
    upload_dev(c, slot_ptr(c, slot), 4 * c->np, host);
    sync(c);
    return DGB_OK;
  });
}

int dgb_download(dgb_ctx* c, int slot, double* host) {
  return guarded([&] {
    set_device(c);
    download_dev(c, slot_ptr(c, slot), 4 * c->np, host);
    return DGB_OK;
  });
}

namespace {
void ensure_copy_streams(dgb_ctx* c) {
  if (c->s_h2d) return;
  CU(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
  for (cudaEvent_t* ev : {&c->ev_h2d, &c->ev_in_free, &c->ev_perm_out, &c->ev_out_free})
    CU(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
}
}  // namespace

int dgb_stage_input_async(dgb_ctx* c, const double* host) {
  return guarded([&] {
    set_device(c);
    ensure_copy_streams(c);
    const size_t n = static_cast<size_t>(4 * c->np) * (c->N + c->n_halo);
    if (c->staging_in.n < n) {
      sync(c);  // a resize must not free a buffer an enqueued permute still reads
      CU(cudaStreamSynchronize(c->s_h2d));
      c->staging_in.alloc(n);
    }
    if (c->staged) throw Fail{DGB_ERR_ARG, "dgb_stage_input_async: an input is already staged (commit it first)"};
    // the previous commit's permute has consumed staging_in
    CU(cudaStreamWaitEvent(c->s_h2d, c->ev_in_free, 0));
    CU(cudaMemcpyAsync(c->staging_in.p, host, sizeof(double) * n, cudaMemcpyHostToDevice, c->s_h2d));
    CU(cudaEventRecord(c->ev_h2d, c->s_h2d));
    c->staged = true;
    return DGB_OK;
  });
}

int dgb_commit_input(dgb_ctx* c, int slot) {
  return guarded([&] {
    set_device(c);
    if (!c->staged) throw Fail{DGB_ERR_ARG, "dgb_commit_input: no staged input (call dgb_stage_input_async)"};
    double* dev = slot_ptr(c, slot);
    const int rows = 4 * c->np, nl = c->N + c->n_halo;
    CU(cudaStreamWaitEvent(c->stream, c->ev_h2d, 0));
    k_permute_in<<<small_grid(static_cast<long long>(rows) * c->ld), 256, 0, c->stream>>>(
        dev, c->staging_in.p, c->d_cmp.p, nl, nl, c->ld, rows);
    CU(cudaGetLastError());
    ++c->launches;
    CU(cudaEventRecord(c->ev_in_free, c->stream));
    c->staged = false;
    return DGB_OK;
  });
}

int dgb_upload_async(dgb_ctx* c, int slot, const double* host) {
  const int rc = dgb_stage_input_async(c, host);
  return rc != DGB_OK ? rc : dgb_commit_input(c, slot);
}

int dgb_download_async(dgb_ctx* c, int slot, double* host) {
  return guarded([&] {
    set_device(c);
    ensure_copy_streams(c);
    const double* dev = slot_ptr(c, slot);
    const int rows = 4 * c->np;
    const size_t n = static_cast<size_t>(rows) * c->N;
    if (c->staging_out.n < n) {
      CU(cudaStreamSynchronize(c->s_d2h));
      c->staging_out.alloc(n);
    }
    // the previous download's device->host copy has drained staging_out
    CU(cudaStreamWaitEvent(c->stream, c->ev_out_free, 0));
    k_permute_out<<<small_grid(static_cast<long long>(rows) * c->ld), 256, 0, c->stream>>>(
        c->staging_out.p, dev, c->d_cmp.p, c->N, c->N, c->ld, rows);
    CU(cudaGetLastError());
    ++c->launches;
    CU(cudaEventRecord(c->ev_perm_out, c->stream));
    CU(cudaStreamWaitEvent(c->s_d2h, c->ev_perm_out, 0));
    CU(cudaMemcpyAsync(host, c->staging_out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->s_d2h));
    CU(cudaEventRecord(c->ev_out_free, c->s_d2h));
    return DGB_OK;
  });
}

int dgb_sync(dgb_ctx* c) {
  return guarded([&] {
    set_device(c);
    if (c->s_h2d) CU(cudaStreamSynchronize(c->s_h2d));
    if (c->s_d2h) CU(cudaStreamSynchronize(c->s_d2h));
    sync(c);
    return DGB_OK;
  });
}

int dgb_copy_slot(dgb_ctx* c, int dst, int src) {
  return guarded([&] {
    set_device(c);
    double* d = slot_ptr(c, dst);
    const double* s = slot_ptr(c, src);
    if (d != s) CU(cudaMemcpyAsync(d, s, c->coeff_count() * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    sync(c);
    return DGB_OK;
  });
}

int dgb_eval_volume_pass(dgb_ctx* c, int in_slot) {
  return guarded([&] {
    set_device(c);
    run_pass(c, dgbk::kModeVolume, slot_ptr(c, in_slot), slot_ptr(c, DGB_SLOT_VOLUME), 0.0, 0);
    return DGB_OK;
  });
}

int dgb_eval_surface_pass(dgb_ctx* c, int in_slot, double t) {
  return guarded([&] {
    set_device(c);
    check_bc(c);
    if (!c->slots.p) {
      c->slots.alloc(3 * c->coeff_count());
      CU(cudaMemsetAsync(c->slots.p, 0, 3 * c->coeff_count() * sizeof(double), c->stream));
    }
    run_pass(c, dgbk::kModeSurface, slot_ptr(c, in_slot), c->slots.p, t, 1);
    return DGB_OK;
  });
}

int dgb_download_surface(dgb_ctx* c, double* left, double* right) {
  return guarded([&] {
    set_device(c);
    if (c->partitioned) throw Fail{DGB_ERR_ARG, "surface slot buffers are whole-mesh only"};
    const size_t per = static_cast<size_t>(4) * c->np * c->N;
    std::vector<double> all(3 * per);
    if (!c->slots.p) throw Fail{DGB_ERR_ARG, "no surface pass has been evaluated"};
    download_dev(c, c->slots.p, 12 * c->np, all.data());
    const int N = c->N, np = c->np;
    std::memset(left, 0, sizeof(double) * 3 * per);
    std::memset(right, 0, sizeof(double) * 3 * per);
    for (int q = 0; q < 3; ++q)
      for (int i = 0; i < N; ++i) {
        const bool from_left = c->eleft[c->elem_edge[3 * i + q]] == i;
        double* dst = from_left ? left : right;
        for (int mm = 0; mm < 4; ++mm)
          for (int j = 0; j < np; ++j) {
            const size_t idx = ((static_cast<size_t>(q) * 4 + mm) * np + j) * N + i;
            dst[idx] = all[idx];
          }
      }
    return DGB_OK;
  });
}

int dgb_upload_surface(dgb_ctx* c, const double* left, const double* right) {
  return guarded([&] {
    set_device(c);
    if (c->partitioned) throw Fail{DGB_ERR_ARG, "surface slot buffers are whole-mesh only"};
    const size_t per = static_cast<size_t>(4) * c->np * c->N;
    std::vector<double> all(3 * per);
    const int N = c->N, np = c->np;
    for (int q = 0; q < 3; ++q)
      for (int i = 0; i < N; ++i) {
        const bool from_left = c->eleft[c->elem_edge[3 * i + q]] == i;
        const double* src = from_left ? left : right;
        for (int mm = 0; mm < 4; ++mm)
          for (int j = 0; j < np; ++j) {
            const size_t idx = ((static_cast<size_t>(q) * 4 + mm) * np + j) * N + i;
            all[idx] = src[idx];
          }
      }
    if (!c->slots.p) c->slots.alloc(3 * c->coeff_count());
    upload_dev(c, c->slots.p, 12 * c->np, all.data());
    sync(c);
    return DGB_OK;
  });
}

int dgb_eval_rhs_pass(dgb_ctx* c) {
  return guarded([&] {
    set_device(c);
    if (!c->slots.p) throw Fail{DGB_ERR_ARG, "no surface pass has been evaluated"};
    double* vol = slot_ptr(c, DGB_SLOT_VOLUME);
    double* der = slot_ptr(c, DGB_SLOT_DERIV);
    Timed tm(c, 2);
    k_gather<<<small_grid(static_cast<long long>(4) * c->np * c->ld), 256, 0, c->stream>>>(
        der, vol, c->slots.p, c->d_inv_det.p, c->N, c->ld, 4 * c->np);
    CU(cudaGetLastError());
    ++c->launches;
    return DGB_OK;
  });
}

int dgb_compute_rhs(dgb_ctx* c, int in_slot, double t, int out_slot) {
  return guarded([&] {
    set_device(c);
    check_bc(c);
    if (in_slot == out_slot) throw Fail{DGB_ERR_ARG, "compute_rhs needs distinct input and output slots"};
    run_pass(c, dgbk::kModeRhs, slot_ptr(c, in_slot), slot_ptr(c, out_slot), t, 2);
    return DGB_OK;
  });
}

int dgb_limit(dgb_ctx* c, int slot) {
  return guarded([&] {
    set_device(c);
    if (c->p != 1) throw Fail{DGB_ERR_ARG, "slope limiting is only supported for p = 1"};
    ensure_tables(c);
    reset_scalars(c, c->t);
    LimArgs la{};
    la.c = slot_ptr(c, slot);
    la.u = la.c;
    la.sc = c->d_sc;
    la.e0 = 0;
    la.e1 = c->N;
    {
      Timed tm(c, 3);
      CU(dgbk::launch_limit(0, c->geo, la, c->stream));
      ++c->launches;
    }
    sync(c);
    return DGB_OK;
  });
}

int dgb_stable_dt(dgb_ctx* c, int slot, double cfl, double* dt) {
  return guarded([&] {
    set_device(c);
    ensure_tables(c);
    reset_scalars(c, c->t);
    {
      Timed tm(c, 4);
      CU(launch_dt(c, slot_ptr(c, slot), 0, 0));
      ++c->launches;
    }
    read_scalars(c);
    if (c->h_sc->err_key != dgbk::kNoError)
      throw Fail{DGB_ERR_INADMISSIBLE, failure_message(c, c->h_sc->err_key, slot_ptr(c, slot), c->t)};
    *dt = cfl * __builtin_bit_cast(double, c->h_sc->dtmin[0]);
    return DGB_OK;
  });
}

int dgb_set_time(dgb_ctx* c, double t, int64_t step) {
  c->t = t;
  c->step_count = step;
  return DGB_OK;
}

int dgb_get_time(dgb_ctx* c, double* t, int64_t* step) {
  if (t) *t = c->t;
  if (step) *step = c->step_count;
  return DGB_OK;
}

int dgb_rk_step(dgb_ctx* c, int scheme, double dt, int limiting, double* residual) {
  return guarded([&] {
    set_device(c);
    RunSpec r;
    r.scheme = scheme;
    r.dt_mode = 0;
    r.dt_host = dt;
    r.limiting = limiting != 0;
    r.max_steps = 1;
    RunOut o = run_steps(c, r);
    if (residual) *residual = o.residual;
    return DGB_OK;
  });
}

int dgb_run_fixed_steps(dgb_ctx* c, int scheme, double cfl, int limiting, int64_t n, double* residual, double* hist) {
  return guarded([&] {
    set_device(c);
    if (n <= 0) {
      if (residual) *residual = 0.0;
      return DGB_OK;
    }
    RunSpec r;
    r.scheme = scheme;
    r.dt_mode = 1;
    r.cfl = cfl;
    r.limiting = limiting != 0;
    r.max_steps = n;
    r.hist = hist;
    r.hist_cap = hist ? n : 0;
    RunOut o = run_steps(c, r);
    if (residual) *residual = o.residual;
    return DGB_OK;
  });
}

int dgb_run_to_time(dgb_ctx* c, int scheme, double cfl, int limiting, double t_end, int64_t max_steps,
                    double* residual, int64_t* steps_taken, double* hist, int64_t hist_cap) {
  return guarded([&] {
    set_device(c);
    RunSpec r;
    r.scheme = scheme;
    r.dt_mode = 1;
    r.cfl = cfl;
    r.limiting = limiting != 0;
    r.max_steps = max_steps;
    r.clip = true;
    r.stop_t = true;
    r.t_end = t_end;
    r.hist = hist;
    r.hist_cap = hist ? hist_cap : 0;
    if (!(c->t < t_end)) {
      if (residual) *residual = 0.0;
      if (steps_taken) *steps_taken = 0;
      return DGB_OK;
    }
    RunOut o = max_steps > 0 ? run_steps(c, r) : RunOut{};
    if (steps_taken) *steps_taken = o.steps;
    if (residual) *residual = o.residual;
    if (!o.halted && c->t < t_end)
      throw Fail{DGB_ERR_NOT_REACHED, "t_end not reached within " + std::to_string(max_steps) + " steps"};
    return DGB_OK;
  });
}

int dgb_run_to_steady(dgb_ctx* c, int scheme, double cfl, int limiting, double tol, int64_t max_steps, int64_t* steps,
                      double* residual, int* converged, double* hist, int64_t hist_cap) {
  return guarded([&] {
    set_device(c);
    RunSpec r;
    r.scheme = scheme;
    r.dt_mode = 1;
    r.cfl = cfl;
    r.limiting = limiting != 0;
    r.max_steps = max_steps;
    r.stop_steady = true;
    r.tol = tol;
    r.hist = hist;
    r.hist_cap = hist ? hist_cap : 0;
    RunOut o = max_steps > 0 ? run_steps(c, r) : RunOut{};
    if (steps) *steps = o.steps;
    if (residual) *residual = o.residual;
    if (converged) *converged = (o.steps > 0 && o.residual <= tol) ? 1 : 0;
    return DGB_OK;
  });
}

int dgb_total_mass(dgb_ctx* c, int slot, double* mass) {
  return guarded([&] {
    set_device(c);
    std::vector<double> row(c->N);
    download_dev(c, slot_ptr(c, slot), 1, row.data());
    const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
    double s = 0.0;  // partition: this rank's partial sum, reference order (ranks add in rank order)
    for (int i = 0; i < c->N; ++i) s += c->det[c->lo + i] * row[i] * inv_sqrt2;
    *mass = s;
    return DGB_OK;
  });
}

int dgb_l2_error(dgb_ctx* c, int slot, const double* exact_rho, double* l2) {
  return guarded([&] {
    set_device(c);
    if (!exact_rho || !l2) throw Fail{DGB_ERR_ARG, "null argument"};
    const int n = c->N, nq = c->nq, np = c->np;
    DevBuf<double> tab, ex, part;
    std::vector<double> h(static_cast<size_t>(nq) * np + nq);
    std::copy(c->t_phi.begin(), c->t_phi.end(), h.begin());
    std::copy(c->t_w.begin(), c->t_w.end(), h.begin() + static_cast<size_t>(nq) * np);
    tab.upload(h.data(), h.size(), c->stream);
    ex.upload(exact_rho, static_cast<size_t>(n) * nq, c->stream);
    part.alloc(n);
    k_l2_partial<<<small_grid(n), 256, 0, c->stream>>>(slot_ptr(c, slot), ex.p, tab.p, c->d_cmp.p, c->d_inv_det.p, n,
                                                        c->ld, np, nq, part.p);
    CU(cudaGetLastError());
    ++c->launches;
    std::vector<double> hp(n);
    CU(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    double total = 0.0;  // element order (runner.cpp:146-148); a partition returns its partial sum squared
    for (int i = 0; i < n; ++i) total += hp[i];
    *l2 = c->partitioned ? total : std::sqrt(total);
    return DGB_OK;
  });
}

int dgb_project_slot(dgb_ctx* c, int slot, const double* point_states) {
  return guarded([&] {
    set_device(c);
    if (!point_states) throw Fail{DGB_ERR_ARG, "null argument"};
    const int nl = c->N + c->n_halo, nq = c->nq, np = c->np;
    std::vector<double> h(static_cast<size_t>(nq) * np + nq);
    std::copy(c->t_phi.begin(), c->t_phi.end(), h.begin());
    std::copy(c->t_w.begin(), c->t_w.end(), h.begin() + static_cast<size_t>(nq) * np);
    DevBuf<double> tab, ps;
    tab.upload(h.data(), h.size(), c->stream);
    ps.upload(point_states, static_cast<size_t>(nl) * nq * 4, c->stream);
    double* dst = slot_ptr(c, slot);
    CU(cudaMemsetAsync(dst, 0, c->coeff_count() * sizeof(double), c->stream));
    *c->h_red = ~0ull;
    CU(cudaMemcpyAsync(c->d_red, c->h_red, sizeof(unsigned long long), cudaMemcpyHostToDevice, c->stream));
    k_project<<<small_grid(nl), 256, 0, c->stream>>>(ps.p, tab.p, c->d_cmp.p, nl, c->ld, np, nq, dst, c->gamma, c->d_red);
    CU(cudaGetLastError());
    ++c->launches;
    CU(cudaMemcpyAsync(c->h_red, c->d_red, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (*c->h_red != ~0ull) {
      const unsigned long long i = *c->h_red / 64, k = *c->h_red % 64;
      const double* u = point_states + (i * nq + k) * 4;
      throw Fail{DGB_ERR_INADMISSIBLE, "project_initial: inadmissible state at id " + std::to_string(i) + ", point " +
                                           std::to_string(k) + " (rho=" + std::to_string(u[0]) +
                                           ", p=" + std::to_string(pressure_ref(u, c->gamma)) + ")"};
    }
    return DGB_OK;
  });
}

int dgb_corner_states(dgb_ctx* c, int slot, const double* phi_corner, double* out) {
  return guarded([&] {
    set_device(c);
    if (!phi_corner || !out) throw Fail{DGB_ERR_ARG, "null argument"};
    DevBuf<double> tab, dev;
    tab.upload(phi_corner, 3 * static_cast<size_t>(c->np), c->stream);
    dev.alloc(12 * static_cast<size_t>(c->N));
    k_corner_states<<<small_grid(c->N), 256, 0, c->stream>>>(slot_ptr(c, slot), tab.p, c->d_cmp.p, c->N, c->ld, c->np,
                                                             dev.p);
    CU(cudaGetLastError());
    ++c->launches;
    CU(cudaMemcpyAsync(out, dev.p, sizeof(double) * 12 * c->N, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    return DGB_OK;
  });
}

int dgb_max_abs_diff(dgb_ctx* c, int sa, int sb, double* diff) {
  return guarded([&] {
    set_device(c);
    const double* a = slot_ptr(c, sa);
    const double* b = slot_ptr(c, sb);
    CU(cudaMemsetAsync(c->d_red, 0, sizeof(unsigned long long), c->stream));
    k_max_abs_diff<<<small_grid(static_cast<long long>(4) * c->np * c->ld), 256, 0, c->stream>>>(
        a, b, c->N, c->ld, 4 * c->np, c->d_red);
    CU(cudaGetLastError());
    ++c->launches;
    CU(cudaMemcpyAsync(c->h_red, c->d_red, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    *diff = __builtin_bit_cast(double, *c->h_red);
    return DGB_OK;
  });
}

int dgb_timers(dgb_ctx* c, dgb_pass_timers* out) {
  return guarded([&] {
    set_device(c);
    sync(c);
    *out = c->timers;
    return DGB_OK;
  });
}

int dgb_reset_timers(dgb_ctx* c) {
  return guarded([&] {
    set_device(c);
    sync(c);
    c->timers = dgb_pass_timers{};
    c->stage_ms = 0.0;
    c->stage_launches = 0;
    for (auto& v : c->samples) v.clear();
    return DGB_OK;
  });
}

int dgb_enable_timers(dgb_ctx* c, int enable) {
  c->timing = enable != 0;
  return DGB_OK;
}

int dgb_last_abort(dgb_ctx* c, dgb_abort_info* out) {
  *out = c->last_abort;
  return DGB_OK;
}

int64_t dgb_launch_count(dgb_ctx* c) { return c->launches; }

int dgb_fp64_peak(int device, double* tflops) {
  return guarded([&] {
    CU(cudaSetDevice(device));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* d = nullptr;
    CU(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    k_fp64_peak<<<blocks, threads>>>(d, 64);  // warm up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CU(cudaEventRecord(a));
      k_fp64_peak<<<blocks, threads>>>(d, iters);
      CU(cudaEventRecord(b));
      CU(cudaEventSynchronize(b));
      float ms = 0.f;
      CU(cudaEventElapsedTime(&ms, a, b));
      best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    *tflops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads / (best * 1e-3) / 1e12;
    return DGB_OK;
  });
}

// ------------------------------------------------------------------ partitions (multi-GPU)
int dgb_part_get_info(dgb_ctx* c, dgb_part_info* out) {
  if (!c || !out) return DGB_ERR_ARG;
  out->rank = c->rank;
  out->world = c->world;
  out->lo = c->lo;
  out->hi = c->hi;
  out->n_owned = c->N;
  out->n_halo = c->n_halo;
  out->n_interior = c->partitioned ? c->n_int : c->N;
  out->ld = c->ld;
  out->neighbor_mask = c->nb_mask;
  return DGB_OK;
}

int dgb_part_plan(const dgb_mesh_view* m, int rank, int world, dgb_part_info* info, int32_t* halo_ids,
                  int32_t* boundary_ids) {
  return guarded([&] {
    if (!m || !info || world < 1 || world > dgbk::kMaxRanks || rank < 0 || rank >= world || m->n_elements < world)
      throw Fail{DGB_ERR_ARG, "bad partition arguments"};
    PartPlan P;
    make_plan(m, rank, world, P);
    info->rank = rank;
    info->world = world;
    info->lo = P.lo;
    info->hi = P.hi;
    info->n_owned = P.hi - P.lo;
    info->n_halo = static_cast<int32_t>(P.halo.size());
    info->n_interior = static_cast<int32_t>(P.interior.size());
    info->ld = (info->n_owned + info->n_halo + 31) / 32 * 32;
    info->neighbor_mask = P.nb_mask;
    if (halo_ids) std::copy(P.halo.begin(), P.halo.end(), halo_ids);
    if (boundary_ids) std::copy(P.boundary.begin(), P.boundary.end(), boundary_ids);
    return DGB_OK;
  });
}

int dgb_part_halo_ids(dgb_ctx* c, int32_t* gids, int32_t* cols) {
  return guarded([&] {
    for (int h = 0; h < c->n_halo; ++h) {
      if (gids) gids[h] = c->halo_gid[h];
      if (cols) cols[h] = c->N + h;
    }
    return DGB_OK;
  });
}

int dgb_part_local_ids(dgb_ctx* c, int32_t* gids) {
  return guarded([&] {
    for (int l = 0; l < c->N; ++l) gids[l] = c->lo + l;
    for (int h = 0; h < c->n_halo; ++h) gids[c->N + h] = c->halo_gid[h];
    return DGB_OK;
  });
}

int dgb_part_peer_view(dgb_ctx* c, dgb_peer_view* out) {
  return guarded([&] {
    if (!c->partitioned) throw Fail{DGB_ERR_ARG, "not a partitioned context"};
    out->buf[0] = c->state[0].p;
    out->buf[1] = c->state[1].p;
    out->buf[2] = c->stage[0].p;
    out->buf[3] = c->stage[1].p;
    out->flags = c->d_xch;
    out->scal = c->d_xch + dgbk::kMaxRanks;
    out->ld = c->ld;
    return DGB_OK;
  });
}

namespace {
void attach_view(dgb_ctx* c, int peer, const dgb_peer_view* v) {
  if (!c->partitioned || peer < 0 || peer >= c->world || peer == c->rank || !v) throw Fail{DGB_ERR_ARG, "bad peer"};
  for (int k = 0; k < 4; ++k) c->h_peers.buf[peer][k] = static_cast<double*>(v->buf[k]);
    c->h_peers.ld[peer] = v->ld;
    c->h_peers.flag[peer] = static_cast<unsigned long long*>(v->flags);
    c->h_peers.scal[peer] = static_cast<unsigned long long*>(v->scal);
}
}  // namespace

int dgb_part_attach_peer(dgb_ctx* c, int peer, const dgb_peer_view* v) {
  return guarded([&] {
    if (!v || !v->buf[0]) throw Fail{DGB_ERR_ARG, "bad peer view"};
    // a peer on another device of this process: this context's kernels store into the peer's
    // buffers, so this device needs peer access to the peer's device (NVLink P2P)
    cudaPointerAttributes pa{};
    CU(cudaPointerGetAttributes(&pa, v->buf[0]));
    if (pa.type == cudaMemoryTypeDevice && pa.device != c->device) {
      int can = 0;
      CU(cudaDeviceCanAccessPeer(&can, c->device, pa.device));
      if (!can)
        throw Fail{DGB_ERR_ARG, "device " + std::to_string(c->device) + " cannot access peer device " +
                                    std::to_string(pa.device) + " (no P2P path)"};
      set_device(c);
      const cudaError_t e = cudaDeviceEnablePeerAccess(pa.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled)
        cudaGetLastError();  // clear the sticky-free "already enabled" status
      else
        CU(e);
    }
    attach_view(c, peer, v);
    return DGB_OK;
  });
}

int dgb_part_ipc_export(dgb_ctx* c, void* handles) {
  return guarded([&] {
    if (!c->partitioned) throw Fail{DGB_ERR_ARG, "not a partitioned context"};
    set_device(c);
    auto* h = static_cast<cudaIpcMemHandle_t*>(handles);
    void* ptrs[5] = {c->state[0].p, c->state[1].p, c->stage[0].p, c->stage[1].p, c->d_xch};
    for (int k = 0; k < 5; ++k) CU(cudaIpcGetMemHandle(&h[k], ptrs[k]));
    return DGB_OK;
  });
}

int dgb_part_attach_peer_ipc(dgb_ctx* c, int peer, const void* handles, int32_t peer_ld) {
  return guarded([&] {
    if (!c->partitioned || peer < 0 || peer >= c->world || peer == c->rank) throw Fail{DGB_ERR_ARG, "bad peer"};
    set_device(c);
    const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
    void* ptrs[5];
    for (int k = 0; k < 5; ++k) {
      CU(cudaIpcOpenMemHandle(&ptrs[k], h[k], cudaIpcMemLazyEnablePeerAccess));
      c->ipc_opened.push_back(ptrs[k]);
    }
    dgb_peer_view v{};
    for (int k = 0; k < 4; ++k) v.buf[k] = ptrs[k];
    v.flags = ptrs[4];
    v.scal = static_cast<unsigned long long*>(ptrs[4]) + dgbk::kMaxRanks;
    v.ld = peer_ld;
    attach_view(c, peer, &v);  // cudaIpcMemLazyEnablePeerAccess already enabled the P2P mapping
    return DGB_OK;
  });
}

int dgb_part_set_sends(dgb_ctx* c, int peer, int64_t n, const int32_t* gids, const int32_t* peer_cols) {
  return guarded([&] {
    if (!c->partitioned || peer < 0 || peer >= c->world || peer == c->rank) throw Fail{DGB_ERR_ARG, "bad peer"};
    auto& v = c->sends[peer];
    v.clear();
    for (int64_t k = 0; k < n; ++k) {
      const int g = gids[k];
      if (g < c->lo || g >= c->hi) throw Fail{DGB_ERR_ARG, "send element not owned by this rank"};
      if (c->col_of[g] < c->n_int) throw Fail{DGB_ERR_ARG, "send element is not on the partition boundary"};
      v.emplace_back(g, peer_cols[k]);
    }
    c->finalized = false;
    return DGB_OK;
  });
}

int dgb_part_finalize(dgb_ctx* c) {
  return guarded([&] {
    if (!c->partitioned) return DGB_OK;
    set_device(c);
    for (int r = 0; r < c->world; ++r)
      if (r != c->rank && (!c->h_peers.flag[r] || !c->h_peers.buf[r][0]))
        throw Fail{DGB_ERR_ARG, "peer " + std::to_string(r) + " not attached"};
    c->send_mask = 0;
    std::vector<int4> ent;
    for (int r = 0; r < c->world; ++r) {
      if (!c->sends[r].empty()) c->send_mask |= 1u << r;
      std::vector<std::pair<int, int>> v;  // (peer column, own column)
      for (auto& e : c->sends[r]) v.emplace_back(e.second, c->col_of[e.first]);
      std::sort(v.begin(), v.end());
      for (auto& x : v) ent.push_back(make_int4(x.second, r, x.first, 0));
    }
    c->n_push = static_cast<int>(ent.size());
    if (!ent.empty()) c->d_push.upload(ent.data(), ent.size(), c->stream);
    CU(cudaMemcpyAsync(c->d_peers, &c->h_peers, sizeof(dgbk::PeerTab), cudaMemcpyHostToDevice, c->stream));
    // every kernel a step may launch is loaded now, not lazily while the peers spin in k_wait
    {
      cudaFuncAttributes fa;
      CU(cudaFuncGetAttributes(&fa, k_signal));
      CU(cudaFuncGetAttributes(&fa, k_wait));
      CU(cudaFuncGetAttributes(&fa, k_push));
    }
    switch (c->p) {
      case 1: CU(dgbk::Launch<1>::preload()); CU(dgbk::preload_limit()); break;
      case 2: CU(dgbk::Launch<2>::preload()); break;
      case 3: CU(dgbk::Launch<3>::preload()); break;
      case 4: CU(dgbk::Launch<4>::preload()); break;
      default: CU(dgbk::Launch<5>::preload()); break;
    }
    sync(c);
    c->finalized = true;
    return DGB_OK;
  });
}

int dgb_part_set_timeout(dgb_ctx* c, double seconds) {
  if (!c || !(seconds > 0)) return DGB_ERR_ARG;
  c->timeout_s = seconds;
  return DGB_OK;
}

int dgb_timer_samples(dgb_ctx* c, int category, double* ms, int64_t cap, int64_t* n) {
  return guarded([&] {
    if (category < 0 || category > 5) throw Fail{DGB_ERR_ARG, "timer category must be in [0,5]"};
    set_device(c);
    sync(c);
    const std::vector<double>& v = c->samples[category];
    if (n) *n = static_cast<int64_t>(v.size());
    if (ms) std::copy(v.begin(), v.begin() + std::min<int64_t>(cap, static_cast<int64_t>(v.size())), ms);
    return DGB_OK;
  });
}

int dgb_stage_kernel_ms(dgb_ctx* c, double* ms, int64_t* launches) {
  return guarded([&] {
    set_device(c);
    sync(c);
    if (ms) *ms = c->stage_ms;
    if (launches) *launches = c->stage_launches;
    return DGB_OK;
  });
}

}  // extern "C"
