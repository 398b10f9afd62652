// One translation unit per polynomial degree: its constant bank, the four
// element-kernel modes and the CFL kernel.  Included by kernels_pN.cu with
// DGB_P defined.
#include <atomic>
#include <cstdlib>

#include "element_mma.cuh"
#include "launch.hpp"

#ifndef DGB_MMA_MINP
#define DGB_MMA_MINP 3  // degrees >= this use the DMMA (FP64 tensor core) element kernel (measured
                        // per stage at p=3: DMMA 0.98 ms vs 1.05 ms for the 4-lane DFMA kernel)
#endif
#ifndef DGB_MMA_THREADS
// DMMA kernel: one block per SM; p=3 16 warps (128 registers), p=4,5 12 warps (168 registers)
#define DGB_MMA_THREADS(P) ((P) == 3 ? 512 : 384)
#endif
#ifndef DGB_MMA_MINB
#define DGB_MMA_MINB(P) 1
#endif

namespace dgbk {

// Everything in this unit is internal: each degree has its own constant bank
// and its own kernel instances.
namespace {
__constant__ Tab<DGB_P> c_tab;
constexpr int kG = Lanes<DGB_P>::value;  // lanes per element
#ifndef DGB_G4_PER_SM
#define DGB_G4_PER_SM 32  // measured on the 2,880-triangle vortex mesh: 11.6 vs 12.5 us per stage; 11,520: 13.6 vs 12.7 (worse)
#endif
constexpr int kG4PerSm = DGB_G4_PER_SM;  // latency-form stage kernel up to this many elements per SM

constexpr bool kMma = DGB_P >= DGB_MMA_MINP;
// trace-buffer stage instances (kVarTrace) exist for the packed-surface DMMA degrees
constexpr bool kTraceOK = (kMma || kG == 1) && DGB_TRACE_P(DGB_P);
constexpr int kMinB = kMma ? DGB_MMA_MINB(DGB_P) : MinBlocks<DGB_P>::value;
constexpr int kThreads = kMma ? DGB_MMA_THREADS(DGB_P) : kBlock;  // threads per block of k_element
// dynamic shared memory (bytes): tables + per-warp staging buffers
constexpr int kSmem = kMma ? (MmaDim<DGB_P>::kBufOff + (kThreads / 32) * MmaDim<DGB_P>::kWarpBuf) * 8
                            : (kG == 1 ? g1_pipe_bytes<DGB_P>() * kThreads : 0);

// One instance per mode, numerical flux (geo.flux) and variant (kVar* bits, dg_kernels.cuh):
// the stage mode with or without the RK4 accumulator (a.kmode != 0) and the CFL epilogue
// (a.want_lambda), and every surface mode with or without physical-boundary code
// (geo.has_bnd).  Without the RK4 branches the midpoint-RK2 / SSP stage needs fewer
// registers (measured per stage: p=1 0.158 vs 0.131 ms, p=2 0.390 vs 0.328, p=4 1.050 vs
// 0.977, p=5 1.726 vs 1.623).
template <int MODE, int FLUX, int VAR>
__global__ void __launch_bounds__(kThreads, kMinB) k_element(Geo geo, StageArgs a) {
  if constexpr (kMma) {
    extern __shared__ __align__(128) double smem[];
    element_body_mma<DGB_P, MODE, FLUX, VAR>(c_tab, geo, a, smem);
  } else if constexpr (kG == 1) {
    element_body_g1<DGB_P, MODE, FLUX, VAR>(c_tab, geo, a);
  } else {
    element_body<DGB_P, MODE, FLUX, VAR>(c_tab, geo, a);
  }
}

// Latency form of the low-degree stage kernel: four lanes per element (element_body, lane =
// conserved variable, each pointwise evaluation on its own lane), for launches too small to
// fill the GPU, where a stage costs one element's dependency chain rather than bandwidth.
// The same operations in the same order as the one-thread body: bit-identical.
template <int FLUX, int VAR>
__global__ void __launch_bounds__(kBlock) k_element4(Geo geo, StageArgs a) {
  if constexpr (!kMma && kG == 1) element_body<DGB_P, kModeStage, FLUX, VAR>(c_tab, geo, a);
}
template <int FLUX, class F>
void with_instance4(int var, F&& f) {
  switch (var & 7) {
    case 0: f(k_element4<FLUX, 0>); break;
    case 1: f(k_element4<FLUX, 1>); break;
    case 2: f(k_element4<FLUX, 2>); break;
    case 3: f(k_element4<FLUX, 3>); break;
    case 4: f(k_element4<FLUX, 4>); break;
    case 5: f(k_element4<FLUX, 5>); break;
    case 6: f(k_element4<FLUX, 6>); break;
    default: f(k_element4<FLUX, 7>); break;
  }
}

// Calls f(kernel) for the instance that serves (mode, flux, var).
template <int FLUX, class F>
void with_instance(int mode, int var, F&& f) {
  switch (mode) {
    case kModeVolume: f(k_element<kModeVolume, FLUX, 0>); break;
    case kModeSurface:
      if (var & kVarBoundary) f(k_element<kModeSurface, FLUX, kVarBoundary>); else f(k_element<kModeSurface, FLUX, 0>);
      break;
    case kModeRhs:
      if (var & kVarBoundary) f(k_element<kModeRhs, FLUX, kVarBoundary>); else f(k_element<kModeRhs, FLUX, 0>);
      break;
    default:
      if constexpr (kTraceOK) {
        if (var & kVarTrace) {
          switch (var & 7) {
            case 0: f(k_element<kModeStage, FLUX, 8>); break;
            case 1: f(k_element<kModeStage, FLUX, 9>); break;
            case 2: f(k_element<kModeStage, FLUX, 10>); break;
            case 3: f(k_element<kModeStage, FLUX, 11>); break;
            case 4: f(k_element<kModeStage, FLUX, 12>); break;
            case 5: f(k_element<kModeStage, FLUX, 13>); break;
            case 6: f(k_element<kModeStage, FLUX, 14>); break;
            default: f(k_element<kModeStage, FLUX, 15>); break;
          }
          break;
        }
      }
      switch (var & 7) {
        case 0: f(k_element<kModeStage, FLUX, 0>); break;
        case 1: f(k_element<kModeStage, FLUX, 1>); break;
        case 2: f(k_element<kModeStage, FLUX, 2>); break;
        case 3: f(k_element<kModeStage, FLUX, 3>); break;
        case 4: f(k_element<kModeStage, FLUX, 4>); break;
        case 5: f(k_element<kModeStage, FLUX, 5>); break;
        case 6: f(k_element<kModeStage, FLUX, 6>); break;
        default: f(k_element<kModeStage, FLUX, 7>); break;
      }
      break;
  }
}
template <class F>
void with_instance(int flux, int mode, int var, F&& f) {
  if (flux == kFluxRoe)
    with_instance<kFluxRoe>(mode, var, f);
  else
    with_instance<kFluxLLF>(mode, var, f);
}
#ifndef DGB_VAR_MASK
// variant bits specialised per degree (the others take the full path).  Round 1 kept the boundary
// code in the p=2 periodic instance (0.307 vs 0.341 ms, register allocation); with the round-2
// kernel the split is faster there too (0.294 vs 0.301 ms, interleaved A/B)
#define DGB_VAR_MASK(P) 7
#endif
int variant_of(int mode, const Geo& g, const StageArgs& a) {
  constexpr int mask = DGB_VAR_MASK(DGB_P);
  int v = g.has_bnd ? kVarBoundary : 0;
  if (mode == kModeStage) v |= (a.kmode != 0 ? kVarRk4 : 0) | (a.want_lambda ? kVarLambda : 0);
  return (v & mask) | (7 & ~mask) | (kTraceOK && mode == kModeStage && a.tr_in ? kVarTrace : 0);
}

__global__ void __launch_bounds__(kBlock) k_dt(Geo geo, const double* __restrict__ c, Scalars* sc, int slot,
                                               unsigned long long seq) {
  dt_body<DGB_P>(c_tab, geo, c, sc, slot, seq);
}

// Per-device caches: contexts on several devices may launch from several host threads
// (dist.run_group), so every entry is an atomic indexed by the current device.
constexpr int kMaxDevices = 64;
std::atomic<int> g_sms[kMaxDevices];
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & (kMaxDevices - 1);
}
int sm_count() {
  std::atomic<int>& s = g_sms[current_device()];
  int v = s.load(std::memory_order_relaxed);
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    s.store(v, std::memory_order_relaxed);
  }
  return v;
}
template <class Kern>
int occupancy(Kern k, int smem = 0, int threads = kBlock) {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, smem);
  return n > 0 ? n : 1;
}
int grid_for(long long threads, int blocks_per_sm, int block = kBlock) {
  const long long need = (threads + block - 1) / block;
  const long long cap = static_cast<long long>(blocks_per_sm) * sm_count();
  return static_cast<int>(need < cap ? need : cap);
}
}  // namespace

template <>
cudaError_t Launch<DGB_P>::upload(const Tab<DGB_P>& t, cudaStream_t s) {
  if constexpr (kSmem > 32 * 1024) {  // opt in to large dynamic shared memory (with the static part > 48 KB): a per-device function attribute
    static std::atomic<unsigned long long> done{0};
    const unsigned long long bit = 1ull << current_device();
    if (!(done.load() & bit)) {
      cudaError_t err = cudaSuccess;
      for (int flux = 0; flux < 2; ++flux)
        for (int mode = 0; mode < 4; ++mode)
          for (int var = 0; var < 16; ++var)
            with_instance(flux, mode, var, [&](auto k) {
              const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
              if (e != cudaSuccess) err = e;
            });
      if (err != cudaSuccess) return err;
      done.fetch_or(bit);
    }
  }
  return cudaMemcpyToSymbolAsync(c_tab, &t, sizeof(t), 0, cudaMemcpyHostToDevice, s);
}

template <>
int Launch<DGB_P>::resident_blocks(int mode) {
  // the LLF instance of the full variant (the others are sized the same by __launch_bounds__)
  static std::atomic<int> cache[4];
  int v = cache[mode].load(std::memory_order_relaxed);
  if (!v) {
    with_instance(kFluxLLF, mode, 7, [&](auto k) { v = occupancy(k, kSmem, kThreads); });
    cache[mode].store(v, std::memory_order_relaxed);
  }
  return v;
}

template <>
cudaError_t Launch<DGB_P>::preload() {
  cudaError_t err = cudaSuccess;
  auto touch = [&](auto k) {
    cudaFuncAttributes fa;
    const cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) err = e;
  };
  for (int flux = 0; flux < 2; ++flux)
    for (int mode = 0; mode < 4; ++mode)
      for (int var = 0; var < 16; ++var) with_instance(flux, mode, var, touch);
  for (int var = 0; var < 8; ++var) {
    with_instance4<kFluxLLF>(var, touch);
    with_instance4<kFluxRoe>(var, touch);
  }
  touch(k_dt);
  return err;
}

template <>
int Launch<DGB_P>::trace_points() {
  return kTraceOK ? 3 * Dim<DGB_P>::K : 0;
}


template <>
int Launch<DGB_P>::lanes() {
  return kMma ? 0 : kG;
}

template <>
int Launch<DGB_P>::mma_table(const Tab<DGB_P>& t, double* out) {
  if constexpr (kMma) {
    if (out) fill_mma_tab<DGB_P>(t, out);
    return MmaDim<DGB_P>::kSize;
  } else {
    return 0;
  }
}

// Elements up to which a low-degree stage launch takes the four-lane latency form
// (k_element4); DGB_G4_MAXN overrides (0: never).
namespace {
int stage_latency_max_n() {
  static std::atomic<int> v{-1};
  int n = v.load(std::memory_order_relaxed);
  if (n < 0) {
    const char* env = std::getenv("DGB_G4_MAXN");
    n = env ? std::atoi(env) : kG4PerSm * sm_count();
    v.store(n, std::memory_order_relaxed);
  }
  return n;
}
}  // namespace

template <>
cudaError_t Launch<DGB_P>::element(int mode, int grid, const Geo& g, const StageArgs& a, cudaStream_t s) {
  if (a.e1 <= a.e0) return cudaSuccess;
  if constexpr (!kMma && kG == 1) {
    // (trace mode always takes the one-thread form: the latency form has no trace path)
    if (mode == kModeStage && !a.tr_in && !a.tr_out &&
        a.e1 - a.e0 <= (g.lat_stage_n >= 0 ? g.lat_stage_n : stage_latency_max_n())) {
      if (grid <= 0) grid = grid_for(static_cast<long long>((a.e1 - a.e0 + 31) & ~31) * 4, 16);
      cudaError_t err = cudaSuccess;
      auto go = [&](auto k) {
        k<<<grid, kBlock, 0, s>>>(g, a);
        err = cudaGetLastError();
      };
      const int var = variant_of(mode, g, a);
      if (g.flux == kFluxRoe) with_instance4<kFluxRoe>(var, go); else with_instance4<kFluxLLF>(var, go);
      return err;
    }
  }
  if (grid <= 0) {
    // DMMA variant: one 8-element tile per warp; others: kG lanes per element
    const long long threads = kMma ? static_cast<long long>((a.e1 - a.e0 + 7) / 8) * 32
                                   : static_cast<long long>((a.e1 - a.e0 + 31) & ~31) * kG;
    grid = grid_for(threads, resident_blocks(mode), kThreads);
  }
  cudaError_t err = cudaSuccess;
  with_instance(g.flux, mode, variant_of(mode, g, a), [&](auto k) {
    k<<<grid, kThreads, kSmem, s>>>(g, a);
    err = cudaGetLastError();
  });
  return err;
}

template <>
cudaError_t Launch<DGB_P>::dt(int grid, const Geo& g, const double* c, Scalars* sc, int slot, unsigned long long seq,
                              cudaStream_t s) {
  static std::atomic<int> occ{0};
  int o = occ.load(std::memory_order_relaxed);
  if (!o) occ.store(o = occupancy(k_dt), std::memory_order_relaxed);
  if (grid <= 0) grid = grid_for(g.ld, o);
  k_dt<<<grid, kBlock, 0, s>>>(g, c, sc, slot, seq);
  return cudaGetLastError();
}

template <>
bool Launch<DGB_P>::trace_wanted(int n, const Geo& g) {
  if constexpr (!kTraceOK) {
    return false;
  } else if constexpr (kMma) {
    // (p=3 on the C3 vortex mesh, the boundary-code instance: 0.478 vs 0.509 ms per stage with the
    // 16-byte trace stores; 0.513 vs 0.505 before them)
    return true;
  } else {  // the one-thread kernel: not where the four-lane latency form serves the mesh
    return n > (g.lat_stage_n >= 0 ? g.lat_stage_n : stage_latency_max_n());
  }
}

}  // namespace dgbk
