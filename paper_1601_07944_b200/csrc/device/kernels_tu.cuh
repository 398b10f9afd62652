// One translation unit per polynomial degree: its constant bank, the four
// element-kernel modes and the CFL kernel.  Included by kernels_pN.cu with
// DGB_P defined.
#include "element_impl.cuh"
#include "launch.hpp"

namespace dgbk {

// Everything in this unit is internal: each degree has its own constant bank
// and its own kernel instances.
namespace {
__constant__ Tab<DGB_P> c_tab;
constexpr int kG = Lanes<DGB_P>::value;  // lanes per element

template <int MODE>
__global__ void __launch_bounds__(kBlock, MinBlocks<DGB_P>::value) k_element(Geo geo, StageArgs a) {
  if constexpr (kG == 1)
    element_body_g1<DGB_P, MODE>(c_tab, geo, a);
  else
    element_body<DGB_P, MODE>(c_tab, geo, a);
}

__global__ void __launch_bounds__(kBlock) k_dt(Geo geo, const double* __restrict__ c, Scalars* sc, int slot,
                                               unsigned long long seq) {
  dt_body<DGB_P>(c_tab, geo, c, sc, slot, seq);
}

int g_sms = 0;
int sm_count() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_sms;
}
template <class Kern>
int occupancy(Kern k) {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, kBlock, 0);
  return n > 0 ? n : 1;
}
int grid_for(long long threads, int blocks_per_sm) {
  const long long need = (threads + kBlock - 1) / kBlock;
  const long long cap = static_cast<long long>(blocks_per_sm) * sm_count();
  return static_cast<int>(need < cap ? need : cap);
}
}  // namespace

template <>
cudaError_t Launch<DGB_P>::upload(const Tab<DGB_P>& t, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(c_tab, &t, sizeof(t), 0, cudaMemcpyHostToDevice, s);
}

template <>
int Launch<DGB_P>::resident_blocks(int mode) {
  static int cache[4] = {0, 0, 0, 0};
  if (!cache[mode]) {
    switch (mode) {
      case kModeVolume: cache[mode] = occupancy(k_element<kModeVolume>); break;
      case kModeSurface: cache[mode] = occupancy(k_element<kModeSurface>); break;
      case kModeRhs: cache[mode] = occupancy(k_element<kModeRhs>); break;
      default: cache[mode] = occupancy(k_element<kModeStage>); break;
    }
  }
  return cache[mode];
}

template <>
int Launch<DGB_P>::lanes() {
  return kG;
}

template <>
cudaError_t Launch<DGB_P>::element(int mode, int grid, const Geo& g, const StageArgs& a, cudaStream_t s) {
  if (a.e1 <= a.e0) return cudaSuccess;
  if (grid <= 0) grid = grid_for(static_cast<long long>((a.e1 - a.e0 + 31) & ~31) * kG, resident_blocks(mode));
  switch (mode) {
    case kModeVolume: k_element<kModeVolume><<<grid, kBlock, 0, s>>>(g, a); break;
    case kModeSurface: k_element<kModeSurface><<<grid, kBlock, 0, s>>>(g, a); break;
    case kModeRhs: k_element<kModeRhs><<<grid, kBlock, 0, s>>>(g, a); break;
    default: k_element<kModeStage><<<grid, kBlock, 0, s>>>(g, a); break;
  }
  return cudaGetLastError();
}

template <>
cudaError_t Launch<DGB_P>::dt(int grid, const Geo& g, const double* c, Scalars* sc, int slot, unsigned long long seq,
                              cudaStream_t s) {
  static int occ = 0;
  if (!occ) occ = occupancy(k_dt);
  if (grid <= 0) grid = grid_for(g.ld, occ);
  k_dt<<<grid, kBlock, 0, s>>>(g, c, sc, slot, seq);
  return cudaGetLastError();
}

}  // namespace dgbk
