// Host-side launchers exported by the per-degree translation units.
#pragma once

#include <cuda_runtime.h>

#include "dg_kernels.cuh"

namespace dgbk {

constexpr int kBlock = 128;

template <int P>
struct Launch {
  static cudaError_t upload(const Tab<P>& t, cudaStream_t s);
  // grid = 0 -> occupancy-sized grid (one wave of resident blocks)
  static cudaError_t element(int mode, int grid, const Geo& g, const StageArgs& a, cudaStream_t s);
  static cudaError_t dt(int grid, const Geo& g, const double* c, Scalars* sc, int slot, unsigned long long seq,
                        cudaStream_t s);
  static int resident_blocks(int mode);  // blocks per SM for the element kernel
  static int lanes();                    // G (0 = DMMA tile kernel)
  static int trace_points();             // 3K when the stage kernel has trace-buffer instances, else 0
  static bool trace_wanted(int n, const Geo& g);  // trace mode pays for whole-mesh runs of n elements
  // DMMA fragment-ordered tables: size in doubles (0 when the degree does not use
  // the DMMA kernel); fills `out` when non-null
  static int mma_table(const Tab<P>& t, double* out);
  // Load every kernel instance of this degree now.  Under CUDA's lazy loading the first launch
  // of a function loads its module, which waits for the device; a partition whose peers are
  // spinning in a flag wait on other streams would then stall until their timeout.
  static cudaError_t preload();
};

cudaError_t upload_limtab(const LimTab& t, cudaStream_t s);
cudaError_t preload_limit();  // every limiter instance (see Launch::preload)
cudaError_t launch_limit(int grid, const Geo& g, const LimArgs& a, cudaStream_t s);
int limit_resident_blocks();
// Stage + limiter in one persistent launch (p = 1, whole-mesh contexts); grid <= 0: one
// wave of resident blocks, stage_limit_grid() (FuseArgs::lag counts it).
int stage_limit_grid();
cudaError_t launch_stage_limit(int grid, const Geo& g, const StageArgs& a, const LimArgs& la, const FuseArgs& f,
                               cudaStream_t s);

}  // namespace dgbk
