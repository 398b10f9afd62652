// Kernels for polynomial degree 3 (see kernels_tu.cuh).
#define DGB_P 3
#include "kernels_tu.cuh"
