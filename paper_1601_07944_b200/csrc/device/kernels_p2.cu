// Kernels for polynomial degree 2 (see kernels_tu.cuh).
#define DGB_P 2
#include "kernels_tu.cuh"
