// Kernels for polynomial degree 4 (see kernels_tu.cuh).
#define DGB_P 4
#include "kernels_tu.cuh"
