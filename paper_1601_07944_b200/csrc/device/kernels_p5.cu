// Kernels for polynomial degree 5 (see kernels_tu.cuh).
#define DGB_P 5
#include "kernels_tu.cuh"
