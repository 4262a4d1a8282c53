// stencil-step kernels for radius r = 1 (space order 2)
#define SF_R 1
#include "inst_body.cuh"
