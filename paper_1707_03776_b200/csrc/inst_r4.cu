// stencil-step kernels for radius r = 4 (space order 8)
#define SF_R 4
#include "inst_body.cuh"
