// stencil-step kernels for radius r = 3 (space order 6)
#define SF_R 3
#include "inst_body.cuh"
