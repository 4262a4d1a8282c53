// stencil-step kernels for radius r = 2 (space order 4)
#define SF_R 2
#include "inst_body.cuh"
