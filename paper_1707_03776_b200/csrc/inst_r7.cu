// stencil-step kernels for radius r = 7 (space order 14)
#define SF_R 7
#include "inst_body.cuh"
