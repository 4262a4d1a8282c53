// stencil-step kernels for radius r = 5 (space order 10)
#define SF_R 5
#include "inst_body.cuh"
