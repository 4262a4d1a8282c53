// stencil-step kernels for radius r = 8 (space order 16)
#define SF_R 8
#include "inst_body.cuh"
