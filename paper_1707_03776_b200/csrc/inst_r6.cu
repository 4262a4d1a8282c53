// stencil-step kernels for radius r = 6 (space order 12)
#define SF_R 6
#include "inst_body.cuh"
