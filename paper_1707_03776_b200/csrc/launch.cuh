// launch.cuh -- per-radius launchers for the stencil-step kernels (one translation unit
// per radius r = space_order/2, compiled in parallel; see inst_body.cuh).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include "stencil_common.cuh"

enum SfVariant { SF_VAR_AUTO = 0, SF_VAR_GENERIC = 1, SF_VAR_TMA = 2 };

struct SfTmaMaps {
    CUtensorMap cur, old, c3, beta, snap, grad;
};

struct SfLaunch {
    int ndim;
    int variant;      // SF_VAR_GENERIC or SF_VAR_TMA (resolved)
    int vy;           // TMA: rows per thread, 2 (14-row tiles) or 1 (7-row tiles)
    int ctas;         // TMA: persistent CTAs (0 = one per SM)
    int sms;          // multiprocessors of the device
    int damp;         // SfDampMode: none, beta array, separable profiles
    int mode;         // SfMode
    int snap_slot;    // GRAD: snapshot slot for the 4D snapshot tensor map
    int lz;           // TMA lane layout: 32 (128-column tiles) or 8 (narrow 32-column tiles)
    int pdl;          // launch with programmatic stream serialisation (SF_OPT_PDL)
    int balance;      // TMA work split: 0 (tile, x-chunk) items, 1 balanced contiguous (SF_OPT_BALANCE)
    const SfTmaMaps *maps;
};

// shared-memory bytes of the TMA kernel for (r, vy, damp, mode); 0 if unsupported
int sf_tma_smem_bytes(int r, int vy, int damp, int mode);

#define SF_DECL_LAUNCH(R) \
    cudaError_t sf_launch_step_r##R(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st);
SF_DECL_LAUNCH(1)
SF_DECL_LAUNCH(2)
SF_DECL_LAUNCH(3)
SF_DECL_LAUNCH(4)
SF_DECL_LAUNCH(5)
SF_DECL_LAUNCH(6)
SF_DECL_LAUNCH(7)
SF_DECL_LAUNCH(8)
#undef SF_DECL_LAUNCH

struct Loop2dArgs;
#define SF_DECL_LOOP(R) cudaError_t sf_launch_loop2d_r##R(const Loop2dArgs &a, cudaStream_t st);
SF_DECL_LOOP(1)
SF_DECL_LOOP(2)
SF_DECL_LOOP(3)
SF_DECL_LOOP(4)
SF_DECL_LOOP(5)
SF_DECL_LOOP(6)
SF_DECL_LOOP(7)
SF_DECL_LOOP(8)
#undef SF_DECL_LOOP

// two steps per pass (temporal blocking, stencil_tb2.cuh), r <= 4
struct TbArgs {
    int n0, n1, n2;
    SfWeights w;
    const float *c3, *beta;    // step 2's coefficients (beta NULL: no damping array)
    float *o1, *o2;            // u^{n+1}, u^{n+2}
    int chunk, nchunk;
    // fused injection: per tile, entries [beg[tile], beg[tile + 1]) sorted by plane:
    // plane e_q, position e_p = ey * 128 + ec in the grown tile, CSR row e_t
    const int *beg, *e_q, *e_p, *e_t;
    const int *rowptr, *pt;
    const float *coef;
    const float *vals1, *vals2;  // source values of step 1 / step 2 (NULL: none)
};

#define SF_DECL_TB(R) cudaError_t sf_launch_tb2_r##R(const SfTmaMaps &m, const TbArgs &a, int ctas, cudaStream_t st);
SF_DECL_TB(1)
SF_DECL_TB(2)
SF_DECL_TB(3)
SF_DECL_TB(4)
#undef SF_DECL_TB

#define SF_DECL_SMEM(R) int sf_tma_smem_r##R(int vy, int damp, int mode);
SF_DECL_SMEM(1)
SF_DECL_SMEM(2)
SF_DECL_SMEM(3)
SF_DECL_SMEM(4)
SF_DECL_SMEM(5)
SF_DECL_SMEM(6)
SF_DECL_SMEM(7)
SF_DECL_SMEM(8)
#undef SF_DECL_SMEM
