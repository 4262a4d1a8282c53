// loop2d.cuh -- the whole 2D time loop of a small grid in ONE launch (SF_OPT_LOOP2D).
//
// BASELINE configs[0] (141 x 141, 500 steps) is launch-bound as one kernel per step: each
// step is ~20 k point updates, ~1 us of work behind a few us of launch and record overhead
// (3.8-4.1 GPts/s even with CUDA-graph replay).  Here a thread-block CLUSTER of SF_LOOP2D_CTAS
// CTAs runs every step of sf_forward / sf_adjoint (PLAIN mode: no snapshots, no gradient):
// CTA c owns a slab of x-rows and keeps both wavefield levels of it (and its c3 / beta) in
// shared memory; the stencil reads the neighbouring slabs' rows straight from the
// neighbours' shared memory (distributed shared memory), and one cluster barrier per phase
// orders the steps:
//   stencil of the own rows (new level over the old one, zero ghost halo) -> CTA barrier
//   -> injection of this step's values into own-row targets (CSR by target, fixed order)
//   -> cluster barrier -> records of the new level (corners read from whichever CTA owns
//      them), concurrent with the next step's stencil (which only reads the new level).
// Every operation is the per-point arithmetic of k_generic2d / k_inject / k_interp_ell (the
// same helper functions, the same order), so the results are bitwise those of the per-step
// kernels (tests/test_gpu_parity.py::test_loop2d_bitwise).
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>
#include "stencil_common.cuh"

#ifndef SF_LOOP2D_CTAS
#define SF_LOOP2D_CTAS 16       // cluster size (non-portable maximum)
#endif
#define SF_LOOP2D_THREADS 512
#define SF_LOOP2D_SMEM_MAX (200 * 1024)
#define SF_LOOP2D_LOC 1024      // injection targets one CTA can hold

struct Loop2dArgs {
    int n0, n2;                // grid [x][z]
    int rpc;                   // rows per CTA (the last CTA may hold fewer, >= 0)
    int nsteps;                // time steps (nt - 1)
    int backward;              // 0: forward (step s injects row s, records row s + 1);
                               // 1: adjoint (step s injects row nt-1-s, records row nt-2-s)
    int nt;
    SfWeights w;
    const float *c3, *beta;    // hoisted coefficients (beta may be NULL)
    const float *sigx, *sigz;  // separable damping profiles (or NULL)
    float hdt;
    float *A, *B;              // state: in (level before, level), out (second-last, last)
    // injection (CSR by target) of vals [nt][nvals]
    int ntgt;
    const int64_t *tgt;
    const int *rowptr, *pt;
    const float *coef, *vals;
    int nvals;
    // records (ELL, K slots x np, zero weights skipped) into rec [nt][np]
    int np, K;
    const int64_t *eidx;
    const float *ew;
    float *rec;
};

// shared-memory layout of one CTA: level buffers L0, L1 [rpc][n2], c3 [rpc][n2], beta [rpc][n2],
// then the CTA's injection targets (local index, CSR range, this step's increment)
__host__ __device__ inline size_t loop2d_smem(int rpc, int n2, bool beta)
{
    return sizeof(float) * (size_t)rpc * (size_t)n2 * (beta ? 4 : 3) + 4 * sizeof(int) * SF_LOOP2D_LOC + 16;
}

template <int R>
__global__ void __launch_bounds__(SF_LOOP2D_THREADS, 1) k_loop2d(const Loop2dArgs a)
{
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ float sm[];
    const int me = (int)cl.block_rank();
    const int n0 = a.n0, n2 = a.n2, rpc = a.rpc;
    const int x0 = me * rpc, x1 = min(n0, x0 + rpc);
    const int M = rpc * n2;
    float *L0 = sm, *L1 = sm + M, *C3 = sm + 2 * M, *BE = sm + 3 * M;
    for (int i = threadIdx.x; i < (x1 - x0) * n2; i += blockDim.x) {
        const int64_t g = (int64_t)x0 * n2 + i;
        L0[i] = a.A[g];
        L1[i] = a.B[g];
        C3[i] = a.c3[g];
        if (a.beta) BE[i] = a.beta[g];
    }
    // this CTA's injection targets (its own rows)
    int *tl = reinterpret_cast<int *>(sm + (a.beta ? 4 : 3) * M);  // [LOC] local index
    int *te0 = tl + SF_LOOP2D_LOC, *te1 = te0 + SF_LOOP2D_LOC;     // CSR entry range
    float *td = reinterpret_cast<float *>(te1 + SF_LOOP2D_LOC);    // this step's increment
    int *cnt = reinterpret_cast<int *>(td + SF_LOOP2D_LOC);
    if (threadIdx.x == 0) *cnt = 0;
    __syncthreads();
    if (a.vals)
        for (int t = threadIdx.x; t < a.ntgt; t += blockDim.x) {
            const int64_t g = a.tgt[t];
            const int x = (int)(g / n2);
            if (x < x0 || x >= x1) continue;
            const int k = atomicAdd(cnt, 1);  // list order is immaterial: one target per entry
            tl[k] = (x - x0) * n2 + (int)(g - (int64_t)x * n2);
            te0[k] = a.rowptr[t];
            te1[k] = a.rowptr[t + 1];
        }
    cl.sync();
    const int nloc = *cnt;
    // level `lv` (0: L0, 1: L1) of global row x, column z, from whichever CTA owns it
    auto at = [&](int lv, int x, int z) -> float {
        const int o = x / rpc;
        const float *base = (lv ? L1 : L0) + (x - o * rpc) * n2 + z;
        return o == me ? *base : *cl.map_shared_rank(base, o);
    };
    auto records = [&](int lv, int row) {
        if (!a.rec) return;  // point p is interpolated by CTA p % CTAS
        for (int p = me + SF_LOOP2D_CTAS * (int)threadIdx.x; p < a.np; p += SF_LOOP2D_CTAS * (int)blockDim.x) {
            float acc = 0.0f;
            for (int c = 0; c < a.K; ++c) {
                const float w = a.ew[(int64_t)c * a.np + p];
                if (w != 0.0f) {
                    const int64_t g = a.eidx[(int64_t)c * a.np + p];
                    acc = __fmaf_rn(w, at(lv, (int)(g / n2), (int)(g % n2)), acc);
                }
            }
            a.rec[(int64_t)row * a.np + p] = acc;
        }
    };
    records(1, a.backward ? a.nt - 1 : 0);
    int lc = 1;  // level buffer holding the current level
    for (int s = 0; s < a.nsteps; ++s) {
        const float *cur = lc ? L1 : L0;
        float *out = lc ? L0 : L1;
        // this step's increments do not depend on the wavefield: formed first, so their global
        // loads overlap the stencil (the k_inject arithmetic, CSR order)
        if (nloc > 0) {
            const float *vrow = a.vals + (int64_t)(a.backward ? a.nt - 1 - s : s) * a.nvals;
            for (int i = threadIdx.x; i < nloc; i += blockDim.x) {
                float d = 0.0f;
                for (int e = te0[i]; e < te1[i]; ++e) d = __fmaf_rn(a.coef[e], vrow[a.pt[e]], d);
                td[i] = d;
            }
        }
        // ---- stencil of the own rows: the k_generic2d arithmetic (warp per row, lanes on z)
        for (int x = x0 + (int)(threadIdx.x >> 5); x < x1; x += SF_LOOP2D_THREADS / 32) {
            for (int z = threadIdx.x & 31; z < n2; z += 32) {
                const int li = (x - x0) * n2 + z;
                const float u = cur[li];
                float P = 0.0f, X = 0.0f;
#pragma unroll
                for (int k = 1; k <= R; ++k) {
                    const float zm = (z - k >= 0) ? cur[li - k] : 0.0f;
                    const float zp = (z + k < n2) ? cur[li + k] : 0.0f;
                    P = __fmaf_rn(a.w.w[k], sf_inplane2(zm, zp, u), P);
                }
#pragma unroll
                for (int k = 1; k <= R; ++k) {
                    const float xm = (x - k >= 0) ? ((x - k >= x0) ? cur[li - k * n2] : at(lc, x - k, z)) : 0.0f;
                    const float xp = (x + k < n0) ? ((x + k < x1) ? cur[li + k * n2] : at(lc, x + k, z)) : 0.0f;
                    X = __fmaf_rn(a.w.w[k], sf_xterm(xm, xp, u), X);
                }
                const float lap = __fadd_rn(P, X);
                const float beta = a.beta ? BE[li]
                                          : a.sigx ? sf_beta_sep(__ldg(a.sigx + x), 0.0f, __ldg(a.sigz + z), a.hdt)
                                                   : 1.0f;
                out[li] = sf_update(u, out[li], beta, C3[li], lap);
            }
        }
        // the own rows' targets only need this CTA's stencil results
        __syncthreads();
        // ---- injection of this step's values into own-row targets
        for (int i = threadIdx.x; i < nloc; i += blockDim.x) out[tl[i]] = __fadd_rn(out[tl[i]], td[i]);
        // the new level is final: the neighbours may read it (next stencil, records), and the
        // old one is no longer read by anyone (it is overwritten by the next step)
        cl.sync();
        lc ^= 1;
        // ---- records of the new level (overlap the next stencil, which only reads it)
        records(lc, a.backward ? a.nt - 2 - s : s + 1);
    }
    cl.sync();
    // state out: (second-last level, last level)
    const float *last = lc ? L1 : L0, *prev = lc ? L0 : L1;
    for (int i = threadIdx.x; i < (x1 - x0) * n2; i += blockDim.x) {
        const int64_t g = (int64_t)x0 * n2 + i;
        a.A[g] = prev[i];
        a.B[g] = last[i];
    }
}
