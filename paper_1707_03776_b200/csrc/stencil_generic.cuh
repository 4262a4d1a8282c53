// stencil_generic.cuh -- thread-per-point stencil step (2D and 3D, any extents).
//
// Used for 2D problems (BASELINE configs[0]), for 3D grids whose innermost extent is
// not a multiple of 4 (TMA needs 16-byte strides), and as an independent-structure
// cross-check of the TMA 2.5D kernel (same per-point arithmetic, stencil_common.cuh).
// Neighbours come straight from global memory through L1/L2 (__ldg); out-of-grid
// neighbours read as zero (zero ghost halo, reading C6).
#pragma once
#include "stencil_common.cuh"

template <int R, int MODE>
__global__ void __launch_bounds__(256)
k_generic3d(SfStepArgs a)
{
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t y = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    const int64_t n1st = a.xb - a.xa;
    const int64_t x = (blockIdx.z < n1st) ? a.xa + blockIdx.z : a.xa2 + (blockIdx.z - n1st);
    if (z >= a.n2 || y >= a.n1 || (blockIdx.z < n1st ? x >= a.xb : x >= a.xb2)) return;
    const int64_t sx = a.n1 * a.n2, sy = a.n2;
    const int64_t idx = (x * a.n1 + y) * a.n2 + z;
    const float *__restrict__ c = a.cur;
    const float u = __ldg(c + idx);
    float lap;
    if constexpr (sf_merged_form(R, MODE)) {
        float L = 0.0f;
#pragma unroll
        for (int k = 1; k <= R; ++k) {
            const float ym = (y - k >= 0) ? __ldg(c + idx - k * sy) : 0.0f;
            const float yp = (y + k < a.n1) ? __ldg(c + idx + k * sy) : 0.0f;
            const float zm = (z - k >= 0) ? __ldg(c + idx - k) : 0.0f;
            const float zp = (z + k < a.n2) ? __ldg(c + idx + k) : 0.0f;
            const float xm = (x - k >= 0) ? __ldg(c + idx - k * sx) : 0.0f;
            const float xp = (x + k < a.n0b) ? __ldg(c + idx + k * sx) : 0.0f;
            L = __fmaf_rn(a.w.w[k], sf_merged3(ym, yp, zm, zp, xm, xp, u), L);
        }
        lap = L;
    } else {
        float P = 0.0f, X = 0.0f;
#pragma unroll
        for (int k = 1; k <= R; ++k) {
            const float ym = (y - k >= 0) ? __ldg(c + idx - k * sy) : 0.0f;
            const float yp = (y + k < a.n1) ? __ldg(c + idx + k * sy) : 0.0f;
            const float zm = (z - k >= 0) ? __ldg(c + idx - k) : 0.0f;
            const float zp = (z + k < a.n2) ? __ldg(c + idx + k) : 0.0f;
            P = __fmaf_rn(a.w.w[k], sf_inplane3(ym, yp, zm, zp, u), P);
        }
#pragma unroll
        for (int k = 1; k <= R; ++k) {
            const float xm = (x - k >= 0) ? __ldg(c + idx - k * sx) : 0.0f;
            const float xp = (x + k < a.n0b) ? __ldg(c + idx + k * sx) : 0.0f;
            X = __fmaf_rn(a.w.w[k], sf_xterm(xm, xp, u), X);
        }
        lap = __fadd_rn(P, X);
    }
    const float old = a.out[idx];
    const float c3 = __ldg(a.c3 + idx);
    const float beta = a.beta ? __ldg(a.beta + idx)
                              : a.sigx ? sf_beta_sep(__ldg(a.sigx + x), __ldg(a.sigy + y), __ldg(a.sigz + z), a.hdt)
                                       : 1.0f;
    const float o = sf_update(u, old, beta, c3, lap);
    if (MODE == SF_MODE_GRAD) {
        const float S = sf_d2(u, old, beta, c3, lap);
        const float sn = a.snap_half ? __half2float(reinterpret_cast<const __half *>(a.snap_in)[idx])
                                     : __ldg(a.snap_in + idx);
        a.grad[idx] = sf_grad(a.grad[idx], a.gscale, sn, S);
    }
    a.out[idx] = o;
    if (x >= a.mq[0] && x < a.mq[1]) *sf_mirror(a.out + idx, a.md[0]) = o;      // peer halo (f1)
    else if (x >= a.mq[2] && x < a.mq[3]) *sf_mirror(a.out + idx, a.md[1]) = o;
    if (MODE == SF_MODE_SAVE) {
        if (a.snap_half) reinterpret_cast<__half *>(a.snap_out)[idx] = __float2half_rn(o);
        else a.snap_out[idx] = o;
    }
}

// 2D, layout [x][z] (n1 == 1 is not used: n1 holds the z extent here).
template <int R, int MODE>
__global__ void __launch_bounds__(256)
k_generic2d(SfStepArgs a)
{
    const int64_t z = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
    const int64_t n1st = a.xb - a.xa;
    const int64_t x = row < n1st ? a.xa + row : a.xa2 + (row - n1st);
    if (z >= a.n2 || (row < n1st ? x >= a.xb : x >= a.xb2)) return;
    const int64_t sx = a.n2;
    const int64_t idx = x * a.n2 + z;
    const float *__restrict__ c = a.cur;
    const float u = __ldg(c + idx);
    float P = 0.0f, X = 0.0f;
#pragma unroll
    for (int k = 1; k <= R; ++k) {
        const float zm = (z - k >= 0) ? __ldg(c + idx - k) : 0.0f;
        const float zp = (z + k < a.n2) ? __ldg(c + idx + k) : 0.0f;
        P = __fmaf_rn(a.w.w[k], sf_inplane2(zm, zp, u), P);
    }
#pragma unroll
    for (int k = 1; k <= R; ++k) {
        const float xm = (x - k >= 0) ? __ldg(c + idx - k * sx) : 0.0f;
        const float xp = (x + k < a.n0b) ? __ldg(c + idx + k * sx) : 0.0f;
        X = __fmaf_rn(a.w.w[k], sf_xterm(xm, xp, u), X);
    }
    const float lap = __fadd_rn(P, X);
    const float old = a.out[idx];
    const float c3 = __ldg(a.c3 + idx);
    // 2D separable damping: profiles of x and z (sigy unused: sy = 0 exactly)
    const float beta = a.beta ? __ldg(a.beta + idx)
                              : a.sigx ? sf_beta_sep(__ldg(a.sigx + x), 0.0f, __ldg(a.sigz + z), a.hdt)
                                       : 1.0f;
    const float o = sf_update(u, old, beta, c3, lap);
    if (MODE == SF_MODE_GRAD) {
        const float S = sf_d2(u, old, beta, c3, lap);
        const float sn = a.snap_half ? __half2float(reinterpret_cast<const __half *>(a.snap_in)[idx])
                                     : __ldg(a.snap_in + idx);
        a.grad[idx] = sf_grad(a.grad[idx], a.gscale, sn, S);
    }
    a.out[idx] = o;
    if (x >= a.mq[0] && x < a.mq[1]) *sf_mirror(a.out + idx, a.md[0]) = o;      // peer halo (f1)
    else if (x >= a.mq[2] && x < a.mq[3]) *sf_mirror(a.out + idx, a.md[1]) = o;
    if (MODE == SF_MODE_SAVE) {
        if (a.snap_half) reinterpret_cast<__half *>(a.snap_out)[idx] = __float2half_rn(o);
        else a.snap_out[idx] = o;
    }
}
