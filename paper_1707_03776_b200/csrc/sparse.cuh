// sparse.cuh -- sparse-point kernels (injection, interpolation), residual/objective,
// and the small setup kernels (coefficient hoisting, min reduction, state swap).
//
//   interpolate (reading C11):
//       out[p] = sum_c W_{p,c} u[idx_{p,c}]        corners in fixed order, zero weights skipped
//   inject (readings C3, C9):
//       u[t] += delta_t,  delta_t = sum_{e in row t} coef_e * vals[pt_e],  coef_e = W_e dt^2/m[t]
//     as a deterministic CSR gather by target grid point (no atomics: bitwise reproducible,
//     SPEC.md:228 rationale).  Fused patches:
//       save step:      snap[t] += delta_t              (snapshot taken before injection)
//       gradient step:  grad[t] -= gscale * snap_n[t] * delta_t   (completes the in-kernel
//                       correlation, which saw v^{n-1} before injection)
//   residual (BASELINE configs[2]): res = d_syn - d_obs, J = 1/2 sum res^2 (fp64, fixed order)
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "stencil_common.cuh"

// snapshot element access: fp32, or fp16 (SF_OPT_SNAP_HALF, reading C23: round to nearest
// even on store, exact widening on load)
__device__ __forceinline__ float snap_ld(const void *s, int64_t i, int half)
{
    return half ? __half2float(static_cast<const __half *>(s)[i]) : static_cast<const float *>(s)[i];
}
__device__ __forceinline__ void snap_st(void *s, int64_t i, float v, int half)
{
    if (half) static_cast<__half *>(s)[i] = __float2half_rn(v);
    else static_cast<float *>(s)[i] = v;
}

__global__ void k_interp(const float *__restrict__ u, const int64_t *__restrict__ idx,
                         const float *__restrict__ W, const int *__restrict__ owned, int np, int nc,
                         float *__restrict__ out)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    float acc = 0.0f;
    for (int c = 0; c < nc; ++c) {
        const float w = W[(int64_t)p * nc + c];
        if (w != 0.0f) acc = __fmaf_rn(w, u[idx[(int64_t)p * nc + c]], acc);
    }
    out[p] = owned ? (owned[p] ? acc : 0.0f) : acc;
}

// Same sum from ELL tables: K slots per point stored slot-major ([K][np], coalesced),
// holding the point's nonzero corners in corner order (zero-padded).  Bitwise equal to
// k_interp (same nonzero terms, same order).
__global__ void k_interp_ell(const float *__restrict__ u, const int64_t *__restrict__ idx,
                             const float *__restrict__ W, const int *__restrict__ owned, int np, int K,
                             float *__restrict__ out)
{
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (int c = 0; c < K; ++c) {
            const float w = W[(int64_t)c * np + p];
            if (w != 0.0f) acc = __fmaf_rn(w, __ldcg(u + idx[(int64_t)c * np + p]), acc);
        }
        out[p] = owned ? (owned[p] ? acc : 0.0f) : acc;
    }
}

// Injection from ELL tables ([K][ntgt] slot-major, zero coefficients pad): bitwise equal
// to k_inject (same terms, same order).
__global__ void k_inject_ell(float *__restrict__ u, const int64_t *__restrict__ tgt, int K,
                             const int *__restrict__ ept, const float *__restrict__ ecoef, int ntgt,
                             const float *__restrict__ vals, void *__restrict__ snap_patch,
                             const void *__restrict__ grad_snap, float *__restrict__ grad, float gscale,
                             int snap_half)
{
    sf_pdl_wait();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntgt) return;
    const int64_t g = tgt[t];
    float d = 0.0f;
    for (int c = 0; c < K; ++c) {
        const float cf = ecoef[(int64_t)c * ntgt + t];
        if (cf != 0.0f) d = __fmaf_rn(cf, vals[ept[(int64_t)c * ntgt + t]], d);
    }
    const float un = __fadd_rn(u[g], d);
    u[g] = un;
    // save step: the snapshot holds the new level after injection (== snap + d in fp32)
    if (snap_patch) snap_st(snap_patch, g, un, snap_half);
    if (grad) grad[g] = __fmaf_rn(-gscale, __fmul_rn(snap_ld(grad_snap, g, snap_half), d), grad[g]);
}

// peer-store halo exchange (SF_OPT_P2P): a target in plane [mq[0], mq[1]) / [mq[2], mq[3])
// also writes its final value at byte offset md[0] / md[1] (the neighbour's halo)
struct SfMirror {
    int64_t plane;   // points per x-plane
    int64_t mq[4];
    int64_t md[2];
};

// k_inject_ell restricted to a list of target rows (split boundary / interior launches)
__global__ void k_inject_ell_list(float *__restrict__ u, const int64_t *__restrict__ tgt, int K,
                                  const int *__restrict__ ept, const float *__restrict__ ecoef, int ntgt,
                                  const int *__restrict__ list, int nl, const float *__restrict__ vals,
                                  void *__restrict__ snap_patch, const void *__restrict__ grad_snap,
                                  float *__restrict__ grad, float gscale, int snap_half, SfMirror mir)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    const int t = list[i];
    const int64_t g = tgt[t];
    float d = 0.0f;
    for (int c = 0; c < K; ++c) {
        const float cf = ecoef[(int64_t)c * ntgt + t];
        if (cf != 0.0f) d = __fmaf_rn(cf, vals[ept[(int64_t)c * ntgt + t]], d);
    }
    const float un = __fadd_rn(u[g], d);
    u[g] = un;
    const int64_t q = g / mir.plane;
    if (q >= mir.mq[0] && q < mir.mq[1]) *reinterpret_cast<float *>(reinterpret_cast<char *>(u + g) + mir.md[0]) = un;
    else if (q >= mir.mq[2] && q < mir.mq[3]) *reinterpret_cast<float *>(reinterpret_cast<char *>(u + g) + mir.md[1]) = un;
    // save step: the snapshot holds the new level after injection (== snap + d in fp32)
    if (snap_patch) snap_st(snap_patch, g, un, snap_half);
    if (grad) grad[g] = __fmaf_rn(-gscale, __fmul_rn(snap_ld(grad_snap, g, snap_half), d), grad[g]);
}

// k_inject restricted to a list of target rows (split launches when some target has more
// than 8 contributions, i.e. no ELL table): the same terms in the same order as k_inject
__global__ void k_inject_csr_list(float *__restrict__ u, const int64_t *__restrict__ tgt,
                                  const int *__restrict__ rowptr, const int *__restrict__ ent_pt,
                                  const float *__restrict__ ent_coef, const int *__restrict__ list, int nl,
                                  const float *__restrict__ vals, void *__restrict__ snap_patch,
                                  const void *__restrict__ grad_snap, float *__restrict__ grad, float gscale,
                                  int snap_half, SfMirror mir)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nl) return;
    const int t = list[i];
    float d = 0.0f;
    for (int e = rowptr[t]; e < rowptr[t + 1]; ++e) d = __fmaf_rn(ent_coef[e], vals[ent_pt[e]], d);
    const int64_t g = tgt[t];
    const float un = __fadd_rn(u[g], d);
    u[g] = un;
    const int64_t q = g / mir.plane;
    if (q >= mir.mq[0] && q < mir.mq[1]) *reinterpret_cast<float *>(reinterpret_cast<char *>(u + g) + mir.md[0]) = un;
    else if (q >= mir.mq[2] && q < mir.mq[3]) *reinterpret_cast<float *>(reinterpret_cast<char *>(u + g) + mir.md[1]) = un;
    if (snap_patch) snap_st(snap_patch, g, un, snap_half);
    if (grad) grad[g] = __fmaf_rn(-gscale, __fmul_rn(snap_ld(grad_snap, g, snap_half), d), grad[g]);
}

// CSR -> ELL (slot-major) for the injection tables
__global__ void k_csr_to_ell(const int *__restrict__ rowptr, const int *__restrict__ pt,
                             const float *__restrict__ coef, int ntgt, int K, int *__restrict__ ept,
                             float *__restrict__ ecoef)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntgt) return;
    const int b = rowptr[t], n = rowptr[t + 1] - b;
    for (int c = 0; c < K; ++c) {
        ept[(int64_t)c * ntgt + t] = c < n ? pt[b + c] : 0;
        ecoef[(int64_t)c * ntgt + t] = c < n ? coef[b + c] : 0.0f;
    }
}

__global__ void k_inject(float *__restrict__ u, const int64_t *__restrict__ tgt,
                         const int *__restrict__ rowptr, const int *__restrict__ ent_pt,
                         const float *__restrict__ ent_coef, int ntgt,
                         const float *__restrict__ vals, void *__restrict__ snap_patch,
                         const void *__restrict__ grad_snap, float *__restrict__ grad, float gscale,
                         int snap_half)
{
    sf_pdl_wait();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntgt) return;
    float d = 0.0f;
    for (int e = rowptr[t]; e < rowptr[t + 1]; ++e) d = __fmaf_rn(ent_coef[e], vals[ent_pt[e]], d);
    const int64_t g = tgt[t];
    const float un = __fadd_rn(u[g], d);
    u[g] = un;
    // save step: the snapshot holds the new level after injection (== snap + d in fp32)
    if (snap_patch) snap_st(snap_patch, g, un, snap_half);
    if (grad) grad[g] = __fmaf_rn(-gscale, __fmul_rn(snap_ld(grad_snap, g, snap_half), d), grad[g]);
}

// coef_e = W_e * dt^2 / m[t_e], computed in fp64, rounded once
__global__ void k_inject_coef(const float *__restrict__ m, const int64_t *__restrict__ ent_tgt,
                              const double *__restrict__ ent_w, int ne, double dt2,
                              float *__restrict__ coef)
{
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    coef[e] = (float)(ent_w[e] * dt2 / (double)m[ent_tgt[e]]);
}

// hoisted per-point coefficients: A = m + eta dt/2, beta = (m - eta dt/2)/A, c3 = dt^2/A (fp64)
__global__ void k_hoist(const float *__restrict__ m, const float *__restrict__ damp, int64_t n,
                        double dt, float *__restrict__ c3, float *__restrict__ beta)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double mm = m[i];
        const double e = damp ? (double)damp[i] : 0.0;
        const double A = mm + 0.5 * e * dt;
        c3[i] = (float)(dt * dt / A);
        if (beta) beta[i] = (float)((mm - 0.5 * e * dt) / A);
    }
}

// fp32 level -> fp16 snapshot slot (slot 0 of a forward with SF_OPT_SNAP_HALF)
__global__ void k_f32_to_f16(__half *__restrict__ dst, const float *__restrict__ src, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = __float2half_rn(src[i]);
}

// hoisted c3 with separable damping (sf_desc.sigma, reading C7): eta = m sigma,
// sigma = sx[x] + sy[y] + sz[z] (fp64), A = m + eta dt/2, c3 = dt^2/A; beta is regenerated
// in the stencil kernels (sf_beta_sep).  2D: n1 == 1 and sy == NULL.
__global__ void k_hoist_sep(const float *__restrict__ m, int64_t n, int64_t n1, int64_t n2, double dt,
                            const float *__restrict__ sx, const float *__restrict__ sy,
                            const float *__restrict__ sz, float *__restrict__ c3)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i / (n1 * n2), y = (i / n2) % n1, z = i % n2;
        const double sig = (double)sx[x] + (sy ? (double)sy[y] : 0.0) + (double)sz[z];
        const double mm = m[i];
        const double A = mm + 0.5 * (mm * sig) * dt;
        c3[i] = (float)(dt * dt / A);
    }
}

// min over a float array (positive floats order like their bit patterns; non-positive
// values and NaN are reported through the flag)
__global__ void k_min_m(const float *__restrict__ m, int64_t n, unsigned int *__restrict__ minbits,
                        int *__restrict__ bad)
{
    unsigned int loc = 0x7f7fffffu;
    int b = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float v = m[i];
        if (!(v > 0.0f) || !(v < 3.0e38f)) b = 1;
        else loc = min(loc, __float_as_uint(v));
    }
    for (int o = 16; o; o >>= 1) {
        loc = min(loc, __shfl_xor_sync(0xffffffffu, loc, o));
        b |= __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(minbits, loc);
        if (b) atomicOr(bad, 1);
    }
}

// res = a - b ; per-block fp64 partial sums of res^2 (fixed tree order)
__global__ void k_residual(const float *__restrict__ a, const float *__restrict__ b,
                           float *__restrict__ res, int64_t n, double *__restrict__ partial)
{
    __shared__ double sh[256];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float r = __fsub_rn(a[i], b[i]);
        res[i] = r;
        acc += (double)r * (double)r;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_sum_partials(const double *__restrict__ partial, int n, double *__restrict__ out)
{
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += partial[i];
        *out = 0.5 * s;
    }
}

// elementwise swap of two arrays (restores the (u^{nt-2}, u^{nt-1}) output order)
__global__ void k_swap(float *__restrict__ a, float *__restrict__ b, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float t = a[i];
        a[i] = b[i];
        b[i] = t;
    }
}
