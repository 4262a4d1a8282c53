// cfd2d.cu -- the paper's two other example workloads on the GPU:
//   linear 2D convection, Eq. 2 (reading C21), and the Laplace equation by
//   Jacobi sweeps, Eq. 4 with the boundary rows of the listing and
//   its l1 stopping rule (reading C22).
//
// Both are tiny 2D stencils in the paper (81^2 / 31^2).  A grid that fits in shared memory
// (both levels, <= SF_CFD_SMEM_PTS points) runs the whole time loop / iteration in ONE
// CTA: both buffers in shared memory, __syncthreads between steps, the l1 norm reduced in
// fp64 in a fixed order -- no launch per step, no host round trip per sweep.  Larger grids:
// convection launches one grid-stride kernel per step; Laplace runs ONE cooperative
// persistent kernel over all SMs with four grid-wide barriers per sweep (after the sweep,
// the boundary rows, the l1 partials and the l1 decision), so the convergence test never
// leaves the device.
//
// Boundary rows of P:411-414 in one pass: the listing's sequential order (rows p[x,0]=0,
// p[x,n1-1]=bc[x], then columns p[0,y]=p[1,y], p[n0-1,y]=p[n0-2,y]) gives the corners
// p[0,0]=p[n0-1,0]=0, p[0,n1-1]=bc[1], p[n0-1,n1-1]=bc[n0-2] and the column copies of the
// interior rows only -- written directly, every value is the one the sequence produces.
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "sf_internal.h"

namespace {

constexpr int SF_CFD_THREADS = 1024;
constexpr int64_t SF_CFD_SMEM_PTS = 25600;  // 2 levels x 25600 x 4 B = 200 KB
constexpr int64_t SF_LAP_ONE_CTA_PTS = 4096;  // Laplace: one CTA up to 64^2, all SMs above

// Eq. 2 at one interior point, in the oracle's operation order (reading C21)
__device__ __forceinline__ float conv_point(float u, float ul, float ud, float a, float b)
{
    const float t1 = __fmul_rn(a, __fsub_rn(u, ul));
    const float t2 = __fmul_rn(b, __fsub_rn(u, ud));
    return __fsub_rn(__fsub_rn(u, t1), t2);
}

__global__ void __launch_bounds__(SF_CFD_THREADS)
k_conv2d_smem(float *__restrict__ u, int n0, int n1, float a, float b, int nt)
{
    extern __shared__ float sm[];
    const int N = n0 * n1;
    float *A = sm, *B = sm + N;
    for (int k = threadIdx.x; k < N; k += blockDim.x) A[k] = B[k] = u[k];
    __syncthreads();
    for (int t = 0; t < nt; ++t) {
        for (int k = threadIdx.x; k < N; k += blockDim.x) {
            const int i = k / n1, j = k - i * n1;
            if (i > 0 && i < n0 - 1 && j > 0 && j < n1 - 1)
                B[k] = conv_point(A[k], A[k - n1], A[k - 1], a, b);
        }
        __syncthreads();
        float *T = A;
        A = B;
        B = T;
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x) u[k] = A[k];
}

__global__ void k_conv2d_step(const float *__restrict__ un, float *__restrict__ u, int64_t n0, int64_t n1,
                              float a, float b)
{
    const int64_t N = n0 * n1;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = k / n1, j = k - i * n1;
        u[k] = (i > 0 && i < n0 - 1 && j > 0 && j < n1 - 1) ? conv_point(un[k], un[k - n1], un[k - 1], a, b) : un[k];
    }
}

// Eq. 4 at one interior point (reading C22): (cx (pn_{i+1} + pn_{i-1}) + cy (pn_{j+1} + pn_{j-1})) / den
__device__ __forceinline__ float jacobi_point(const float *pn, int64_t k, int64_t n1, float cx, float cy, float den)
{
    const float s1 = __fadd_rn(pn[k + n1], pn[k - n1]);
    const float s2 = __fadd_rn(pn[k + 1], pn[k - 1]);
    return __fdiv_rn(__fadd_rn(__fmul_rn(cx, s1), __fmul_rn(cy, s2)), den);
}

// fixed-order block reduction of two fp64 sums (deterministic): warp shuffles, then the
// warp totals in warp order; red: >= 64 doubles of shared memory
__device__ void block_sum2(double &a, double &b, double *red)
{
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
    }
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[w] = a;
        red[32 + w] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0;
        for (int i = 0; i < nw; ++i) {
            x += red[i];
            y += red[32 + i];
        }
        red[0] = x;
        red[32] = y;
    }
    __syncthreads();
    a = red[0];
    b = red[32];
    __syncthreads();
}

// boundary rows of P:411-414 at index e of the combined boundary pass (see the header):
// e < n0 - 2: rows of interior x; then n1 - 2 column copies; then the 4 corners
__device__ __forceinline__ void laplace_boundary(float *p, const float *bc, int64_t e, int64_t n0, int64_t n1)
{
    if (e < n0 - 2) {
        const int64_t i = e + 1;
        p[i * n1] = 0.0f;
        p[i * n1 + n1 - 1] = bc[i];
    } else if (e < (n0 - 2) + (n1 - 2)) {
        const int64_t j = e - (n0 - 2) + 1;
        p[j] = p[n1 + j];
        p[(n0 - 1) * n1 + j] = p[(n0 - 2) * n1 + j];
    } else if (e < (n0 - 2) + (n1 - 2) + 4) {
        const int c = (int)(e - (n0 - 2) - (n1 - 2));
        if (c == 0) p[0] = 0.0f;
        if (c == 1) p[n1 - 1] = bc[1];
        if (c == 2) p[(n0 - 1) * n1] = 0.0f;
        if (c == 3) p[(n0 - 1) * n1 + n1 - 1] = bc[n0 - 2];
    }
}

__global__ void __launch_bounds__(SF_CFD_THREADS)
k_laplace2d_smem(float *__restrict__ p, const float *__restrict__ bc, int n0, int n1, float cx, float cy,
                 float den, double tol, int max_iter, int *iters_out, double *l1_out)
{
    extern __shared__ float sm[];
    __shared__ double red[64];
    __shared__ double l1s;
    const int N = n0 * n1;
    float *PN = sm, *P = sm + N;
    for (int k = threadIdx.x; k < N; k += blockDim.x) PN[k] = P[k] = p[k];
    if (threadIdx.x == 0) l1s = 1.0;
    __syncthreads();
    int it = 0;
    while (it < max_iter && l1s > tol) {
        // interior sweep
        for (int k = threadIdx.x; k < N; k += blockDim.x) {
            const int i = k / n1, j = k - i * n1;
            if (i > 0 && i < n0 - 1 && j > 0 && j < n1 - 1) P[k] = jacobi_point(PN, k, n1, cx, cy, den);
        }
        __syncthreads();
        // boundary rows of P:411-414 (one pass, see the header)
        for (int e = threadIdx.x; e < (n0 - 2) + (n1 - 2) + 4; e += blockDim.x) laplace_boundary(P, bc, e, n0, n1);
        __syncthreads();
        // l1 = sum(|p| - |pn|) / sum(|pn|), fp64, fixed order
        double num = 0.0, dsum = 0.0;
        for (int k = threadIdx.x; k < N; k += blockDim.x) {
            num += (double)fabsf(P[k]) - (double)fabsf(PN[k]);
            dsum += (double)fabsf(PN[k]);
        }
        block_sum2(num, dsum, red);
        if (threadIdx.x == 0) l1s = num / dsum;
        ++it;
        float *T = PN;
        PN = P;
        P = T;
        __syncthreads();
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x) p[k] = PN[k];  // the last computed p
    if (threadIdx.x == 0) {
        *iters_out = it;
        *l1_out = l1s;
    }
}

// cooperative persistent Laplace solver for grids beyond one CTA's shared memory: every
// phase grid-strided over all CTAs, grid-wide barriers between phases, the l1 decision
// taken by block 0 from per-block partials (fixed order) and read by all
__global__ void __launch_bounds__(512)
k_laplace2d_coop(float *__restrict__ A, float *__restrict__ B, const float *__restrict__ bc, int64_t n0, int64_t n1,
                 float cx, float cy, float den, double tol, int max_iter, double *__restrict__ part,
                 volatile double *__restrict__ l1g, int *__restrict__ iters_out, double *__restrict__ l1_out)
{
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[64];
    const int64_t N = n0 * n1;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    const int64_t nb = (n0 - 2) + (n1 - 2) + 4;
    float *pn = A, *p = B;
    double l1 = 1.0;
    int it = 0;
    while (it < max_iter && l1 > tol) {
        for (int64_t k = tid; k < N; k += nth) {
            const int64_t i = k / n1, j = k - i * n1;
            if (i > 0 && i < n0 - 1 && j > 0 && j < n1 - 1) p[k] = jacobi_point(pn, k, n1, cx, cy, den);
        }
        grid.sync();
        for (int64_t e = tid; e < nb; e += nth) laplace_boundary(p, bc, e, n0, n1);
        grid.sync();
        double num = 0.0, dsum = 0.0;
        for (int64_t k = tid; k < N; k += nth) {
            num += (double)fabsf(p[k]) - (double)fabsf(pn[k]);
            dsum += (double)fabsf(pn[k]);
        }
        block_sum2(num, dsum, red);
        if (threadIdx.x == 0) {
            part[2 * blockIdx.x] = num;
            part[2 * blockIdx.x + 1] = dsum;
        }
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            double x = 0.0, y = 0.0;
            for (unsigned b = 0; b < gridDim.x; ++b) {
                x += part[2 * b];
                y += part[2 * b + 1];
            }
            *l1g = x / y;
        }
        grid.sync();
        l1 = *l1g;
        ++it;
        float *T = pn;
        pn = p;
        p = T;
    }
    if (tid == 0) {
        *iters_out = it;
        *l1_out = l1;
    }
    // the last computed p ends in pn; the host copies it to the caller's buffer if needed
}

}  // namespace

extern "C" sf_status sf_convection2d(float *u, float *work, int64_t n0, int64_t n1, double c, double dt,
                                     double dx, double dy, int nt, void *stream)
{
    if (!u || n0 < 2 || n1 < 2 || nt < 0 || !(dx > 0.0) || !(dy > 0.0))
        return sf_set_error(SF_ERR_INVALID_ARG, "convection2d: bad arguments");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const float a = (float)(c * dt / dx), b = (float)(c * dt / dy);
    const int64_t N = n0 * n1;
    if (N <= SF_CFD_SMEM_PTS) {
        const size_t smem = sizeof(float) * 2 * (size_t)N;
        SF_CUDA_TRY(cudaFuncSetAttribute(k_conv2d_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_conv2d_smem<<<1, SF_CFD_THREADS, smem, st>>>(u, (int)n0, (int)n1, a, b, nt);
        SF_CUDA_TRY(cudaGetLastError());
        return SF_OK;
    }
    if (!work) return sf_set_error(SF_ERR_WORKSPACE, "convection2d: grid of %lld points needs `work`", (long long)N);
    float *src = u, *dst = work;
    for (int t = 0; t < nt; ++t) {
        k_conv2d_step<<<592, 256, 0, st>>>(src, dst, n0, n1, a, b);
        float *T = src;
        src = dst;
        dst = T;
    }
    SF_CUDA_TRY(cudaGetLastError());
    if (src != u) SF_CUDA_TRY(cudaMemcpyAsync(u, src, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
    return SF_OK;
}

extern "C" sf_status sf_laplace2d(float *p, float *work, const float *bc, int64_t n0, int64_t n1, double dx,
                                  double dy, double tol, int max_iter, int *iters, double *l1, void *stream)
{
    if (!p || !bc || n0 < 3 || n1 < 3 || max_iter < 0 || !(dx > 0.0) || !(dy > 0.0))
        return sf_set_error(SF_ERR_INVALID_ARG, "laplace2d: bad arguments");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const float cx = (float)(dy * dy), cy = (float)(dx * dx), den = (float)(2.0 * (dx * dx + dy * dy));
    const int64_t N = n0 * n1;
    int *d_it = nullptr;
    double *d_l1 = nullptr;
    SF_CUDA_TRY(cudaMalloc(&d_it, sizeof(int)));
    SF_CUDA_TRY(cudaMalloc(&d_l1, sizeof(double)));
    int it = 0;
    double l1v = 1.0;
    if (N <= SF_LAP_ONE_CTA_PTS) {
        const size_t smem = sizeof(float) * 2 * (size_t)N;
        SF_CUDA_TRY(cudaFuncSetAttribute(k_laplace2d_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // ~4 points per thread: fewer warps make the per-sweep barriers and the warp-total
        // pass of the l1 reduction cheaper (31^2: 256 threads)
        const int thr = (int)std::min<int64_t>(SF_CFD_THREADS, std::max<int64_t>(64, ((N / 4 + 31) / 32) * 32));
        k_laplace2d_smem<<<1, thr, smem, st>>>(p, bc, (int)n0, (int)n1, cx, cy, den, tol, max_iter, d_it, d_l1);
        SF_CUDA_TRY(cudaGetLastError());
        SF_CUDA_TRY(cudaMemcpyAsync(&it, d_it, sizeof(int), cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaMemcpyAsync(&l1v, d_l1, sizeof(double), cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaStreamSynchronize(st));
    } else {
        if (!work) return sf_set_error(SF_ERR_WORKSPACE, "laplace2d: grid of %lld points needs `work`", (long long)N);
        int dev = 0, sms = 0, per = 0;
        SF_CUDA_TRY(cudaGetDevice(&dev));
        SF_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        SF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_laplace2d_coop, 512, 0));
        // up to ~1M points one CTA of 512 threads per SM (the fewest CTAs to meet at each grid
        // barrier: 160^2 76 ms vs 96 ms with four); larger grids fill the SMs for bandwidth
        // (2048^2: 15 ms vs 43 ms)
        const int nb = std::max(1, sms * std::max(1, std::min(per, N > (int64_t(1) << 20) ? 4 : 1)));
        double *part = nullptr, *l1g = nullptr;
        SF_CUDA_TRY(cudaMalloc(&part, sizeof(double) * 2 * nb));
        SF_CUDA_TRY(cudaMalloc(&l1g, sizeof(double)));
        SF_CUDA_TRY(cudaMemcpyAsync(work, p, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
        float *A = p, *B = work;
        void *args[] = {&A, &B, (void *)&bc, (void *)&n0, (void *)&n1, (void *)&cx, (void *)&cy, (void *)&den,
                        (void *)&tol, (void *)&max_iter, &part, &l1g, &d_it, &d_l1};
        SF_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_laplace2d_coop, dim3(nb), dim3(512), args, 0, st));
        SF_CUDA_TRY(cudaMemcpyAsync(&it, d_it, sizeof(int), cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaMemcpyAsync(&l1v, d_l1, sizeof(double), cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaStreamSynchronize(st));
        if (it % 2 == 1)  // the last sweep wrote into `work`
            SF_CUDA_TRY(cudaMemcpyAsync(p, work, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
        SF_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(part);
        cudaFree(l1g);
    }
    cudaFree(d_it);
    cudaFree(d_l1);
    if (iters) *iters = it;
    if (l1) *l1 = l1v;
    return SF_OK;
}
