// inst_body.cuh -- instantiates every stencil-step kernel for one radius SF_R
// (included by inst_r<R>.cu).  Dispatch: variant x (by, damp, mode).
#include "launch.cuh"
#include "stencil_generic.cuh"
#include "stencil_tma.cuh"

#ifndef SF_R
#error "define SF_R"
#endif
#define SF_CAT_(a, b) a##b
#define SF_CAT(a, b) SF_CAT_(a, b)

namespace {

template <int BY, int VZ, bool DAMP, int MODE>
cudaError_t launch_tma(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    using C = sftma::Cfg<SF_R, BY, VZ, DAMP, MODE>;
    auto kern = sftma::k_tma3d<SF_R, BY, VZ, DAMP, MODE>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int64_t planes = a.xb - a.xa;
    const int nchunks = L.chunks > 0 ? L.chunks : 1;
    const int chunk = (int)((planes + nchunks - 1) / nchunks);
    const int nch = (int)((planes + chunk - 1) / chunk) + (int)((a.xb2 - a.xa2 + chunk - 1) / chunk);
    dim3 grid((unsigned)((a.n2 + C::TZ - 1) / C::TZ), (unsigned)((a.n1 + BY - 1) / BY), (unsigned)nch);
    dim3 block(32, BY + 1);  // BY consumer warps + 1 TMA producer warp
    kern<<<grid, block, C::SMEM, st>>>(L.maps->cur, L.maps->old, L.maps->c3, L.maps->beta,
                                       L.maps->snap, L.maps->grad, a, L.snap_slot, chunk);
    return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_generic(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    const int64_t planes = (a.xb - a.xa) + (a.xb2 - a.xa2);
    dim3 block(32, 8);
    if (L.ndim == 3) {
        dim3 grid((unsigned)((a.n2 + 31) / 32), (unsigned)((a.n1 + 7) / 8), (unsigned)planes);
        k_generic3d<SF_R, MODE><<<grid, block, 0, st>>>(a);
    } else {
        dim3 grid((unsigned)((a.n2 + 31) / 32), (unsigned)((planes + 7) / 8));
        k_generic2d<SF_R, MODE><<<grid, block, 0, st>>>(a);
    }
    return cudaGetLastError();
}

template <int BY, int VZ>
cudaError_t launch_tma_by(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    if (L.damp) {
        switch (L.mode) {
        case SF_MODE_PLAIN: return launch_tma<BY, VZ, true, SF_MODE_PLAIN>(L, a, st);
        case SF_MODE_SAVE: return launch_tma<BY, VZ, true, SF_MODE_SAVE>(L, a, st);
        default: return launch_tma<BY, VZ, true, SF_MODE_GRAD>(L, a, st);
        }
    }
    switch (L.mode) {
    case SF_MODE_PLAIN: return launch_tma<BY, VZ, false, SF_MODE_PLAIN>(L, a, st);
    case SF_MODE_SAVE: return launch_tma<BY, VZ, false, SF_MODE_SAVE>(L, a, st);
    default: return launch_tma<BY, VZ, false, SF_MODE_GRAD>(L, a, st);
    }
}

template <int BY, int VZ, bool DAMP, int MODE>
int smem_of() { return sftma::Cfg<SF_R, BY, VZ, DAMP, MODE>::SMEM; }

template <int BY, int VZ>
int smem_by(int damp, int mode)
{
    if (damp) return mode == 0 ? smem_of<BY, VZ, true, 0>() : mode == 1 ? smem_of<BY, VZ, true, 1>() : smem_of<BY, VZ, true, 2>();
    return mode == 0 ? smem_of<BY, VZ, false, 0>() : mode == 1 ? smem_of<BY, VZ, false, 1>() : smem_of<BY, VZ, false, 2>();
}

}  // namespace

// Tile shapes: r <= 4: BY = 16 or 8 warps of 4 z per lane (128-column tiles); r >= 5:
// BY = 8 with 4 z per lane, or BY = 16 with 2 z per lane (64-column tiles) -- the
// (2r+1)-deep register queues must fit the 96-register budget of 17 warps.
cudaError_t SF_CAT(sf_launch_step_r, SF_R)(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    if (L.variant == SF_VAR_TMA) {
#if SF_R <= 4
        if (L.by == 16) return launch_tma_by<16, 4>(L, a, st);
        return launch_tma_by<8, 4>(L, a, st);
#else
        if (L.by == 16) return launch_tma_by<16, 2>(L, a, st);
        return launch_tma_by<8, 4>(L, a, st);
#endif
    }
    switch (L.mode) {
    case SF_MODE_PLAIN: return launch_generic<SF_MODE_PLAIN>(L, a, st);
    case SF_MODE_SAVE: return launch_generic<SF_MODE_SAVE>(L, a, st);
    default: return launch_generic<SF_MODE_GRAD>(L, a, st);
    }
}

int SF_CAT(sf_tma_smem_r, SF_R)(int by, int damp, int mode)
{
#if SF_R <= 4
    if (by == 16) return smem_by<16, 4>(damp, mode);
    return smem_by<8, 4>(damp, mode);
#else
    if (by == 16) return smem_by<16, 2>(damp, mode);
    return smem_by<8, 4>(damp, mode);
#endif
}
