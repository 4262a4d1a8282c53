// inst_body.cuh -- instantiates every stencil-step kernel for one radius SF_R
// (included by inst_r<R>.cu).  Dispatch: variant x (by, damp, mode).
#include <algorithm>
#include <atomic>
#include "launch.cuh"
#include "stencil_generic.cuh"
#include "stencil_tma.cuh"
#include "loop2d.cuh"
#if SF_R <= 4
#include "stencil_tb2.cuh"
#endif

#ifndef SF_R
#error "define SF_R"
#endif
#define SF_CAT_(a, b) a##b
#define SF_CAT(a, b) SF_CAT_(a, b)

namespace {

template <int VY, int DM, int MODE, int LZ, int BIDIR = 0, int LAY = 0>
cudaError_t launch_tma(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    if constexpr (BIDIR == 0 && LZ == 32 && LAY == 0) {
        // the one-launch slab schedule has its own instances (direction and boundary-signal
        // code compiled out of the plain ones: it cost up to 7 % at r = 8 when only inactive;
        // the per-plane peer-store test another 12 %: a third instance for SF_OPT_P2P)
        if (a.bidir) {
            if (a.mq[1] > a.mq[0] || a.mq[3] > a.mq[2]) return launch_tma<VY, DM, MODE, LZ, 2>(L, a, st);
            return launch_tma<VY, DM, MODE, LZ, 1>(L, a, st);
        }
    }
    using C = sftma::Cfg<SF_R, VY, DM, MODE, LZ, LAY>;
    auto kern = sftma::k_tma3d<SF_R, VY, DM, MODE, LZ, BIDIR, LAY>;
    // the dynamic shared-memory limit is a per-device function attribute: cached per device
    // in an atomic bitmask (handles on several GPUs, concurrent rank threads)
    static std::atomic<uint64_t> attr{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
    if (!bit || !(attr.load(std::memory_order_acquire) & bit)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr.fetch_or(bit, std::memory_order_release);
    }
    // persistent grid: (tile, x-chunk) items, at most one CTA per SM (shared memory admits
    // one), items dealt round-robin.  The chunk count minimises rounds x (chunk + 2r): each
    // item re-reads 2r warm-up planes of u^n.  L.ctas overrides the CTA count.
    const int64_t PT = (a.xb - a.xa) + (a.xb2 - a.xa2);
    const int64_t tiles = ((a.n2t - a.zbase + C::TZ - 1) / C::TZ) * ((a.n1 + C::BY - 1) / C::BY);
    if (PT <= 0 || tiles <= 0) return cudaSuccess;
    const int64_t slots = L.ctas > 0 ? L.ctas : L.sms;
    // one-launch slab schedule (a.bidir): at least two chunks per tile (the last one streams
    // downward) of at least r planes each, so each boundary range lies in one chunk
    double best = 1e300;
    int64_t chunk = PT, nch = 1;
    for (int64_t c = a.bidir ? 2 : 1; c <= std::min<int64_t>(PT, 256); ++c) {
        const int64_t ch = (PT + c - 1) / c, ce = (PT + ch - 1) / ch;
        if (a.bidir && (ce < 2 || ch < SF_R)) continue;
        const int64_t items = tiles * ce, g = std::min(items, slots);
        const double t = (double)((items + g - 1) / g) * (double)(ch + 2 * SF_R);
        if (t < best - 1e-9) {
            best = t;
            chunk = ch;
            nch = ce;
        }
    }
    int64_t g = std::min(tiles * nch, slots);
    // balanced contiguous split (SF_OPT_BALANCE / sf_autotune; kernel nchunk = 0): every CTA
    // streams the same number of planes, at most ~2 segments (2 warm-ups) each -- faster where
    // the tile count packs badly into the chunked rounds (configs[4], 8-warp layout: -4 %),
    // much slower where the neighbours' re-read halo rows cost HBM time (configs[1], [3])
    if (!a.bidir && L.balance == 1) {
        g = std::min<int64_t>(slots, tiles * PT);
        nch = 0;
    }
    dim3 block(32, C::THREADS / 32);  // NW consumer warps + the TMA producer warp(s)
    // programmatic dependent launch (SF_OPT_PDL): the CTAs' prologue (barrier init, tensor-map
    // prefetch) overlaps the previous kernel's tail; they wait (griddepcontrol.wait) before
    // their first global access
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = L.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, L.maps->cur, L.maps->old, L.maps->c3, L.maps->beta, L.maps->snap,
                              L.maps->grad, a, L.snap_slot, (int)chunk, (int)nch);
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

template <int VY, int DM, int LZ, int LAY = 0>
cudaError_t launch_tma_dm(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    switch (L.mode) {
    case SF_MODE_PLAIN: return launch_tma<VY, DM, SF_MODE_PLAIN, LZ, 0, LAY>(L, a, st);
    case SF_MODE_SAVE: return launch_tma<VY, DM, SF_MODE_SAVE, LZ, 0, LAY>(L, a, st);
    default: return launch_tma<VY, DM, SF_MODE_GRAD, LZ, 0, LAY>(L, a, st);
    }
}

template <int VY, int LZ, int LAY = 0>
cudaError_t launch_tma_vy(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    if (L.damp == SF_DAMP_ARRAY) return launch_tma_dm<VY, SF_DAMP_ARRAY, LZ, LAY>(L, a, st);
    if (L.damp == SF_DAMP_SEP) return launch_tma_dm<VY, SF_DAMP_SEP, LZ, LAY>(L, a, st);
    return launch_tma_dm<VY, SF_DAMP_NONE, LZ, LAY>(L, a, st);
}

template <int VY, int DM, int MODE, int LAY>
int smem_of() { return sftma::Cfg<SF_R, VY, DM, MODE, 32, LAY>::SMEM; }

template <int VY, int DM, int LAY>
int smem_dm(int mode)
{
    return mode == 0 ? smem_of<VY, DM, 0, LAY>() : mode == 1 ? smem_of<VY, DM, 1, LAY>() : smem_of<VY, DM, 2, LAY>();
}

template <int VY, int LAY = 0>
int smem_vy(int damp, int mode)
{
    if (damp == SF_DAMP_ARRAY) return smem_dm<VY, SF_DAMP_ARRAY, LAY>(mode);
    if (damp == SF_DAMP_SEP) return smem_dm<VY, SF_DAMP_SEP, LAY>(mode);
    return smem_dm<VY, SF_DAMP_NONE, LAY>(mode);
}

}  // namespace

// Tile shapes (stencil_tma.cuh Geo): vy = 2 -> two rows per thread, 14 x 128 tiles; vy = 1
// -> one row per thread, 7 x 128 tiles; narrow (lz = 8, the z remainder): 56 x 32 tiles.
cudaError_t SF_CAT(sf_launch_step_r, SF_R)(const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    if (L.variant == SF_VAR_TMA) {
        if (L.lz == 8) return L.vy == 4 ? launch_tma_vy<2, 8, 2>(L, a, st) : launch_tma_vy<2, 8>(L, a, st);
        if (L.vy == 1) return launch_tma_vy<1, 32>(L, a, st);
        if (L.vy == 4) return launch_tma_vy<2, 32, 2>(L, a, st);  // 8 consumer warps (Geo LAY = 2)
#if SF_R >= 5
        if (L.vy == 3) return launch_tma_vy<2, 32, 1>(L, a, st);  // wide layout (Geo LAY = 1)
#endif
        return launch_tma_vy<2, 32>(L, a, st);
    }
    switch (L.mode) {
    case SF_MODE_PLAIN: return launch_generic<SF_MODE_PLAIN>(L, a, st);
    case SF_MODE_SAVE: return launch_generic<SF_MODE_SAVE>(L, a, st);
    default: return launch_generic<SF_MODE_GRAD>(L, a, st);
    }
}

int SF_CAT(sf_tma_smem_r, SF_R)(int vy, int damp, int mode)
{
    if (vy == 1) return smem_vy<1>(damp, mode);
    if (vy == 3) return SF_R >= 5 ? smem_vy<2, 1>(damp, mode) : 0;
    if (vy == 4) return smem_vy<2, 2>(damp, mode);
    return smem_vy<2>(damp, mode);
}

// whole 2D time loop of a small grid in one CTA cluster (loop2d.cuh, SF_OPT_LOOP2D)
cudaError_t SF_CAT(sf_launch_loop2d_r, SF_R)(const Loop2dArgs &a, cudaStream_t st)
{
    const size_t smem = loop2d_smem(a.rpc, a.n2, a.beta != nullptr);
    auto kern = k_loop2d<SF_R>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(SF_LOOP2D_CTAS);
    cfg.blockDim = dim3(SF_LOOP2D_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = SF_LOOP2D_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

#if SF_R <= 4
// two steps per pass (temporal blocking, stencil_tb2.cuh, SF_OPT_TBLOCK): persistent grid of
// (tile, x-chunk) items; the chunk count minimises rounds x (chunk + 4r)
cudaError_t SF_CAT(sf_launch_tb2_r, SF_R)(const SfTmaMaps &m, const TbArgs &a0, int ctas, cudaStream_t st)
{
    TbArgs a = a0;
    const bool damp = a.beta != nullptr;
    const int64_t tiles = (int64_t)((a.n2 + sftb::TZ - 1) / sftb::TZ) * ((a.n1 + sftb::TY - 1) / sftb::TY);
    if (tiles <= 0 || a.n0 <= 0) return cudaSuccess;
    double best = 1e300;
    int chunk = a.n0, nch = 1;
    for (int c = 1; c <= std::min(a.n0, 64); ++c) {
        const int ch = (a.n0 + c - 1) / c, ce = (a.n0 + ch - 1) / ch;
        const int64_t items = tiles * ce, g = std::min<int64_t>(items, ctas);
        const double t = (double)((items + g - 1) / g) * (double)(ch + 4 * SF_R);
        if (t < best - 1e-9) {
            best = t;
            chunk = ch;
            nch = ce;
        }
    }
    a.chunk = chunk;
    a.nchunk = nch;
    const int64_t g = std::min<int64_t>(tiles * nch, ctas);
    int smem;
    cudaError_t e;
    if (damp) {
        smem = sftb::TbCfg<SF_R, true>::SMEM;
        e = cudaFuncSetAttribute(sftb::k_tb2<SF_R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        sftb::k_tb2<SF_R, true><<<(unsigned)g, 256, smem, st>>>(m.cur, m.old, m.c3, m.beta, a);
    } else {
        smem = sftb::TbCfg<SF_R, false>::SMEM;
        e = cudaFuncSetAttribute(sftb::k_tb2<SF_R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        sftb::k_tb2<SF_R, false><<<(unsigned)g, 256, smem, st>>>(m.cur, m.old, m.c3, m.c3, a);
    }
    return cudaGetLastError();
}
#endif
