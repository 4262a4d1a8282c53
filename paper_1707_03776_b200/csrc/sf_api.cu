// sf_api.cu -- host side of libsf.so: the C-ABI of include/sf.h.
//
// Validation, host FD weights, sparse tables, coefficient hoisting, the time-loop
// drivers (forward, adjoint, gradient), the residual/objective and the end-to-end
// host-buffer form.  Every step of the path runs in this library's CUDA kernels
// (stencil_*.cuh, sparse.cuh); there is no CPU fallback: without a CUDA device every
// compute call fails with SF_ERR_CUDA.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include "sf_internal.h"
#include "sparse.cuh"
#include "loop2d.cuh"

#define SF_VERSION 1
#ifndef SF_SIDE_MIN_POINTS
#define SF_SIDE_MIN_POINTS (1 << 22)  // grids below this record in stream order
#endif

static thread_local char g_err[1024] = "";

sf_status sf_set_error(sf_status s, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return s;
}

extern "C" const char *sf_last_error(void) { return g_err; }
extern "C" int sf_version(void) { return SF_VERSION; }

// ------------------------------------------------------------------ FD weights (host)
// Closed form of the centred 2nd-derivative weights of order 2r:
//   w_k = 2 (-1)^{k+1} (r!)^2 / (k^2 (r-k)! (r+k)!),  w_0 = -2 sum_{k>=1} w_k.
// (All factorials up to 16! are exact in fp64.)
static double fact(int n)
{
    double f = 1.0;
    for (int i = 2; i <= n; ++i) f *= (double)i;
    return f;
}

extern "C" sf_status sf_fd_weights(int space_order, double *w)
{
    if (!w) return sf_set_error(SF_ERR_INVALID_ARG, "sf_fd_weights: w is NULL");
    if (space_order < 2 || space_order > 2 * SF_MAXR || (space_order & 1))
        return sf_set_error(SF_ERR_ORDER, "space_order %d not in {2,4,...,16}", space_order);
    const int r = space_order / 2;
    double s = 0.0;
    for (int k = 1; k <= r; ++k) {
        const double sgn = (k & 1) ? 1.0 : -1.0;
        w[k] = 2.0 * sgn * fact(r) * fact(r) / ((double)k * k * fact(r - k) * fact(r + k));
        s += w[k];
    }
    w[0] = -2.0 * s;
    return SF_OK;
}

// ------------------------------------------------------------------ stream memory operations
// (SF_OPT_P2P counters: a stream-ordered 32-bit write after the boundary work, a stream wait
// on the value in the neighbour -- no kernel ever spins on another rank)
typedef CUresult (*sf_pfn_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static sf_pfn_value32 memop_fn(const char *name)
{
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        return reinterpret_cast<sf_pfn_value32>(p);
    return nullptr;
}
static sf_status stream_write32(cudaStream_t st, uint32_t *addr, uint32_t v)
{
    static sf_pfn_value32 fn = memop_fn("cuStreamWriteValue32");
    if (!fn) return sf_set_error(SF_ERR_CUDA, "cuStreamWriteValue32 unavailable");
    // default flags: a memory fence orders the preceding peer stores before the value
    if (fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v, 0) != CUDA_SUCCESS)
        return sf_set_error(SF_ERR_CUDA, "cuStreamWriteValue32 failed");
    return SF_OK;
}
static sf_status stream_wait32(cudaStream_t st, uint32_t *addr, uint32_t v)
{
    static sf_pfn_value32 fn = memop_fn("cuStreamWaitValue32");
    if (!fn) return sf_set_error(SF_ERR_CUDA, "cuStreamWaitValue32 unavailable");
    // CU_STREAM_WAIT_VALUE_GEQ (0): (int32)(*addr - v) >= 0, wrap-around safe
    if (fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v, 0) != CUDA_SUCCESS)
        return sf_set_error(SF_ERR_CUDA, "cuStreamWaitValue32 failed");
    return SF_OK;
}

// ------------------------------------------------------------------ tensor maps (TMA)
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// fp32 tensor [dims[rank-1]]...[dims[0]] (dims[0] fastest), dense strides, box `box`.
static sf_status make_map(CUtensorMap *m, const void *base, int rank, const int64_t *dims,
                          const uint32_t *box, bool half = false)
{
    auto enc = tmap_encoder();
    if (!enc) return sf_set_error(SF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5], es[5];
    uint64_t stride = half ? 2 : 4;
    for (int i = 0; i < rank; ++i) {
        gd[i] = (cuuint64_t)dims[i];
        bx[i] = box[i];
        es[i] = 1;
        if (i > 0) gs[i - 1] = stride;
        stride *= (uint64_t)dims[i];
    }
    CUresult r = enc(m, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     (cuuint32_t)rank, const_cast<void *>(base),
                     gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return sf_set_error(SF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SF_OK;
}

// ------------------------------------------------------------------ launch plumbing
static inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

static cudaError_t launch_step_r(int r, const SfLaunch &L, const SfStepArgs &a, cudaStream_t st)
{
    switch (r) {
    case 1: return sf_launch_step_r1(L, a, st);
    case 2: return sf_launch_step_r2(L, a, st);
    case 3: return sf_launch_step_r3(L, a, st);
    case 4: return sf_launch_step_r4(L, a, st);
    case 5: return sf_launch_step_r5(L, a, st);
    case 6: return sf_launch_step_r6(L, a, st);
    case 7: return sf_launch_step_r7(L, a, st);
    default: return sf_launch_step_r8(L, a, st);
    }
}

int sf_tma_smem_bytes(int r, int vy, int damp, int mode)
{
    switch (r) {
    case 1: return sf_tma_smem_r1(vy, damp, mode);
    case 2: return sf_tma_smem_r2(vy, damp, mode);
    case 3: return sf_tma_smem_r3(vy, damp, mode);
    case 4: return sf_tma_smem_r4(vy, damp, mode);
    case 5: return sf_tma_smem_r5(vy, damp, mode);
    case 6: return sf_tma_smem_r6(vy, damp, mode);
    case 7: return sf_tma_smem_r7(vy, damp, mode);
    default: return sf_tma_smem_r8(vy, damp, mode);
    }
}

static bool tma_ok(const sf_handle *h)
{
    // 16-byte global strides for TMA: n2 % 4 (fp32 fields), n2 % 8 with fp16 snapshots
    return h->ndim == 3 && (h->nb[2] % (h->snap_half ? 8 : 4)) == 0 && h->nb[2] >= 4 && h->nb[1] >= 1 &&
           h->N < (int64_t(1) << 40) && h->nb[0] < (int64_t(1) << 31);
}

// bytes per snapshot element (fp32, or fp16 with SF_OPT_SNAP_HALF)
static size_t snap_es(const sf_handle *h) { return h->snap_half ? 2 : 4; }
template <class T>
static T *snap_slot(T *base, const sf_handle *h, int64_t slot)
{
    using B = typename std::conditional<std::is_const<T>::value, const char, char>::type;
    return reinterpret_cast<T *>(reinterpret_cast<B *>(base) + (size_t)slot * (size_t)h->N * snap_es(h));
}

static int resolve_variant(const sf_handle *h)
{
    if (h->variant == SF_VAR_GENERIC) return SF_VAR_GENERIC;
    if (tma_ok(h)) return SF_VAR_TMA;
    return SF_VAR_GENERIC;
}

// TMA layout of a step of `mode`: GRAD-mode steps may use their own (sf_autotune times them
// separately: the 8-warp layout is faster for the plain step at high order, slower in GRAD)
static int resolve_vy(const sf_handle *h, int mode)
{
    const int vy = (mode == SF_MODE_GRAD && h->vy_grad) ? h->vy_grad : h->vy;
    if (vy == 1) return 1;
    if (vy == 3 && h->r >= 5) return 3;  // the wide layout exists for r >= 5 only
    if (vy == 4) return 4;
    return 2;
}

// TMA kernel tile geometry (stencil_tma.cuh Geo): VY rows per thread (tuning `vy`, auto
// 2), 7 consumer warps -> BY = 7 VY tile rows; 4 z per lane -> 128-column tiles.
// vy = 3: the wide layout (Geo LAY = 1, r >= 5): 11 consumer warps x 2 rows, 2 z per lane ->
// 22 x 64 tiles.  vy = 4: the warp-specialised layout (Geo LAY = 2): 8 consumer warps x 2 rows
// x 4 z per lane -> 16 x 128 tiles, a producer warpgroup handing its registers over.
static int tile_nw(int vy) { return vy == 3 ? 11 : vy == 4 ? 8 : 7; }
static int tile_rows(int vy) { return vy >= 3 ? 2 : vy; }  // rows per thread
static int tile_vz(const sf_handle *, int vy) { return vy == 3 ? 2 : 4; }
static int tile_tz(const sf_handle *h, int vy) { return 32 * tile_vz(h, vy); }
static int tile_by(int vy) { return tile_nw(vy) * tile_rows(vy); }
// narrow tiles of the z remainder (Geo<R, 2, 8, LAY>): 8 lanes x 4 z, 4 lane rows x 2 rows x
// 7 warps (8 with the warp-specialised layout)
static const int NARROW_TZ = 32;
static int narrow_by(int vy) { return 4 * 2 * (vy == 4 ? 8 : 7); }

// persistent CTAs of the TMA kernel (0 = one per SM)
static int resolve_ctas(const sf_handle *h) { return h->ctas > 0 ? h->ctas : h->sms; }

// ---- profiling: CUDA events around every launch, grouped by kind (stream-ordered)
enum { PK_STENCIL = 0, PK_INJECT = 1, PK_INTERP = 2, PK_OTHER = 3, PK_N = 4 };

static cudaEvent_t next_event(sf_handle *h)
{
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        h->ev_pool.push_back(e);
    }
    return h->ev_pool[h->ev_used++];
}

struct ProfScope {
    sf_handle *h;
    cudaStream_t st;
    cudaEvent_t e1 = nullptr;
    ProfScope(sf_handle *h_, int kind, cudaStream_t st_) : h(h_), st(st_)
    {
        h->n_all++;
        // SF_OPT_PROF_EVERY = n: time every n-th launch of each kind (the event pair between
        // two kernels costs ~1-3 % and defeats PDL); totals are scaled by launches / timed
        if (h->prof && (h->n_kind[kind] % h->prof_every) == 0) {
            cudaEvent_t e0 = next_event(h);
            e1 = next_event(h);
            h->ev_kind.push_back(kind);
            h->n_samp[kind]++;
            cudaEventRecord(e0, st);
        }
        h->n_kind[kind]++;
    }
    ~ProfScope()
    {
        if (e1) cudaEventRecord(e1, st);
    }
};

struct StepBufs {
    const float *cur;
    float *out;
    float *snap_out;       // SAVE
    const float *snaps;    // GRAD: snapshot array base
    int snap_slot;
    int64_t nsnap;
    float *grad;
    float gscale;
    SfSparse *inj;         // point set injected after this step (or NULL)
    const float *inj_vals; // its values for this step ([npoint])
    SfSparse *itp;         // point set interpolated from the new level (or NULL)
    float *itp_row;        // its record row for the new level ([npoint])
    int64_t xa = 0, xb = 0;  // planes to compute (xa == xb: the handle's full range)
    int64_t xa2 = 0, xb2 = 0;  // optional second range in the same launch
    int ctas_cap = 0;          // > 0: at most this many persistent TMA CTAs (split interior)
    int itp_cur = -1;          // side-stream record index of the `cur` level (SF_OPT_P2P ordering)
    bool force_generic = false;            // thread-per-point kernel (P2P boundary launch)
    bool bidir = false;                    // one-launch slab schedule (SfStepArgs::bidir / sig)
    bool nosig = false;                    // bidir without the device counters (peer-store form)
    bool dry = false;                      // launch_step: decide (fused, tiles), launch nothing
    const int64_t *mq = nullptr, *md = nullptr;  // peer-store mirror (SfStepArgs::mq / md)
};

// Library-internal device allocations come from the device's stream-ordered memory pool
// (kept, not released to the OS: release threshold = max), ordered on the legacy stream.
// Creating and destroying handles then costs no device-wide synchronisation and no page
// unmapping -- sf_forward_host builds a handle per call.
static cudaError_t sf_dalloc(void **p, size_t bytes)
{
    static thread_local int pool_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (pool_dev != dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_dev = dev;
    }
    return cudaMallocAsync(p, bytes, 0);
}
static void sf_dfree(void *p)
{
    if (p) cudaFreeAsync(p, 0);
}
#define cudaMalloc(p, n) sf_dalloc((void **)(p), (n))
#define cudaFree(p) sf_dfree((void *)(p))

static void drop_graphs(sf_handle *h);

template <class T>
static sf_status upload(T **dst, const std::vector<T> &v)
{
    if (v.empty()) return SF_OK;
    SF_CUDA_TRY(cudaMalloc((void **)dst, v.size() * sizeof(T)));
    SF_CUDA_TRY(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return SF_OK;
}



static void free_inj(SfInjTiles &T)
{
    cudaFree(T.beg);
    cudaFree(T.q);
    cudaFree(T.lj);
    cudaFree(T.t);
    T = SfInjTiles{};
}

// where grid offset `off` lives in the TMA kernel: (tile * NW + warp, plane, lane, row of
// the warp jy, z in the lane jz)
struct TileLoc {
    int wl, q, lane, jy, j;
};
static TileLoc tile_loc(const sf_handle *h, int vy, int64_t off)
{
    const int64_t n1 = h->nb[1], n2 = h->nb[2];
    const int tz = tile_tz(h, vy), vz = tile_vz(h, vy), by = tile_by(vy);
    const int64_t ntz = (n2 + tz - 1) / tz;
    const int64_t x = off / (n1 * n2), y = (off / n2) % n1, z = off % n2;
    const int64_t tile = (y / by) * ntz + z / tz;
    const int ry = tile_rows(vy);
    return {(int)(tile * tile_nw(vy) + (y % by) / ry), (int)x, (int)((z % tz) / vz), (int)((y % by) % ry),
            (int)(z % vz)};
}

static int64_t n_warp_lists(const sf_handle *h, int vy)
{
    const int tz = tile_tz(h, vy), by = tile_by(vy);
    return ((h->nb[2] + tz - 1) / tz) * ((h->nb[1] + by - 1) / by) * tile_nw(vy);
}

// Per-(tile, warp) lists of the injection targets for the TMA kernel's fused injection.
static sf_status ensure_split_lists(sf_handle *h, SfSparse &sp);

static sf_status ensure_inj_tiles(sf_handle *h, SfSparse &sp, int by)
{
    SfInjTiles &T = sp.tiles;
    if (T.by == by) return SF_OK;
    if (T.by) cudaDeviceSynchronize();  // lists of another tile shape may still be in use
    free_inj(T);
    const int64_t nl = n_warp_lists(h, by);
    struct E {
        int wl, q, lj, t;
    };
    std::vector<E> es;
    for (size_t t = 0; t < sp.h_tgt.size(); ++t) {
        const TileLoc L = tile_loc(h, by, sp.h_tgt[t]);
        es.push_back({L.wl, L.q, (L.jy * 32 + L.lane) * 4 + L.j, (int)t});
    }
    std::sort(es.begin(), es.end(), [](const E &a, const E &b) {
        return std::tie(a.wl, a.q, a.lj) < std::tie(b.wl, b.q, b.lj);
    });
    std::vector<int> beg(nl + 1, 0), q, lj, tt;
    for (const E &e : es) beg[e.wl + 1]++;
    for (int64_t i = 0; i < nl; ++i) beg[i + 1] += beg[i];
    for (const E &e : es) {
        q.push_back(e.q);
        lj.push_back(e.lj);
        tt.push_back(e.t);
    }
    sf_status s;
    if ((s = upload(&T.beg, beg))) return s;
    if (!es.empty()) {
        if ((s = upload(&T.q, q))) return s;
        if ((s = upload(&T.lj, lj))) return s;
        if ((s = upload(&T.t, tt))) return s;
    }
    T.by = by;
    return SF_OK;
}

static sf_status launch_step(sf_handle *h, const StepBufs &b, int mode, cudaStream_t st, bool *fused)
{
    *fused = false;
    SfStepArgs a{};
    a.cur = b.cur;
    a.out = b.out;
    a.c3 = h->c3;
    a.beta = h->beta;
    a.snap_out = b.snap_out;
    a.snap_in = b.snaps ? snap_slot(b.snaps, h, b.snap_slot) : nullptr;
    a.snap_half = h->snap_half ? 1 : 0;
    a.grad = b.grad;
    a.gscale = b.gscale;
    if (h->ndim == 3) {
        a.n0b = h->nb[0];
        a.n1 = h->nb[1];
        a.n2 = h->nb[2];
    } else {
        a.n0b = h->nb[0];
        a.n1 = 1;
        a.n2 = h->nb[1];
    }
    a.xa = b.xa < b.xb ? b.xa : h->xa;
    a.xb = b.xa < b.xb ? b.xb : h->xb;
    a.xa2 = b.xa2;
    a.xb2 = b.xb2;
    a.zbase = 0;
    a.n2t = a.n2;
    a.w = h->w;
    a.l2_prefetch = h->l2_prefetch;

    SfLaunch L{};
    L.ndim = h->ndim;
    L.variant = b.force_generic ? SF_VAR_GENERIC : resolve_variant(h);
    L.vy = resolve_vy(h, mode);
    if (b.mq) {
        for (int k = 0; k < 4; ++k) a.mq[k] = b.mq[k];
        a.md[0] = b.md[0];
        a.md[1] = b.md[1];
    }
    L.ctas = resolve_ctas(h);
    if (b.ctas_cap > 0 && b.ctas_cap < L.ctas) L.ctas = b.ctas_cap;
    L.sms = h->sms;
    L.damp = h->beta ? SF_DAMP_ARRAY : h->sep ? SF_DAMP_SEP : SF_DAMP_NONE;
    a.sigx = h->sig[0];
    a.sigy = h->sig[1];
    a.sigz = h->sig[2];
    a.hdt = (float)(0.5 * h->dt);
    L.mode = mode;
    L.snap_slot = b.snap_slot;
    L.lz = 32;
    L.balance = (mode == SF_MODE_GRAD && h->balance_grad >= 0) ? h->balance_grad : h->balance;
    // PDL only after a standalone injection kernel: stencil -> stencil gains nothing measurable
    // (a persistent launch cannot co-reside with the previous one), and plain launches keep
    // the sampled event timing of the stencil exact
    L.pdl = (h->pdl && h->prev_inject) ? 1 : 0;
    h->prev_inject = false;
    // z remainder (SF_OPT_ZSPLIT): n2 = 128 k + rem with 0 < rem <= 64 -> the 128-column tiles
    // cover [0, 128 k) and a second launch of narrow 56 x 32 tiles covers the rem columns
    // (the 128-column tiles there would be mostly idle lanes; configs[4]: 400 = 3 x 128 + 16).
    // Only for r >= 5, where the kernel is latency-bound and idle lanes cost time (400^3 so12:
    // 256 vs 296 us); at r <= 4 it runs at the HBM roofline and the extra launch costs
    // (400^3 so8: 233 vs 225 us).
    int64_t zrem = 0;
    if (L.variant == SF_VAR_TMA && h->ndim == 3 && h->zsplit && (L.vy == 2 || L.vy == 4) && h->r >= 5) {
        const int64_t rem = a.n2 % tile_tz(h, 2);
        if (rem > 0 && rem <= 64 && a.n2 > tile_tz(h, 2)) zrem = rem;
    }
    auto build_maps = [&](SfTmaMaps &m, int TZ, int BY) -> sf_status {
        memset(&m, 0, sizeof m);
        const int HZ = ((h->r + 3) / 4) * 4;
        const int64_t d3[3] = {h->nb[2], h->nb[1], h->nb[0]};
        const uint32_t bcur[3] = {(uint32_t)(TZ + 2 * HZ), (uint32_t)(BY + 2 * h->r), 1};
        const uint32_t bpl[3] = {(uint32_t)TZ, (uint32_t)BY, 1};
        sf_status s;
        if ((s = make_map(&m.cur, b.cur, 3, d3, bcur))) return s;
        if ((s = make_map(&m.old, b.out, 3, d3, bpl))) return s;
        if ((s = make_map(&m.c3, h->c3, 3, d3, bpl))) return s;
        if (h->beta && (s = make_map(&m.beta, h->beta, 3, d3, bpl))) return s;
        if (mode == SF_MODE_GRAD) {
            const int64_t d4[4] = {h->nb[2], h->nb[1], h->nb[0], b.nsnap};
            const uint32_t b4[4] = {(uint32_t)TZ, (uint32_t)BY, 1, 1};
            if ((s = make_map(&m.snap, b.snaps, 4, d4, b4, h->snap_half))) return s;
            if ((s = make_map(&m.grad, b.grad, 3, d3, bpl))) return s;
        }
        return SF_OK;
    };
    SfTmaMaps maps, nmaps;
    memset(&maps, 0, sizeof maps);
    if (L.variant == SF_VAR_TMA) {
        sf_status s;
        if ((s = build_maps(maps, tile_tz(h, L.vy), tile_by(L.vy)))) return s;
        if (zrem && (s = build_maps(nmaps, NARROW_TZ, narrow_by(L.vy)))) return s;
    }
    L.maps = &maps;
    // fuse only small point sets (a few shots' sources): large sets (receiver grids) would
    // put dependent table loads on the stencil's critical path -> standalone kernels (an
    // in-kernel injection of receiver surfaces from a dense per-plane table, its loads
    // pipelined two planes ahead, measured 9 % slower even where inactive and 23 % slower on
    // configs[2]: DESIGN.md section 7).  Not with the z split (the fused lists index the
    // 128-column tiles only)
    if (L.variant == SF_VAR_TMA && !zrem && mode != SF_MODE_GRAD && b.inj && b.inj->ntgt > 0 &&
        b.inj->ntgt <= h->fuse_max && b.inj_vals) {
        sf_status s = ensure_inj_tiles(h, *b.inj, L.vy);
        if (s) return s;
        a.inj_beg = b.inj->tiles.beg;
        a.inj_q = b.inj->tiles.q;
        a.inj_lj = b.inj->tiles.lj;
        a.inj_t = b.inj->tiles.t;
        a.inj_rowptr = b.inj->j_rowptr;
        a.inj_pt = b.inj->j_pt;
        a.inj_coef = b.inj->j_coef;
        a.inj_vals = b.inj_vals;
        *fused = true;
    }
    // (records are interpolated by k_interp_ell on the side stream, concurrently with the
    //  next step: no in-kernel interpolation)

    if (b.bidir) {
        if (L.variant != SF_VAR_TMA || zrem || L.vy != 2)
            return sf_set_error(SF_ERR_INVALID_ARG, "one-launch schedule needs the TMA kernel (7-warp layout) without a z split");
        a.bidir = 1;
        a.sig = b.nosig ? nullptr : h->sigc;
        h->last_tiles = (int)(((a.n2 + tile_tz(h, L.vy) - 1) / tile_tz(h, L.vy)) *
                              ((a.n1 + tile_by(L.vy) - 1) / tile_by(L.vy)));
    }
    if (b.dry) return SF_OK;
    cudaError_t e;
    {
        ProfScope ps(h, PK_STENCIL, st);  // one scope over both launches of a z split
        if (zrem) a.n2t = a.n2 - zrem;
        e = launch_step_r(h->r, L, a, st);
        if (e == cudaSuccess && zrem) {
            SfLaunch Ln = L;
            Ln.lz = 8;
            Ln.maps = &nmaps;
            SfStepArgs an = a;
            an.zbase = a.n2 - zrem;
            an.n2t = a.n2;
            h->n_all++;
            h->n_kind[PK_OTHER]++;  // counted; its time is inside the stencil scope
            e = launch_step_r(h->r, Ln, an, st);
        }
    }
    if (e != cudaSuccess) return sf_set_error(SF_ERR_CUDA, "stencil launch: %s", cudaGetErrorString(e));
    return SF_OK;
}

static sf_status launch_interp(sf_handle *h, const SfSparse &sp, const float *u, float *out,
                               cudaStream_t st)
{
    if (sp.np == 0 || !out) return SF_OK;
    ProfScope ps(h, PK_INTERP, st);
    // grid-stride over at most one block per SM: the record kernel runs beside the persistent
    // stencil (side stream), where fewer, longer-lived blocks disturb it less
    // 512 threads per block (measured on configs[1]: the records' cost beside the stencil fell
    // from 4-5 % with 128-thread blocks to ~2 %: more loads in flight per block, fewer blocks
    // squeezed in beside the persistent CTAs)
    const int tpb = 512;
    const int nb = std::min((sp.np + tpb - 1) / tpb, h->sms);
    k_interp_ell<<<nb, tpb, 0, st>>>(u, sp.e_idx, sp.e_w, sp.i_owned, sp.np, sp.ik, out);
    SF_CUDA_TRY(cudaGetLastError());
    return SF_OK;
}


static sf_status launch_inject(sf_handle *h, const SfSparse &sp, float *u, const float *vals,
                               float *snap_patch, const float *grad_snap, float *grad, float gscale,
                               cudaStream_t st)
{
    if (sp.ntgt == 0 || !vals) return SF_OK;
    ProfScope ps(h, PK_INJECT, st);
    // (SF_OPT_PDL: launched with programmatic stream serialisation -- its launch overlaps the
    // stencil's tail; the kernel waits for the stencil's writes before touching them)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((sp.ntgt + 127) / 128));
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = h->pdl ? 1 : 0;
    h->prev_inject = true;
    const int half = h->snap_half ? 1 : 0;
    if (sp.jk > 0)
        SF_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_inject_ell, u, (const int64_t *)sp.j_tgt, sp.jk, (const int *)sp.ej_pt,
                                       (const float *)sp.ej_coef, sp.ntgt, vals, (void *)snap_patch,
                                       (const void *)grad_snap, grad, gscale, half));
    else
        SF_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_inject, u, (const int64_t *)sp.j_tgt, (const int *)sp.j_rowptr,
                                       (const int *)sp.j_pt, (const float *)sp.j_coef, sp.ntgt, vals,
                                       (void *)snap_patch, (const void *)grad_snap, grad, gscale, half));
    return SF_OK;
}

// ------------------------------------------------------------------ sparse tables
static void free_sparse(SfSparse &s)
{
    cudaFree(s.i_owned);
    cudaFree(s.j_tgt);
    cudaFree(s.j_rowptr);
    cudaFree(s.j_pt);
    cudaFree(s.j_coef);
    free_inj(s.tiles);
    cudaFree(s.e_idx);
    cudaFree(s.e_w);
    cudaFree(s.ej_pt);
    cudaFree(s.ej_coef);
    cudaFree(s.jl_bnd);
    cudaFree(s.jl_int);
    s = SfSparse{};
}


// Reading C11: pos = x/h; base = min(floor(pos), n-2); xi = pos - base; weights =
// product of (1 - xi) / xi; corners ordered last-axis fastest; outside [0, n-1] is an
// error.  Slab mode (C18): axis-0 corners are mapped to the local buffer; a record row
// is owned by the rank owning the base plane; injection corners by the rank owning
// the corner's plane.
// Host half of the sparse tables (coordinates only: runs before / while m is uploaded).
struct SparsePlan {
    int np = 0, nc = 0;
    std::vector<int> owned;
    std::vector<int64_t> tgt, etgt;  // injection targets (CSR rows) / per-entry targets
    std::vector<int> rowptr, pt;
    std::vector<double> ew;          // per-entry interpolation weight (the coefficient's W)
    int K = 1;                       // interpolation ELL slots
    std::vector<int64_t> eidx;       // [K][np]
    std::vector<float> ewf;          // [K][np]
};

static sf_status plan_sparse(const sf_handle *h, int np, const double *coords, SparsePlan &pl,
                             const char *what)
{
    pl = SparsePlan{};
    if (np <= 0) return SF_OK;
    if (!coords) return sf_set_error(SF_ERR_INVALID_ARG, "%s coordinates are NULL", what);
    const int nd = h->ndim;
    const int nc = 1 << nd;
    std::vector<int64_t> iidx((size_t)np * nc);
    std::vector<float> iw((size_t)np * nc);
    std::vector<int> owned(np, 1);
    struct Ent {
        int64_t tgt;
        int pt;
        int c;
        double w;
    };
    std::vector<Ent> ents;
    ents.reserve((size_t)np * nc);
    for (int p = 0; p < np; ++p) {
        int64_t base[3];
        double xi[3];
        for (int a = 0; a < nd; ++a) {
            const double x = coords[(size_t)p * nd + a];
            const double pos = x / h->h;
            const int64_t n = h->gshape[a];
            if (!(pos >= 0.0) || pos > (double)(n - 1))
                return sf_set_error(SF_ERR_OUT_OF_DOMAIN,
                                    "%s %d coordinate %d = %g m outside [0, %g] m", what, p, a, x,
                                    (double)(n - 1) * h->h);
            int64_t b = (int64_t)std::floor(pos);
            if (b > n - 2) b = n - 2;
            base[a] = b;
            xi[a] = pos - (double)b;
        }
        if (h->nranks > 1) owned[p] = (base[0] >= h->x0 && base[0] < h->x0 + h->n0_loc) ? 1 : 0;
        for (int c = 0; c < nc; ++c) {
            double wt = 1.0;
            int64_t off = 0;
            int64_t gx = 0;
            for (int a = 0; a < nd; ++a) {
                const int bit = (c >> (nd - 1 - a)) & 1;
                wt *= bit ? xi[a] : (1.0 - xi[a]);
                int64_t ia = base[a] + bit;
                if (a == 0) {
                    gx = ia;
                    ia = ia - h->x0 + (h->nranks > 1 ? h->r : 0);
                }
                off = off * h->nb[a] + ia;
            }
            // interpolation corner (zero weights dropped from the ELL below; non-owned rows
            // point at a valid in-buffer index only when owned)
            const bool inbuf = (h->nranks == 1) || owned[p];
            iidx[(size_t)p * nc + c] = inbuf ? off : 0;
            iw[(size_t)p * nc + c] = inbuf ? (float)wt : 0.0f;
            const bool own_corner =
                (h->nranks == 1) || (gx >= h->x0 && gx < h->x0 + h->n0_loc);
            if (wt != 0.0 && own_corner) ents.push_back({off, p, c, wt});
        }
    }
    // deterministic order: target, then point, then corner (unique keys); points given in
    // grid order (receiver grids) arrive sorted already -> skip the sort
    auto key_less = [](const Ent &a, const Ent &b) {
        return std::tie(a.tgt, a.pt, a.c) < std::tie(b.tgt, b.pt, b.c);
    };
    if (!std::is_sorted(ents.begin(), ents.end(), key_less)) std::sort(ents.begin(), ents.end(), key_less);
    pl.pt.reserve(ents.size());
    pl.etgt.reserve(ents.size());
    pl.ew.reserve(ents.size());
    for (size_t e = 0; e < ents.size(); ++e) {
        if (e == 0 || ents[e].tgt != ents[e - 1].tgt) {
            pl.tgt.push_back(ents[e].tgt);
            pl.rowptr.push_back((int)e);
        }
        pl.pt.push_back(ents[e].pt);
        pl.etgt.push_back(ents[e].tgt);
        pl.ew.push_back(ents[e].w);
    }
    pl.rowptr.push_back((int)ents.size());
    // interpolation ELL (slot-major): nonzero corners in corner order, zero padded
    int K = 1;
    for (int p = 0; p < np; ++p) {
        int k = 0;
        for (int c = 0; c < nc; ++c) k += iw[(size_t)p * nc + c] != 0.0f;
        K = std::max(K, k);
    }
    pl.eidx.assign((size_t)K * np, 0);
    pl.ewf.assign((size_t)K * np, 0.0f);
    for (int p = 0; p < np; ++p) {
        int k = 0;
        for (int c = 0; c < nc; ++c) {
            const float w = iw[(size_t)p * nc + c];
            if (w == 0.0f) continue;
            pl.eidx[(size_t)k * np + p] = iidx[(size_t)p * nc + c];
            pl.ewf[(size_t)k * np + p] = w;
            ++k;
        }
    }
    pl.np = np;
    pl.nc = nc;
    pl.K = K;
    pl.owned = std::move(owned);
    return SF_OK;
}

// Device half: upload the planned tables, injection coefficients W dt^2 / m at the targets.
static sf_status commit_sparse(sf_handle *h, const SparsePlan &pl, const float *m_dev, SfSparse &out)
{
    out = SfSparse{};
    if (pl.np <= 0) return SF_OK;
    out.np = pl.np;
    out.nc = pl.nc;
    out.h_tgt = pl.tgt;
    out.ntgt = (int)pl.tgt.size();
    out.nent = (int)pl.pt.size();
    sf_status s;
    if (h->nranks > 1 && (s = upload(&out.i_owned, pl.owned))) return s;
    if (out.ntgt > 0) {
        if ((s = upload(&out.j_tgt, pl.tgt))) return s;
        if ((s = upload(&out.j_rowptr, pl.rowptr))) return s;
        if ((s = upload(&out.j_pt, pl.pt))) return s;
        int64_t *d_etgt = nullptr;
        double *d_ew = nullptr;
        if ((s = upload(&d_etgt, pl.etgt))) return s;
        if ((s = upload(&d_ew, pl.ew))) return s;
        SF_CUDA_TRY(cudaMalloc(&out.j_coef, sizeof(float) * out.nent));
        k_inject_coef<<<(out.nent + 255) / 256, 256>>>(m_dev, d_etgt, d_ew, out.nent, h->dt * h->dt,
                                                       out.j_coef);
        SF_CUDA_TRY(cudaGetLastError());
        SF_CUDA_TRY(cudaDeviceSynchronize());
        cudaFree(d_etgt);
        cudaFree(d_ew);
        // injection ELL (slot-major), when every target has few contributions
        int kmax = 0;
        for (size_t t = 0; t + 1 < pl.rowptr.size(); ++t) kmax = std::max(kmax, pl.rowptr[t + 1] - pl.rowptr[t]);
        if (kmax <= 8) {
            out.jk = kmax;
            SF_CUDA_TRY(cudaMalloc(&out.ej_pt, sizeof(int) * (size_t)kmax * out.ntgt));
            SF_CUDA_TRY(cudaMalloc(&out.ej_coef, sizeof(float) * (size_t)kmax * out.ntgt));
            k_csr_to_ell<<<(out.ntgt + 255) / 256, 256>>>(out.j_rowptr, out.j_pt, out.j_coef, out.ntgt, kmax,
                                                          out.ej_pt, out.ej_coef);
            SF_CUDA_TRY(cudaGetLastError());
            SF_CUDA_TRY(cudaDeviceSynchronize());
        }
    }
    out.ik = pl.K;
    if ((s = upload(&out.e_idx, pl.eidx))) return s;
    if ((s = upload(&out.e_w, pl.ewf))) return s;
    return SF_OK;
}

// ------------------------------------------------------------------ create / destroy
static sf_status validate_desc(const sf_desc *d)
{
    if (!d) return sf_set_error(SF_ERR_INVALID_ARG, "desc is NULL");
    if (d->ndim != 2 && d->ndim != 3) return sf_set_error(SF_ERR_SHAPE, "ndim %d not 2 or 3", d->ndim);
    for (int a = 0; a < d->ndim; ++a)
        if (d->shape[a] < 2) return sf_set_error(SF_ERR_SHAPE, "shape[%d] = %lld < 2", a, (long long)d->shape[a]);
    if (d->space_order < 2 || d->space_order > 16 || (d->space_order & 1))
        return sf_set_error(SF_ERR_ORDER, "space_order %d not in {2,4,...,16}", d->space_order);
    if (!d->m) return sf_set_error(SF_ERR_INVALID_ARG, "m is NULL");
    if (d->nt < 2) return sf_set_error(SF_ERR_INVALID_ARG, "nt = %d < 2", d->nt);
    if (!(d->dt > 0.0)) return sf_set_error(SF_ERR_INVALID_ARG, "dt = %g <= 0", d->dt);
    if (!(d->h > 0.0)) return sf_set_error(SF_ERR_INVALID_ARG, "h = %g <= 0", d->h);
    if (d->nsrc < 0 || d->nrec < 0) return sf_set_error(SF_ERR_INVALID_ARG, "negative point count");
    if (d->sigma[0] || d->sigma[1] || d->sigma[2]) {
        if (d->damp) return sf_set_error(SF_ERR_INVALID_ARG, "damp and sigma profiles are exclusive");
        for (int a = 0; a < 3; ++a) {
            if ((a < d->ndim) != (d->sigma[a] != nullptr))
                return sf_set_error(SF_ERR_INVALID_ARG, "sigma[%d] must be %s", a, a < d->ndim ? "given" : "NULL");
            if (a < d->ndim)
                for (int64_t i = 0; i < d->shape[a]; ++i)
                    if (!(d->sigma[a][i] >= 0.0f) || !std::isfinite(d->sigma[a][i]))
                        return sf_set_error(SF_ERR_INVALID_ARG, "sigma[%d][%lld] = %g", a, (long long)i,
                                            (double)d->sigma[a][i]);
        }
    }
    return SF_OK;
}

extern "C" void sf_destroy(sf_handle *h)
{
    if (!h) return;
    // the pool frees below are ordered on the legacy stream: finish any work still using
    // the handle's buffers on other (possibly non-blocking) streams first
    cudaDeviceSynchronize();
    cudaFree(h->c3);
    cudaFree(h->beta);
    for (int a = 0; a < 3; ++a) cudaFree(h->sig[a]);
    cudaFree(h->partial);
    cudaFree(h->dJ);
    free_sparse(h->src);
    free_sparse(h->rec);
    cudaFree(h->tb_buf);
    cudaFree(h->tb_beg);
    cudaFree(h->tb_q);
    cudaFree(h->tb_p);
    cudaFree(h->tb_t);
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    if (h->ev_ready) cudaEventDestroy(h->ev_ready);
    for (int k = 0; k < 2; ++k)
        if (h->ev_itp[k]) cudaEventDestroy(h->ev_itp[k]);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->comm_stream) cudaStreamDestroy(h->comm_stream);
    if (h->hi_stream) cudaStreamDestroy(h->hi_stream);
    sf_comm_p2p_release(h);
    if (h->p2p_flags) (cudaFree)(h->p2p_flags);
    if (h->sigc) (cudaFree)(h->sigc);
    if (h->ev_pre) cudaEventDestroy(h->ev_pre);
    if (h->ev_bnd) cudaEventDestroy(h->ev_bnd);
    if (h->ev_xch) cudaEventDestroy(h->ev_xch);
    drop_graphs(h);
    if (h->gstream) cudaStreamDestroy(h->gstream);
    if (h->ev_gin) cudaEventDestroy(h->ev_gin);
    if (h->ev_gout) cudaEventDestroy(h->ev_gout);
    delete h;
}

static sf_status create_common(const sf_desc *d, sf_handle *h)
{
    if (const char *e = getenv("SF_L2_PREFETCH")) h->l2_prefetch = atoi(e);
    // sparse tables first (host work on the coordinates only: overlaps an upload of m still
    // in flight, sf_forward_host), receivers -- the large set -- before sources
    SparsePlan prec, psrc;
    {
        const int r0 = d->space_order / 2;
        h->r = r0;
        h->h = d->h;
        sf_status s0;
        if ((s0 = plan_sparse(h, d->nrec, d->rec_coords, prec, "receiver"))) return s0;
        if ((s0 = plan_sparse(h, d->nsrc, d->src_coords, psrc, "source"))) return s0;
    }
    {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
            h->sms = v;
    }
    const int r = d->space_order / 2;
    h->so = d->space_order;
    h->r = r;
    h->nt = d->nt;
    h->dt = d->dt;
    h->h = d->h;
    double w[SF_MAXR + 1];
    sf_fd_weights(d->space_order, w);
    for (int k = 0; k <= SF_MAXR; ++k) h->w.w[k] = k <= r ? (float)(w[k] / (d->h * d->h)) : 0.0f;
    // coefficient hoisting (same bytes as streaming m and eta)
    SF_CUDA_TRY(cudaMalloc(&h->c3, sizeof(float) * h->N));
    h->damp = d->damp != nullptr;
    h->sep = d->sigma[0] != nullptr;
    if (h->sep) {
        // local profiles: x over the buffer planes (slab halo planes outside the global grid
        // get 0: they are never computed), y and z whole
        const int nd = d->ndim;
        const int64_t off = h->x0 - (h->nranks > 1 ? h->r : 0);
        std::vector<float> px((size_t)h->nb[0], 0.0f);
        for (int64_t i = 0; i < h->nb[0]; ++i) {
            const int64_t g = off + i;
            if (g >= 0 && g < d->shape[0]) px[(size_t)i] = d->sigma[0][g];
        }
        sf_status s;
        if ((s = upload(&h->sig[0], px))) return s;
        for (int a = 1; a < nd; ++a) {
            std::vector<float> pa(d->sigma[a], d->sigma[a] + d->shape[a]);
            if ((s = upload(&h->sig[a == nd - 1 ? 2 : 1], pa))) return s;
        }
        const int64_t n1 = nd == 3 ? h->nb[1] : 1, n2 = nd == 3 ? h->nb[2] : h->nb[1];
        k_hoist_sep<<<1184, 256>>>(d->m, h->N, n1, n2, d->dt, h->sig[0], h->sig[1], h->sig[2], h->c3);
    } else {
        if (h->damp) SF_CUDA_TRY(cudaMalloc(&h->beta, sizeof(float) * h->N));
        k_hoist<<<1184, 256>>>(d->m, d->damp, h->N, d->dt, h->c3, h->beta);
    }
    SF_CUDA_TRY(cudaGetLastError());
    // min m over the computed planes -> CFL (SF_ERR_CFL) and positivity (SF_ERR_INVALID_ARG)
    unsigned int *dmin = nullptr;
    int *dbad = nullptr;
    SF_CUDA_TRY(cudaMalloc(&dmin, sizeof(unsigned int)));
    SF_CUDA_TRY(cudaMalloc(&dbad, sizeof(int)));
    const unsigned int init = 0x7f7fffffu;
    SF_CUDA_TRY(cudaMemcpy(dmin, &init, sizeof init, cudaMemcpyHostToDevice));
    SF_CUDA_TRY(cudaMemset(dbad, 0, sizeof(int)));
    const int64_t plane = h->N / h->nb[0];
    k_min_m<<<592, 256>>>(d->m + h->xa * plane, (h->xb - h->xa) * plane, dmin, dbad);
    SF_CUDA_TRY(cudaGetLastError());
    unsigned int minbits = 0;
    int bad = 0;
    SF_CUDA_TRY(cudaMemcpy(&minbits, dmin, sizeof minbits, cudaMemcpyDeviceToHost));
    SF_CUDA_TRY(cudaMemcpy(&bad, dbad, sizeof bad, cudaMemcpyDeviceToHost));
    cudaFree(dmin);
    cudaFree(dbad);
    if (bad) return sf_set_error(SF_ERR_INVALID_ARG, "m has a non-positive or non-finite value");
    float mmin;
    memcpy(&mmin, &minbits, sizeof mmin);
    double sabs = 0.0;
    for (int k = 0; k <= r; ++k) sabs += (k ? 2.0 : 1.0) * std::fabs(w[k]);
    const double vmax = 1.0 / std::sqrt((double)mmin);
    const double courant = d->dt * vmax / d->h;
    const double lim = 2.0 / std::sqrt((double)d->ndim * sabs);
    if (courant > lim)
        return sf_set_error(SF_ERR_CFL, "Courant number %.4f exceeds the stability limit %.4f "
                            "(so %d, %dD)", courant, lim, d->space_order, d->ndim);
    sf_status s;
    if ((s = commit_sparse(h, psrc, d->m, h->src))) return s;
    if ((s = commit_sparse(h, prec, d->m, h->rec))) return s;
    SF_CUDA_TRY(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    SF_CUDA_TRY(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
    {
        int lo = 0, hi = 0;
        SF_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        SF_CUDA_TRY(cudaStreamCreateWithPriority(&h->hi_stream, cudaStreamNonBlocking, hi));
    }
    SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_pre, cudaEventDisableTiming));
    SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming));
    SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_xch, cudaEventDisableTiming));
    h->split = h->nranks > 1;
    SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_ready, cudaEventDisableTiming));
    SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_itp[0], cudaEventDisableTiming));
    SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_itp[1], cudaEventDisableTiming));
    SF_CUDA_TRY(cudaMalloc(&h->partial, sizeof(double) * 1024));
    SF_CUDA_TRY(cudaMalloc(&h->dJ, sizeof(double)));
    // one-launch schedule counters (stream memory operations: plain cudaMalloc, not the pool)
    SF_CUDA_TRY((cudaMalloc)((void **)&h->sigc, 2 * sizeof(unsigned int)));
    SF_CUDA_TRY(cudaMemset(h->sigc, 0, 2 * sizeof(unsigned int)));
    // the tables the time loops would otherwise build on first use (no per-call
    // allocation): fused-injection lists for the default tile shape, split-schedule lists in
    // slab mode.  (A later sf_set_tuning to another tile shape rebuilds the lists once.)
    if (resolve_variant(h) == SF_VAR_TMA) {
        if (h->src.ntgt > 0 && h->src.ntgt <= h->fuse_max && (s = ensure_inj_tiles(h, h->src, resolve_vy(h, SF_MODE_PLAIN)))) return s;
        if (h->rec.ntgt > 0 && h->rec.ntgt <= h->fuse_max && (s = ensure_inj_tiles(h, h->rec, resolve_vy(h, SF_MODE_PLAIN)))) return s;
    }
    if (h->split) {
        if (h->src.ntgt > 0 && (s = ensure_split_lists(h, h->src))) return s;
        if (h->rec.ntgt > 0 && (s = ensure_split_lists(h, h->rec))) return s;
    }
    SF_CUDA_TRY(cudaDeviceSynchronize());
    return SF_OK;
}

extern "C" sf_status sf_create(const sf_desc *d, sf_handle **out)
{
    if (!out) return sf_set_error(SF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    sf_status s = validate_desc(d);
    if (s) return s;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return sf_set_error(SF_ERR_CUDA, "no CUDA device (libsf has no CPU fallback)");
    sf_handle *h = new sf_handle();
    h->ndim = d->ndim;
    h->N = 1;
    for (int a = 0; a < d->ndim; ++a) {
        h->gshape[a] = d->shape[a];
        h->nb[a] = d->shape[a];
        h->N *= d->shape[a];
    }
    h->xa = 0;
    h->xb = d->shape[0];
    h->n0_loc = d->shape[0];
    s = create_common(d, h);
    if (s) {
        sf_destroy(h);
        return s;
    }
    *out = h;
    return SF_OK;
}

extern "C" sf_status sf_slab_plan(int64_t n0, int space_order, int rank, int nranks, int64_t *x0,
                                  int64_t *n0_loc)
{
    if (!x0 || !n0_loc || nranks < 1 || rank < 0 || rank >= nranks)
        return sf_set_error(SF_ERR_INVALID_ARG, "bad slab plan arguments");
    if (space_order < 2 || space_order > 16 || (space_order & 1))
        return sf_set_error(SF_ERR_ORDER, "space_order %d", space_order);
    const int64_t base = n0 / nranks, rem = n0 % nranks;
    *n0_loc = base + (rank < rem ? 1 : 0);
    *x0 = rank * base + std::min<int64_t>(rank, rem);
    if (*n0_loc < space_order / 2)
        return sf_set_error(SF_ERR_SHAPE, "slab of %lld planes < r = %d", (long long)*n0_loc,
                            space_order / 2);
    return SF_OK;
}

extern "C" sf_status sf_slab_halo_plan(int64_t n0, int space_order, int rank, int nranks, int64_t plan[7])
{
    if (!plan) return sf_set_error(SF_ERR_INVALID_ARG, "plan is NULL");
    int64_t x0, nl;
    sf_status s = sf_slab_plan(n0, space_order, rank, nranks, &x0, &nl);
    if (s) return s;
    const int64_t r = space_order / 2;
    plan[0] = r;        // owned planes [r, 2r) -> left neighbour's right halo
    plan[1] = 0;        // left halo [0, r) <- left neighbour's last owned planes
    plan[2] = nl;       // owned planes [nl, nl + r) -> right neighbour's left halo
    plan[3] = nl + r;   // right halo [nl + r, nl + 2r) <- right neighbour's first owned planes
    plan[4] = r;
    plan[5] = rank > 0;
    plan[6] = rank < nranks - 1;
    return SF_OK;
}

extern "C" sf_status sf_sparse_owner(int64_t n0, int space_order, int nranks, double h,
                                     double coord0, int *owner)
{
    if (!owner || !(h > 0) || nranks < 1) return sf_set_error(SF_ERR_INVALID_ARG, "bad arguments");
    const double pos = coord0 / h;
    if (!(pos >= 0.0) || pos > (double)(n0 - 1))
        return sf_set_error(SF_ERR_OUT_OF_DOMAIN, "coordinate %g outside the grid", coord0);
    int64_t b = (int64_t)std::floor(pos);
    if (b > n0 - 2) b = n0 - 2;
    for (int p = 0; p < nranks; ++p) {
        int64_t x0, nl;
        sf_status s = sf_slab_plan(n0, space_order, p, nranks, &x0, &nl);
        if (s) return s;
        if (b >= x0 && b < x0 + nl) {
            *owner = p;
            return SF_OK;
        }
    }
    return sf_set_error(SF_ERR_OUT_OF_DOMAIN, "no owner");
}

extern "C" sf_status sf_create_slab(const sf_desc *d, void *comm, int rank, int nranks,
                                    sf_handle **out)
{
    if (!out) return sf_set_error(SF_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    sf_status s = validate_desc(d);
    if (s) return s;
    if (nranks > 1 && !comm) return sf_set_error(SF_ERR_INVALID_ARG, "comm is NULL");
    int64_t x0, nl;
    if ((s = sf_slab_plan(d->shape[0], d->space_order, rank, nranks, &x0, &nl))) return s;
    sf_handle *h = new sf_handle();
    h->ndim = d->ndim;
    h->rank = rank;
    h->nranks = nranks;
    h->comm = comm;
    h->x0 = x0;
    h->n0_loc = nl;
    const int r = d->space_order / 2;
    for (int a = 0; a < d->ndim; ++a) {
        h->gshape[a] = d->shape[a];
        h->nb[a] = d->shape[a];
    }
    if (nranks > 1) {
        h->nb[0] = nl + 2 * r;
        h->xa = r;
        h->xb = r + nl;
    } else {
        h->xa = 0;
        h->xb = d->shape[0];
    }
    h->N = 1;
    for (int a = 0; a < d->ndim; ++a) h->N *= h->nb[a];
    s = create_common(d, h);
    if (s) {
        sf_destroy(h);
        return s;
    }
    *out = h;
    return SF_OK;
}

// ------------------------------------------------------------------ tuning / profiling
extern "C" sf_status sf_set_tuning(sf_handle *h, int variant, int vy, int ctas)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    if (variant < 0 || variant > 2 || vy < 0 || vy > 4 || ctas < 0)
        return sf_set_error(SF_ERR_INVALID_ARG, "bad tuning (%d, %d, %d)", variant, vy, ctas);
    if (variant == SF_VAR_TMA && !tma_ok(h))
        return sf_set_error(SF_ERR_INVALID_ARG, "TMA variant needs 3D and n2 %% 4 == 0");
    h->variant = variant;
    h->vy = vy;
    h->vy_grad = 0;
    h->balance_grad = -1;
    h->ctas = ctas;
    drop_graphs(h);
    return SF_OK;
}

// Setup-time tuning (the GPU counterpart of the paper's runtime block-size auto-tuning of
// its loop engine): time `steps` stencil steps (no sparse work) of every feasible
// launch configuration on the caller's scratch state and keep the fastest.  Every
// configuration computes the same bits, so the choice only changes speed.
extern "C" sf_status sf_autotune(sf_handle *h, float *u, int steps, int *chosen, float *ms_out, void *stream)
{
    if (!h || !u || steps < 1) return sf_set_error(SF_ERR_INVALID_ARG, "autotune: NULL handle/state or steps < 1");
    cudaStream_t st = S(stream);
    struct Cand {
        int variant, vy, zsplit, bal;
    };
    std::vector<Cand> cands;
    if (tma_ok(h)) {
        // the balanced work split only where the kernel is FP-bound (r >= 5): at r <= 4 its
        // re-read halo rows cost HBM time (configs[1]: 0.150 vs 0.121 ms)
        for (int bal = 0; bal <= (h->r >= 5 ? 1 : 0); ++bal) {
            cands.push_back({SF_VAR_TMA, 2, 1, bal});
            if (h->r >= 5) cands.push_back({SF_VAR_TMA, 2, 0, bal});  // narrow remainder tiles off
            cands.push_back({SF_VAR_TMA, 1, 1, bal});
            if (h->r >= 5 && h->ndim == 3) cands.push_back({SF_VAR_TMA, 3, 1, bal});  // wide layout
            cands.push_back({SF_VAR_TMA, 4, 1, bal});  // warp-specialised 8-consumer-warp layout
        }
    }
    cands.push_back({SF_VAR_GENERIC, 0, 1, 0});
    const Cand keep{h->variant, h->vy, h->zsplit ? 1 : 0, h->balance};
    const bool keep_prof = h->prof;
    h->prof = false;
    cudaEvent_t e0, e1;
    SF_CUDA_TRY(cudaEventCreate(&e0));
    SF_CUDA_TRY(cudaEventCreate(&e1));
    float best = 1e30f;
    int bi = -1;
    sf_status s = SF_OK;
    float *A = u, *B = u + h->N;
    for (size_t c = 0; c < cands.size() && !s; ++c) {
        h->variant = cands[c].variant;
        h->vy = cands[c].vy;
        h->zsplit = cands[c].zsplit != 0;
        h->balance = cands[c].bal;
        h->balance_grad = -1;
        for (int it = -2; it < steps && !s; ++it) {  // two untimed warm-up steps
            if (it == 0) SF_CUDA_TRY(cudaEventRecord(e0, st));
            StepBufs b{};
            b.cur = (it & 1) ? A : B;
            b.out = (it & 1) ? B : A;
            bool fused = false;
            s = launch_step(h, b, SF_MODE_PLAIN, st, &fused);
        }
        if (s) break;
        SF_CUDA_TRY(cudaEventRecord(e1, st));
        SF_CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        SF_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        ms /= (float)steps;
        if (ms < best) {
            best = ms;
            bi = (int)c;
        }
    }
    const Cand pick = (s || bi < 0) ? keep : cands[bi];
    h->variant = pick.variant;
    h->vy = pick.vy;
    h->zsplit = pick.zsplit != 0;
    h->balance = pick.bal;
    h->vy_grad = 0;
    h->balance_grad = -1;
    // GRAD-mode steps (the gradient's adjoint: snapshot and gradient planes streamed beside
    // the stencil) get their own layout: time the TMA layouts with the winner's z split in GRAD
    // mode on the same scratch state, with a snapshot and a gradient buffer of their own
    // (zeroed scratch: only the time counts).  Aliasing them to the state's two levels, as
    // an earlier form did, hid their 12 B/pt of HBM traffic in L2 and could pick a layout
    // whose traffic is 1.4x the algorithmic bytes in the real adjoint (configs[4], ncu:
    // profiles/r02_step_traffic_c4.json); the aliased form stays as the fallback when the
    // scratch allocation fails.
    float best_g = 1e30f;
    float *gsc = nullptr;
    if (!s && pick.variant == SF_VAR_TMA && h->ndim == 3) {
        if (cudaMalloc(&gsc, 2 * (size_t)h->N * sizeof(float)) != cudaSuccess) {
            cudaGetLastError();
            gsc = nullptr;
        } else if (cudaMemsetAsync(gsc, 0, 2 * (size_t)h->N * sizeof(float), st) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(gsc);
            gsc = nullptr;
        }
    }
    if (!s && pick.variant == SF_VAR_TMA && h->ndim == 3) {
        for (int cg = 0; cg < (h->r >= 5 ? 4 : 2); ++cg) {
            const int vg = (cg & 1) ? 4 : 2, bg = cg >> 1;
            h->vy = vg;
            h->balance = bg;
            for (int it = -2; it < steps && !s; ++it) {
                if (it == 0) SF_CUDA_TRY(cudaEventRecord(e0, st));
                StepBufs b{};
                b.cur = (it & 1) ? A : B;
                b.out = (it & 1) ? B : A;
                b.snaps = gsc ? gsc : b.cur;
                b.nsnap = 1;
                b.snap_slot = 0;
                b.grad = gsc ? gsc + h->N : b.out;
                b.gscale = 0.0f;
                bool fused = false;
                s = launch_step(h, b, SF_MODE_GRAD, st, &fused);
            }
            if (s) break;
            SF_CUDA_TRY(cudaEventRecord(e1, st));
            SF_CUDA_TRY(cudaEventSynchronize(e1));
            float ms = 0.f;
            SF_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
            ms /= (float)steps;
            if (ms < best_g) {
                best_g = ms;
                h->vy_grad = vg;
                h->balance_grad = bg;
            }
        }
        h->vy = pick.vy;
        h->balance = pick.bal;
    }
    if (gsc) cudaFree(gsc);  // (synchronises the device: setup time)
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    h->prof = keep_prof;
    drop_graphs(h);
    if (s) return s;
    if (chosen) {
        chosen[0] = pick.variant;
        chosen[1] = pick.vy;
        chosen[2] = pick.zsplit;
    }
    if (ms_out) *ms_out = best;
    return SF_OK;
}

static sf_status ensure_tb(sf_handle *h);

extern "C" sf_status sf_set_option(sf_handle *h, int option, int value)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    switch (option) {
    case SF_OPT_L2_PREFETCH:
        if (value < 0 || value > 64) return sf_set_error(SF_ERR_INVALID_ARG, "prefetch distance %d", value);
        h->l2_prefetch = value;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_SPLIT:
        if (h->nranks > 1 && !value) return sf_set_error(SF_ERR_INVALID_ARG, "slab mode always splits");
        h->split = value != 0;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_FUSE_MAX:
        if (value < 0) return sf_set_error(SF_ERR_INVALID_ARG, "fuse max %d", value);
        h->fuse_max = value;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_COMM_SMS:
        if (value < 0 || value > 64) return sf_set_error(SF_ERR_INVALID_ARG, "comm SMs %d", value);
        h->comm_sms = value;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_P2P:
        if (value) {
            if (h->nranks < 2) return sf_set_error(SF_ERR_INVALID_ARG, "SF_OPT_P2P needs a slab handle (nranks > 1)");
            for (int q = 0; q < h->nranks; ++q) {  // every rank must run the split step
                int64_t x0 = 0, nl = 0;
                sf_status s = sf_slab_plan(h->gshape[0], h->so, q, h->nranks, &x0, &nl);
                if (s) return s;
                if (nl <= 2 * h->r)
                    return sf_set_error(SF_ERR_SHAPE, "SF_OPT_P2P: rank %d owns %lld planes <= 2r", q, (long long)nl);
            }
            if (!h->p2p_flags) {
                // plain cudaMalloc (not the stream-ordered pool): CUDA IPC exports it
                SF_CUDA_TRY((cudaMalloc)((void **)&h->p2p_flags, 2 * sizeof(uint32_t)));
                SF_CUDA_TRY(cudaMemset(h->p2p_flags, 0, 2 * sizeof(uint32_t)));
                SF_CUDA_TRY(cudaDeviceSynchronize());
                h->p2p_seq = 0;
            }
        }
        h->p2p = value != 0;
        return SF_OK;
    case SF_OPT_ZSPLIT:
        h->zsplit = value != 0;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_PROF_EVERY:
        if (value < 1) return sf_set_error(SF_ERR_INVALID_ARG, "SF_OPT_PROF_EVERY %d < 1", value);
        h->prof_every = value;
        return SF_OK;
    case SF_OPT_LOOP2D:
        h->loop2d = value != 0;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_PDL:
        h->pdl = value != 0;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_ONE_LAUNCH:
        if (value < 0 || value > 2) return sf_set_error(SF_ERR_INVALID_ARG, "SF_OPT_ONE_LAUNCH %d", value);
        h->one_launch = value;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_SNAP_HALF:
        h->snap_half = value != 0;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_BALANCE:
        if (value < 0 || value > 1) return sf_set_error(SF_ERR_INVALID_ARG, "SF_OPT_BALANCE %d", value);
        h->balance = value;
        h->balance_grad = -1;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_TBLOCK:
        if (value) {
            sf_status st = ensure_tb(h);
            if (st) return st;
        }
        h->tblock = value != 0;
        drop_graphs(h);
        return SF_OK;
    case SF_OPT_GRAPH:
        if (value && !h->gstream) {
            SF_CUDA_TRY(cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
            SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_gin, cudaEventDisableTiming));
            SF_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_gout, cudaEventDisableTiming));
        }
        h->use_graph = value != 0;
        drop_graphs(h);
        return SF_OK;
    default:
        return sf_set_error(SF_ERR_INVALID_ARG, "unknown option %d", option);
    }
}

extern "C" sf_status sf_get_tuning_modes(const sf_handle *h, int *vy_grad, int *balance, int *balance_grad)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    const bool tma = resolve_variant(h) == SF_VAR_TMA;
    if (vy_grad) *vy_grad = tma ? resolve_vy(h, SF_MODE_GRAD) : 0;
    if (balance) *balance = tma ? h->balance : 0;
    if (balance_grad) *balance_grad = tma ? (h->balance_grad >= 0 ? h->balance_grad : h->balance) : 0;
    return SF_OK;
}

extern "C" sf_status sf_get_tuning(const sf_handle *h, int *variant, int *vy, int *ctas)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    const int v = resolve_variant(h);
    const int b = resolve_vy(h, SF_MODE_PLAIN);
    if (variant) *variant = v;
    if (vy) *vy = v == SF_VAR_TMA ? b : 0;
    if (ctas) *ctas = v == SF_VAR_TMA ? resolve_ctas(h) : 0;
    return SF_OK;
}

extern "C" sf_status sf_set_profiling(sf_handle *h, int on)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    h->prof = on != 0;
    return SF_OK;
}

static sf_status collect_profile(sf_handle *h, double *ms_kind, long long *n_kind, long long *nall,
                                 int reset)
{
    double tot[PK_N] = {0, 0, 0, 0};
    for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
        SF_CUDA_TRY(cudaEventSynchronize(h->ev_pool[i + 1]));
        float t = 0.f;
        SF_CUDA_TRY(cudaEventElapsedTime(&t, h->ev_pool[i], h->ev_pool[i + 1]));
        tot[h->ev_kind[i / 2]] += t;
    }
    for (int k = 0; k < PK_N; ++k) {
        if (ms_kind) ms_kind[k] = h->n_samp[k] ? tot[k] * (double)h->n_kind[k] / (double)h->n_samp[k] : 0.0;
        if (n_kind) n_kind[k] = h->n_kind[k];
    }
    if (nall) *nall = h->n_all;
    if (reset) {
        h->ev_used = 0;
        h->ev_kind.clear();
        for (int k = 0; k < PK_N; ++k) h->n_kind[k] = h->n_samp[k] = 0;
        h->n_all = 0;
    }
    return SF_OK;
}

extern "C" sf_status sf_get_profile(sf_handle *h, double *ms, long long *nst, long long *nall, int reset)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    double mk[PK_N];
    long long nk[PK_N];
    sf_status s = collect_profile(h, mk, nk, nall, reset);
    if (s) return s;
    if (ms) *ms = mk[PK_STENCIL];
    if (nst) *nst = nk[PK_STENCIL];
    return SF_OK;
}

extern "C" sf_status sf_debug_probe(sf_handle *h, float *dst, long long *one_launch_steps)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    h->probe = dst;
    if (one_launch_steps) *one_launch_steps = h->n_onelaunch;
    return SF_OK;
}

extern "C" sf_status sf_get_profile_detail(sf_handle *h, double *ms_by_kind, long long *launches_by_kind,
                                           int reset)
{
    if (!h) return sf_set_error(SF_ERR_INVALID_ARG, "handle is NULL");
    return collect_profile(h, ms_by_kind, launches_by_kind, nullptr, reset);
}

// ------------------------------------------------------------------ time loops
static sf_status post_step_exchange(sf_handle *h, float *buf, cudaStream_t st)
{
    if (h->nranks <= 1) return SF_OK;
    return sf_comm_halo_exchange(h, buf, st);
}

static sf_status swap_halves(sf_handle *h, float *a, float *b, cudaStream_t st)
{
    ProfScope ps(h, PK_OTHER, st);
    k_swap<<<1184, 256, 0, st>>>(a, b, h->N);
    SF_CUDA_TRY(cudaGetLastError());
    return SF_OK;
}

// target rows of a point set split into boundary planes [xa, xa+r) U [xb-r, xb) and the
// interior (built once per handle)
static sf_status ensure_split_lists(sf_handle *h, SfSparse &sp)
{
    if (sp.n_bnd >= 0) return SF_OK;
    const int64_t plane = h->N / h->nb[0];
    std::vector<int> bnd, itr;
    for (size_t t = 0; t < sp.h_tgt.size(); ++t) {
        const int64_t x = sp.h_tgt[t] / plane;
        if (x < h->xa + h->r || x >= h->xb - h->r) bnd.push_back((int)t);
        else itr.push_back((int)t);
    }
    sf_status s;
    if ((s = upload(&sp.jl_bnd, bnd))) return s;
    if ((s = upload(&sp.jl_int, itr))) return s;
    sp.n_bnd = (int)bnd.size();
    sp.n_int = (int)itr.size();
    return SF_OK;
}

static sf_status launch_inject_list(sf_handle *h, const SfSparse &sp, float *u, const float *vals,
                                    const int *list, int nl, float *snap_patch, const float *grad_snap,
                                    float *grad, float gscale, cudaStream_t st,
                                    const int64_t *mq = nullptr, const int64_t *md = nullptr)
{
    if (nl <= 0 || !vals) return SF_OK;
    ProfScope ps(h, PK_INJECT, st);
    SfMirror mir{};
    mir.plane = h->N / h->nb[0];
    if (mq) {
        for (int k = 0; k < 4; ++k) mir.mq[k] = mq[k];
        mir.md[0] = md[0];
        mir.md[1] = md[1];
    }
    if (sp.jk > 0) {
        k_inject_ell_list<<<(nl + 127) / 128, 128, 0, st>>>(u, sp.j_tgt, sp.jk, sp.ej_pt, sp.ej_coef, sp.ntgt,
                                                            list, nl, vals, snap_patch, grad_snap, grad, gscale,
                                                            h->snap_half ? 1 : 0, mir);
    } else {
        k_inject_csr_list<<<(nl + 127) / 128, 128, 0, st>>>(u, sp.j_tgt, sp.j_rowptr, sp.j_pt, sp.j_coef, list,
                                                            nl, vals, snap_patch, grad_snap, grad, gscale,
                                                            h->snap_half ? 1 : 0, mir);
    }
    SF_CUDA_TRY(cudaGetLastError());
    return SF_OK;
}

// Split step with the peer-store halo exchange (SF_OPT_P2P).  High-priority
// stream: the boundary planes by the thread-per-point kernel, which also stores each owned
// boundary plane into the neighbour's halo of the same level (peer-mapped pointer), and
// their injection (mirrored likewise); then one counter write per neighbour.  The main
// stream computes the interior meanwhile and finally waits until both neighbours' counters
// reach this step (their planes are in this rank's halo).  Ordering across ranks:
//   RAW  the halo of level n+1 is read (next step's boundary launch, this level's
//        record) only after the counter wait of step n;
//   WAR  a neighbour overwrites the buffer of this rank's `cur` level (its halo) at step
//        n+1, after this step's counter -- written after this rank's last reads of that halo
//        (the boundary launch above and the side-stream record of `cur`).
// The boundary launch uses the generic kernel: a mirror test in the hot TMA loop measured
// 17 % slower on configs[1], and the boundary launch is 2r planes (the TMA kernel would
// re-read 2r warm-up planes for them anyway).
static sf_status do_step_p2p(sf_handle *h, const StepBufs &b, StepBufs bb, StepBufs bi, int mode,
                             float *snap_patch, const float *grad_snap, cudaStream_t st)
{
    sf_status s;
    const int64_t r = h->r;
    const int ob = b.out == h->p2p_own[0] ? 0 : b.out == h->p2p_own[1] ? 1 : -1;
    if (ob < 0) return sf_set_error(SF_ERR_INVALID_ARG, "P2P step on a buffer outside the published state");
    int64_t plan[7], qp[7];
    if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank, h->nranks, plan))) return s;
    const int64_t plane = h->N / h->nb[0];
    auto delta = [](const float *to, const float *from) {
        return (int64_t)(reinterpret_cast<uintptr_t>(to) - reinterpret_cast<uintptr_t>(from));
    };
    int64_t mq[4] = {0, 0, 0, 0}, md[2] = {0, 0};
    if (plan[5]) {  // owned [r, 2r) -> left neighbour's right halo
        if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank - 1, h->nranks, qp))) return s;
        mq[0] = plan[0];
        mq[1] = plan[0] + r;
        md[0] = delta(h->p2p_nbr[0][ob] + qp[3] * plane, b.out + plan[0] * plane);
    }
    if (plan[6]) {  // owned [nl, nl + r) -> right neighbour's left halo
        if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank + 1, h->nranks, qp))) return s;
        mq[2] = plan[2];
        mq[3] = plan[2] + r;
        md[1] = delta(h->p2p_nbr[1][ob] + qp[1] * plane, b.out + plan[2] * plane);
    }
    bb.force_generic = true;
    bb.mq = mq;
    bb.md = md;
    bool fused = false, f2 = false;
    SF_CUDA_TRY(cudaEventRecord(h->ev_pre, st));
    SF_CUDA_TRY(cudaStreamWaitEvent(h->hi_stream, h->ev_pre, 0));
    if ((s = launch_step(h, bb, mode, h->hi_stream, &fused))) return s;
    const bool need_inj = !fused && b.inj && b.inj->ntgt > 0 && b.inj_vals;
    if (need_inj) {
        if ((s = ensure_split_lists(h, *b.inj))) return s;
        if ((s = launch_inject_list(h, *b.inj, b.out, b.inj_vals, b.inj->jl_bnd, b.inj->n_bnd, snap_patch,
                                    grad_snap, b.grad, b.gscale, h->hi_stream, mq, md)))
            return s;
    }
    if (b.itp_cur >= 0 && h->itp_pending[b.itp_cur & 1])
        SF_CUDA_TRY(cudaStreamWaitEvent(h->hi_stream, h->ev_itp[b.itp_cur & 1], 0));
    SF_CUDA_TRY(cudaEventRecord(h->ev_bnd, h->hi_stream));
    const uint32_t seq = h->p2p_seq + 1;
    const bool local = sf_comm_p2p_local(h);  // in-process ranks: events, not counters
    for (int side = 0; side < 2 && !local; ++side)
        if (h->p2p_nflag[side] && (s = stream_write32(h->hi_stream, h->p2p_nflag[side], seq))) return s;
    if ((s = launch_step(h, bi, mode, st, &f2))) return s;
    // (the interior TMA launch may inject its own planes' targets itself)
    if (need_inj && !f2 && (s = launch_inject_list(h, *b.inj, b.out, b.inj_vals, b.inj->jl_int, b.inj->n_int,
                                                   snap_patch, grad_snap, b.grad, b.gscale, st)))
        return s;
    SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_bnd, 0));
    if (local) {
        if ((s = sf_comm_p2p_local_step(h, st, plan[5] != 0, plan[6] != 0))) return s;
    } else {
        if (plan[5] && (s = stream_wait32(st, h->p2p_flags + 0, seq))) return s;
        if (plan[6] && (s = stream_wait32(st, h->p2p_flags + 1, seq))) return s;
    }
    h->p2p_seq = seq;
    return SF_OK;
}

// One time step: stencil (+ fused sparse work), standalone injection if not fused, and in
// slab mode the halo exchange.  Split mode computes the r boundary planes at each end
// first, injects there, hands them to NCCL on the comm stream and computes the interior
// while the halos travel; the stream then waits for the exchange.
// One-launch slab schedule (SF_OPT_ONE_LAUNCH): ONE persistent
// stencil launch per step whose last x-chunk of every tile streams downward, so both
// boundary ranges are finished r output planes in; each CTA signals a finished boundary range
// on the handle's device counters (fence + atomic), the comm stream waits on the counters
// (cuStreamWaitValue32) and runs the NCCL exchange while the same launch computes the
// interior.  Injection must happen inside the launch (fused list or plane injection) so the
// boundary planes are final when signalled.  One GPU (SF_OPT_ONE_LAUNCH 2 with SF_OPT_SPLIT):
// the same schedule, the "exchange" being a copy of the boundary planes into a test probe.
static bool one_launch_ok(sf_handle *h, const StepBufs &b, int mode, cudaStream_t st)
{
    if (!h->one_launch || h->ndim != 3 || !h->sigc) return false;
    // NCCL exchange: separate processes only (local groups keep the two-launch split);
    // peer stores (SF_OPT_P2P): local groups and processes alike
    if (h->nranks > 1 ? (!h->p2p && sf_comm_is_local(h->comm)) : h->one_launch < 2) return false;
    StepBufs bd = b;
    bd.bidir = true;
    bd.dry = true;
    bool fused = false;
    if (launch_step(h, bd, mode, st, &fused) != SF_OK) return false;
    const bool need = b.inj && b.inj->ntgt > 0 && b.inj_vals;
    return fused || !need;
}

// Peer-store form of the one-launch schedule (SF_OPT_P2P + SF_OPT_ONE_LAUNCH): the single
// persistent launch stores its boundary planes a second time, straight into the neighbours'
// halos of the same level (peer-mapped; the transfer overlaps the stencil tile by tile), then
// -- in stream order after the launch and after the side-stream record of the level it read
// (the neighbour overwrites that buffer's halo at its next step: write-after-read) -- bumps
// the neighbours' counters and waits on its own (RAW: the neighbours' planes have landed).
static sf_status do_step_onelaunch_p2p(sf_handle *h, StepBufs b, int mode, cudaStream_t st)
{
    sf_status s;
    const int64_t r = h->r;
    const int ob = b.out == h->p2p_own[0] ? 0 : b.out == h->p2p_own[1] ? 1 : -1;
    if (ob < 0) return sf_set_error(SF_ERR_INVALID_ARG, "P2P step on a buffer outside the published state");
    int64_t plan[7], qp[7];
    if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank, h->nranks, plan))) return s;
    const int64_t plane = h->N / h->nb[0];
    auto delta = [](const float *to, const float *from) {
        return (int64_t)(reinterpret_cast<uintptr_t>(to) - reinterpret_cast<uintptr_t>(from));
    };
    int64_t mq[4] = {0, 0, 0, 0}, md[2] = {0, 0};
    if (plan[5]) {  // owned [r, 2r) -> left neighbour's right halo
        if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank - 1, h->nranks, qp))) return s;
        mq[0] = plan[0];
        mq[1] = plan[0] + r;
        md[0] = delta(h->p2p_nbr[0][ob] + qp[3] * plane, b.out + plan[0] * plane);
    }
    if (plan[6]) {  // owned [nl, nl + r) -> right neighbour's left halo
        if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank + 1, h->nranks, qp))) return s;
        mq[2] = plan[2];
        mq[3] = plan[2] + r;
        md[1] = delta(h->p2p_nbr[1][ob] + qp[1] * plane, b.out + plan[2] * plane);
    }
    StepBufs bm = b;
    bm.bidir = true;
    bm.nosig = true;
    bm.mq = mq;
    bm.md = md;
    bool fused = false;
    if ((s = launch_step(h, bm, mode, st, &fused))) return s;
    h->n_onelaunch++;
    if (b.itp_cur >= 0 && h->itp_pending[b.itp_cur & 1])
        SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_itp[b.itp_cur & 1], 0));
    SF_CUDA_TRY(cudaEventRecord(h->ev_bnd, st));
    const uint32_t seq = h->p2p_seq + 1;
    if (sf_comm_p2p_local(h)) {
        if ((s = sf_comm_p2p_local_step(h, st, plan[5] != 0, plan[6] != 0))) return s;
    } else {
        for (int side = 0; side < 2; ++side)
            if (h->p2p_nflag[side] && (s = stream_write32(st, h->p2p_nflag[side], seq))) return s;
        if (plan[5] && (s = stream_wait32(st, h->p2p_flags + 0, seq))) return s;
        if (plan[6] && (s = stream_wait32(st, h->p2p_flags + 1, seq))) return s;
    }
    h->p2p_seq = seq;
    return SF_OK;
}

static sf_status do_step_onelaunch(sf_handle *h, StepBufs b, int mode, cudaStream_t st)
{
    if (h->p2p && h->nranks > 1) return do_step_onelaunch_p2p(h, b, mode, st);
    sf_status s;
    bool fused = false;
    SF_CUDA_TRY(cudaEventRecord(h->ev_pre, st));  // orders the exchange after earlier readers of `out`
    b.bidir = true;
    // the persistent launch would hold every SM until it ends: leave some free so the NCCL
    // kernels of the exchange run while it computes the interior
    const int reserve = h->comm_sms >= 0 ? h->comm_sms : (h->nranks > 1 ? 8 : 0);
    if (reserve > 0) b.ctas_cap = std::max(1, h->sms - reserve);
    if ((s = launch_step(h, b, mode, st, &fused))) return s;
    h->sig_tgt += (uint32_t)h->last_tiles;       // one signal per tile and side
    h->n_onelaunch++;
    cudaStream_t cs = h->comm_stream;
    SF_CUDA_TRY(cudaStreamWaitEvent(cs, h->ev_pre, 0));
    if ((s = stream_wait32(cs, h->sigc + 0, h->sig_tgt))) return s;
    if ((s = stream_wait32(cs, h->sigc + 1, h->sig_tgt))) return s;
    if (h->nranks > 1) {
        if ((s = sf_comm_halo_exchange(h, b.out, cs))) return s;
    } else if (h->probe) {
        const int64_t plane = h->N / h->nb[0], r = h->r;
        const size_t bytes = sizeof(float) * (size_t)(r * plane);
        SF_CUDA_TRY(cudaMemcpyAsync(h->probe, b.out + h->xa * plane, bytes, cudaMemcpyDeviceToDevice, cs));
        SF_CUDA_TRY(cudaMemcpyAsync(h->probe + r * plane, b.out + (h->xb - r) * plane, bytes,
                                    cudaMemcpyDeviceToDevice, cs));
    }
    SF_CUDA_TRY(cudaEventRecord(h->ev_xch, cs));
    SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_xch, 0));
    return SF_OK;
}

static sf_status do_step(sf_handle *h, StepBufs b, int mode, float *snap_patch, const float *grad_snap,
                         cudaStream_t st)
{
    sf_status s;
    bool fused = false;
    const int64_t r = h->r, xa = h->xa, xb = h->xb;
    if (!h->split || xb - xa <= 2 * r) {
        if ((s = launch_step(h, b, mode, st, &fused))) return s;
        if (!fused && (s = launch_inject(h, *b.inj, b.out, b.inj_vals, snap_patch, grad_snap, b.grad,
                                         b.gscale, st)))
            return s;
        if (h->nranks > 1) return sf_comm_halo_exchange(h, b.out, st);
        return SF_OK;
    }
    if (one_launch_ok(h, b, mode, st)) return do_step_onelaunch(h, b, mode, st);
    // boundary planes at both ends in ONE launch on the high-priority stream, overlapping
    // the interior launch on `st`; then the exchange on the comm stream
    bool f2 = false;
    StepBufs bb = b, bi = b;
    bb.xa = xa, bb.xb = xa + r, bb.xa2 = xb - r, bb.xb2 = xb;
    bi.xa = xa + r, bi.xb = xb - r;
    // the persistent interior launch would hold every SM until it ends: leave some free so
    // the NCCL exchange kernels (and the side-stream records) run concurrently
    const int reserve = h->comm_sms >= 0 ? h->comm_sms : (h->nranks > 1 ? 8 : 0);
    if (reserve > 0) bi.ctas_cap = std::max(1, h->sms - reserve);
    if (h->p2p && h->nranks > 1) return do_step_p2p(h, b, bb, bi, mode, snap_patch, grad_snap, st);
    SF_CUDA_TRY(cudaEventRecord(h->ev_pre, st));
    SF_CUDA_TRY(cudaStreamWaitEvent(h->hi_stream, h->ev_pre, 0));
    if ((s = launch_step(h, bb, mode, h->hi_stream, &fused))) return s;
    const bool need_inj = !fused && b.inj && b.inj->ntgt > 0 && b.inj_vals;
    if (need_inj) {
        if ((s = ensure_split_lists(h, *b.inj))) return s;
        if ((s = launch_inject_list(h, *b.inj, b.out, b.inj_vals, b.inj->jl_bnd, b.inj->n_bnd, snap_patch,
                                    grad_snap, b.grad, b.gscale, h->hi_stream)))
            return s;
    }
    SF_CUDA_TRY(cudaEventRecord(h->ev_bnd, h->hi_stream));
    if (h->nranks > 1) {
        SF_CUDA_TRY(cudaStreamWaitEvent(h->comm_stream, h->ev_bnd, 0));
        if ((s = sf_comm_halo_exchange(h, b.out, h->comm_stream))) return s;
        SF_CUDA_TRY(cudaEventRecord(h->ev_xch, h->comm_stream));
    }
    if ((s = launch_step(h, bi, mode, st, &f2))) return s;
    if (need_inj && (s = launch_inject_list(h, *b.inj, b.out, b.inj_vals, b.inj->jl_int, b.inj->n_int, snap_patch,
                                            grad_snap, b.grad, b.gscale, st)))
        return s;
    SF_CUDA_TRY(cudaStreamWaitEvent(st, h->nranks > 1 ? h->ev_xch : h->ev_bnd, 0));
    return SF_OK;
}

// Records of a level run on the handle's side stream, concurrently with the next
// stencil step (which only reads that level); the stencil two steps later overwrites
// the level, so it waits for the record first.  ev_itp[level & 1] marks completion.
static sf_status side_interp(sf_handle *h, SfSparse &sp, const float *lvl, float *row, int level,
                             cudaStream_t st)
{
    if (!row || sp.np == 0) return SF_OK;
    if (h->N < SF_SIDE_MIN_POINTS) {
        // small grids are launch-bound: the cross-stream events would cost more than the
        // overlap buys -> interpolate in stream order
        return launch_interp(h, sp, lvl, row, st);
    }
    SF_CUDA_TRY(cudaEventRecord(h->ev_ready, st));
    SF_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_ready, 0));
    sf_status s = launch_interp(h, sp, lvl, row, h->side);
    if (s) return s;
    SF_CUDA_TRY(cudaEventRecord(h->ev_itp[level & 1], h->side));
    h->itp_pending[level & 1] = true;
    return SF_OK;
}

// before a stencil step writes into the buffer holding `level`
static sf_status wait_interp(sf_handle *h, int level, cudaStream_t st)
{
    if (level < 0 || !h->itp_pending[level & 1]) return SF_OK;
    SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_itp[level & 1], 0));
    h->itp_pending[level & 1] = false;
    return SF_OK;
}

static sf_status join_side(sf_handle *h, cudaStream_t st)
{
    for (int k = 0; k < 2; ++k) {
        if (h->itp_pending[k]) {
            SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_itp[k], 0));
            h->itp_pending[k] = false;
        }
    }
    return SF_OK;
}

// SF_OPT_LOOP2D: a small 2D grid (both levels in one CTA's shared memory) runs its whole time
// loop -- stencil, injection, records -- in one launch (loop2d.cuh; bitwise the per-step path)
static int loop2d_rpc(const sf_handle *h) { return (int)((h->nb[0] + SF_LOOP2D_CTAS - 1) / SF_LOOP2D_CTAS); }
static bool loop2d_ok(const sf_handle *h)
{
    return h->loop2d && h->ndim == 2 && h->nranks == 1 && h->variant != SF_VAR_TMA &&
           loop2d_smem(loop2d_rpc(h), (int)h->nb[1], h->beta != nullptr) <= SF_LOOP2D_SMEM_MAX &&
           h->src.ntgt <= SF_LOOP2D_LOC && h->rec.ntgt <= SF_LOOP2D_LOC;
}

static sf_status launch_loop2d(sf_handle *h, float *A, float *B, const SfSparse &inj, const float *vals,
                               const SfSparse &itp, float *rec, bool backward, cudaStream_t st)
{
    Loop2dArgs a{};
    a.n0 = (int)h->nb[0];
    a.n2 = (int)h->nb[1];
    a.rpc = loop2d_rpc(h);
    a.nsteps = h->nt - 1;
    a.backward = backward ? 1 : 0;
    a.nt = h->nt;
    a.w = h->w;
    a.c3 = h->c3;
    a.beta = h->beta;
    a.sigx = h->sig[0];
    a.sigz = h->sig[2];
    a.hdt = (float)(0.5 * h->dt);
    a.A = A;
    a.B = B;
    a.ntgt = vals ? inj.ntgt : 0;
    a.tgt = inj.j_tgt;
    a.rowptr = inj.j_rowptr;
    a.pt = inj.j_pt;
    a.coef = inj.j_coef;
    a.vals = vals;
    a.nvals = inj.np;
    a.np = rec ? itp.np : 0;
    a.K = itp.ik;
    a.eidx = itp.e_idx;
    a.ew = itp.e_w;
    a.rec = rec;
    ProfScope ps(h, PK_STENCIL, st);
    cudaError_t e;
    switch (h->r) {
    case 1: e = sf_launch_loop2d_r1(a, st); break;
    case 2: e = sf_launch_loop2d_r2(a, st); break;
    case 3: e = sf_launch_loop2d_r3(a, st); break;
    case 4: e = sf_launch_loop2d_r4(a, st); break;
    case 5: e = sf_launch_loop2d_r5(a, st); break;
    case 6: e = sf_launch_loop2d_r6(a, st); break;
    case 7: e = sf_launch_loop2d_r7(a, st); break;
    default: e = sf_launch_loop2d_r8(a, st); break;
    }
    if (e != cudaSuccess) {
        // (a device without 16-CTA clusters: fall back to one launch per step for good)
        if (e == cudaErrorInvalidValue || e == cudaErrorNotSupported || e == cudaErrorInvalidConfiguration ||
            e == cudaErrorLaunchOutOfResources) {
            cudaGetLastError();
            h->loop2d = false;
            return SF_ERR_INVALID_ARG;  // caller retries on the per-step path
        }
        return sf_set_error(SF_ERR_CUDA, "loop2d launch: %s", cudaGetErrorString(e));
    }
    return SF_OK;
}

// ------------------------------------------------------------------ two steps per pass (SF_OPT_TBLOCK)
// stencil_tb2.cuh: tiles of 8 rows x 120 columns, step 1 on the tile grown by r rows and
// 4 columns per side (8 + 2r rows x 128 columns)
static const int TB_TY = 8, TB_TZ = 120, TB_MZ = 4;

static bool tb_ok(const sf_handle *h)
{
    return h->ndim == 3 && h->r <= 4 && h->nranks == 1 && !h->sep && h->nb[2] % 4 == 0 &&
           resolve_variant(h) == SF_VAR_TMA;
}

// the second state pair and the per-tile source lists: entries (plane, ey * 128 + ec, CSR row)
// for every tile whose grown region holds the target, sorted by (tile, plane)
static sf_status ensure_tb(sf_handle *h)
{
    if (!tb_ok(h))
        return sf_set_error(SF_ERR_INVALID_ARG, "SF_OPT_TBLOCK: needs a 3D one-GPU handle, space order <= 8, "
                                                "no separable profiles, n_z %% 4 == 0, the TMA kernel");
    if (h->tb_buf) return SF_OK;
    SF_CUDA_TRY(cudaMalloc((void **)&h->tb_buf, 2 * sizeof(float) * h->N));
    const int64_t n1 = h->nb[1], n2 = h->nb[2], R = h->r;
    const int64_t ntz = (n2 + TB_TZ - 1) / TB_TZ, nty = (n1 + TB_TY - 1) / TB_TY, tiles = ntz * nty;
    struct E {
        int64_t tile;
        int q, p, t;
    };
    std::vector<E> es;
    for (size_t t = 0; t < h->src.h_tgt.size(); ++t) {
        const int64_t g = h->src.h_tgt[t];
        const int64_t x = g / (n1 * n2), y = (g / n2) % n1, z = g % n2;
        for (int64_t ty = std::max<int64_t>(0, (y - R) / TB_TY - 1); ty < nty && ty * TB_TY - R <= y; ++ty)
            for (int64_t tz = std::max<int64_t>(0, (z - TB_MZ) / TB_TZ - 1); tz < ntz && tz * TB_TZ - TB_MZ <= z; ++tz) {
                const int64_t ey = y - (ty * TB_TY - R), ec = z - (tz * TB_TZ - TB_MZ);
                if (ey < 0 || ey >= TB_TY + 2 * R || ec < 0 || ec >= 128) continue;
                es.push_back({ty * ntz + tz, (int)x, (int)(ey * 128 + ec), (int)t});
            }
    }
    std::sort(es.begin(), es.end(), [](const E &a, const E &b) {
        return std::tie(a.tile, a.q, a.p) < std::tie(b.tile, b.q, b.p);
    });
    std::vector<int> beg(tiles + 1, 0), q, p, tt;
    for (const E &e : es) beg[e.tile + 1]++;
    for (int64_t i = 0; i < tiles; ++i) beg[i + 1] += beg[i];
    for (const E &e : es) {
        q.push_back(e.q);
        p.push_back(e.p);
        tt.push_back(e.t);
    }
    sf_status s;
    if ((s = upload(&h->tb_beg, beg))) return s;
    if (!es.empty()) {
        if ((s = upload(&h->tb_q, q))) return s;
        if ((s = upload(&h->tb_p, p))) return s;
        if ((s = upload(&h->tb_t, tt))) return s;
    }
    // the pool allocations are ordered on the legacy stream: complete them before the
    // caller's (possibly non-blocking) stream uses the buffers
    SF_CUDA_TRY(cudaStreamSynchronize(cudaStreamLegacy));
    return SF_OK;
}

// one two-step launch: (u^{n-1} = X, u^n = Y) -> (u^{n+1} = Z, u^{n+2} = W); source rows
// v1 (step n) and v2 (step n + 1), or NULL
static sf_status launch_tb(sf_handle *h, const float *X, const float *Y, float *Z, float *W, const float *v1,
                           const float *v2, cudaStream_t st)
{
    const int R = h->r, EY = TB_TY + 2 * R;
    SfTmaMaps m;
    memset(&m, 0, sizeof m);
    const int64_t d3[3] = {h->nb[2], h->nb[1], h->nb[0]};
    const uint32_t bu[3] = {128 + 2 * TB_MZ, (uint32_t)(EY + 2 * R), 1};
    const uint32_t bc[3] = {128, (uint32_t)EY, 1};
    sf_status s;
    if ((s = make_map(&m.cur, Y, 3, d3, bu))) return s;
    if ((s = make_map(&m.old, X, 3, d3, bc))) return s;
    if ((s = make_map(&m.c3, h->c3, 3, d3, bc))) return s;
    if (h->beta && (s = make_map(&m.beta, h->beta, 3, d3, bc))) return s;
    TbArgs a{};
    a.n0 = (int)h->nb[0];
    a.n1 = (int)h->nb[1];
    a.n2 = (int)h->nb[2];
    a.w = h->w;
    a.c3 = h->c3;
    a.beta = h->beta;
    a.o1 = Z;
    a.o2 = W;
    if (h->src.ntgt > 0 && (v1 || v2)) {
        a.beg = h->tb_beg;
        a.e_q = h->tb_q;
        a.e_p = h->tb_p;
        a.e_t = h->tb_t;
        a.rowptr = h->src.j_rowptr;
        a.pt = h->src.j_pt;
        a.coef = h->src.j_coef;
        a.vals1 = v1;
        a.vals2 = v2;
    }
    cudaError_t e;
    {
        ProfScope ps(h, PK_STENCIL, st);
        switch (R) {
        case 1: e = sf_launch_tb2_r1(m, a, resolve_ctas(h), st); break;
        case 2: e = sf_launch_tb2_r2(m, a, resolve_ctas(h), st); break;
        case 3: e = sf_launch_tb2_r3(m, a, resolve_ctas(h), st); break;
        default: e = sf_launch_tb2_r4(m, a, resolve_ctas(h), st); break;
        }
    }
    if (e != cudaSuccess) return sf_set_error(SF_ERR_CUDA, "two-step launch: %s", cudaGetErrorString(e));
    h->n_tb++;
    return SF_OK;
}

// records of the levels a launch wrote (side stream, overlapping the next launch); the
// launch that overwrites that buffer pair waits for them (ev_itp[pair])
static sf_status tb_records(sf_handle *h, const float *l1, float *r1, const float *l2, float *r2, int pair,
                            cudaStream_t st)
{
    if (h->rec.np == 0 || !r1) return SF_OK;
    SF_CUDA_TRY(cudaEventRecord(h->ev_ready, st));
    SF_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_ready, 0));
    sf_status s;
    if ((s = launch_interp(h, h->rec, l1, r1, h->side))) return s;
    if (l2 && (s = launch_interp(h, h->rec, l2, r2, h->side))) return s;
    SF_CUDA_TRY(cudaEventRecord(h->ev_itp[pair], h->side));
    h->itp_pending[pair] = true;
    return SF_OK;
}

static sf_status tb_wait(sf_handle *h, int pair, cudaStream_t st)
{
    if (!h->itp_pending[pair]) return SF_OK;
    SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_itp[pair], 0));
    h->itp_pending[pair] = false;
    return SF_OK;
}

// sf_forward without snapshots, two steps per launch: the state pair alternates between the
// caller's u (pair 0) and tb_buf (pair 1); an odd step count ends with one single step, and
// the final (u^{nt-2}, u^{nt-1}) is moved back into u
static sf_status forward_tb(sf_handle *h, const float *wavelet, float *rec, float *u, cudaStream_t st)
{
    const int64_t N = h->N;
    float *PR[2][2] = {{u, u + N}, {h->tb_buf, h->tb_buf + N}};
    const int np = h->src.np, nr = h->rec.np;
    sf_status s;
    h->itp_pending[0] = h->itp_pending[1] = false;
    int pp = 0;  // pair holding (u^{n-1}, u^n)
    if ((s = tb_records(h, PR[0][1], rec, nullptr, nullptr, 0, st))) return s;
    int n = 0;
    for (; n + 2 <= h->nt - 1; n += 2) {
        const int o = pp ^ 1;
        if ((s = tb_wait(h, o, st))) return s;
        const float *v1 = wavelet ? wavelet + (int64_t)n * np : nullptr;
        const float *v2 = wavelet ? wavelet + (int64_t)(n + 1) * np : nullptr;
        if ((s = launch_tb(h, PR[pp][0], PR[pp][1], PR[o][0], PR[o][1], v1, v2, st))) return s;
        if ((s = tb_records(h, PR[o][0], rec ? rec + (int64_t)(n + 1) * nr : nullptr, PR[o][1],
                            rec ? rec + (int64_t)(n + 2) * nr : nullptr, o, st)))
            return s;
        pp = o;
    }
    float *prev = PR[pp][0], *last = PR[pp][1];
    if (n < h->nt - 1) {  // one single step in place: u^{n+1} over u^{n-1}
        if ((s = tb_wait(h, pp, st))) return s;
        const float *wrow = wavelet ? wavelet + (int64_t)n * np : nullptr;
        float *rrow = rec ? rec + (int64_t)(n + 1) * nr : nullptr;
        StepBufs b{PR[pp][1], PR[pp][0], nullptr, nullptr, 0, 0, nullptr, 0.f, &h->src, wrow, &h->rec, rrow};
        if ((s = do_step(h, b, SF_MODE_PLAIN, nullptr, nullptr, st))) return s;
        if ((s = tb_records(h, PR[pp][0], rrow, nullptr, nullptr, pp, st))) return s;
        prev = PR[pp][1];
        last = PR[pp][0];
    }
    if ((s = join_side(h, st))) return s;
    if (prev == u && last == u + N) return SF_OK;
    if (prev == u + N && last == u) return swap_halves(h, u, u + N, st);
    SF_CUDA_TRY(cudaMemcpyAsync(u, prev, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
    SF_CUDA_TRY(cudaMemcpyAsync(u + N, last, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
    return SF_OK;
}

static sf_status forward_body(sf_handle *h, const float *wavelet, float *rec, float *u, float *snaps,
                              int save_every, void *stream)
{
    if (!h || !u) return sf_set_error(SF_ERR_INVALID_ARG, "handle or u is NULL");
    if (h->src.np > 0 && !wavelet) return sf_set_error(SF_ERR_INVALID_ARG, "wavelet is NULL");
    if (h->rec.np > 0 && !rec) return sf_set_error(SF_ERR_INVALID_ARG, "rec is NULL");
    if (snaps && save_every < 1) return sf_set_error(SF_ERR_INVALID_ARG, "save_every < 1 with snaps");
    cudaStream_t st = S(stream);
    const int64_t N = h->N;
    float *A = u, *B = u + N;  // A = u^{-1}, B = u^0
    sf_status s;
    if (!snaps && loop2d_ok(h)) {
        s = launch_loop2d(h, A, B, h->src, wavelet, h->rec, rec, false, st);
        if (s != SF_ERR_INVALID_ARG || h->loop2d) return s;
    }
    if (!snaps && h->tblock && tb_ok(h)) return forward_tb(h, wavelet, rec, u, st);
    h->itp_pending[0] = h->itp_pending[1] = false;
    if (h->nranks > 1) {  // make the halo of u^0 valid for the first stencil / record
        if (h->p2p && (s = sf_comm_p2p_setup(h, A, B, st))) return s;
        if ((s = post_step_exchange(h, B, st))) return s;
    }
    if ((s = side_interp(h, h->rec, B, rec, 0, st))) return s;
    if (snaps && h->snap_half) {
        k_f32_to_f16<<<592, 256, 0, st>>>(reinterpret_cast<__half *>(snaps), B, N);
        SF_CUDA_TRY(cudaGetLastError());
    } else if (snaps) {
        SF_CUDA_TRY(cudaMemcpyAsync(snaps, B, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
    }
    for (int n = 0; n <= h->nt - 2; ++n) {
        float *cur = (n % 2 == 0) ? B : A;
        float *out = (n % 2 == 0) ? A : B;   // holds u^{n-1}, becomes u^{n+1}
        const bool save = snaps && ((n + 1) % save_every == 0);
        float *slot = save ? snap_slot(snaps, h, (n + 1) / save_every) : nullptr;
        const float *wrow = wavelet ? wavelet + (int64_t)n * h->src.np : nullptr;
        float *rrow = rec ? rec + (int64_t)(n + 1) * h->rec.np : nullptr;
        if ((s = wait_interp(h, n - 1, st))) return s;
        StepBufs b{cur, out, slot, nullptr, 0, 0, nullptr, 0.f, &h->src, wrow, &h->rec, rrow};
        b.itp_cur = n;
        if ((s = do_step(h, b, save ? SF_MODE_SAVE : SF_MODE_PLAIN, slot, nullptr, st))) return s;
        if ((s = side_interp(h, h->rec, out, rrow, n + 1, st))) return s;
    }
    if ((s = join_side(h, st))) return s;
    // u^{nt-1} was written into A when nt is even: restore (u^{nt-2}, u^{nt-1}) order
    if (h->nt % 2 == 0) return swap_halves(h, A, B, st);
    return SF_OK;
}

static sf_status adjoint_body(sf_handle *h, const float *res, float *srca, float *v, const float *snaps,
                              int save_every, float *grad, void *stream)
{
    if (!h || !v) return sf_set_error(SF_ERR_INVALID_ARG, "handle or v is NULL");
    if (h->rec.np > 0 && !res) return sf_set_error(SF_ERR_INVALID_ARG, "res is NULL");
    if (h->src.np > 0 && !srca) return sf_set_error(SF_ERR_INVALID_ARG, "srca is NULL");
    const bool dograd = grad != nullptr;
    if (dograd && (!snaps || save_every < 1))
        return sf_set_error(SF_ERR_INVALID_ARG, "gradient needs snaps and save_every >= 1");
    cudaStream_t st = S(stream);
    const int64_t N = h->N;
    const int64_t nsnap = dograd ? (h->nt - 1) / save_every + 1 : 0;
    const float gscale = dograd ? (float)((double)save_every / (h->dt * h->dt)) : 0.f;
    float *A = v, *B = v + N;  // A = v^{nt}, B = v^{nt-1}
    sf_status s;
    if (!dograd && loop2d_ok(h)) {
        s = launch_loop2d(h, A, B, h->rec, res, h->src, srca, true, st);
        if (s != SF_ERR_INVALID_ARG || h->loop2d) return s;
    }
    if (h->nranks > 1) {
        if (h->p2p && (s = sf_comm_p2p_setup(h, A, B, st))) return s;
        if ((s = post_step_exchange(h, B, st))) return s;
    }
    h->itp_pending[0] = h->itp_pending[1] = false;
    if ((s = side_interp(h, h->src, B, srca ? srca + (int64_t)(h->nt - 1) * h->src.np : nullptr,
                         0, st)))
        return s;
    for (int n = h->nt - 1, j = 0; n >= 1; --n, ++j) {
        float *cur = (j % 2 == 0) ? B : A;
        float *out = (j % 2 == 0) ? A : B;
        const bool g = dograd && (n % save_every == 0);
        if ((s = wait_interp(h, j - 1, st))) return s;   // level written at step j-2
        const float *rrow = res ? res + (int64_t)n * h->rec.np : nullptr;
        float *srow = srca ? srca + (int64_t)(n - 1) * h->src.np : nullptr;
        StepBufs b{cur, out, nullptr, g ? snaps : nullptr, g ? n / save_every : 0, nsnap,
                   g ? grad : nullptr, gscale, &h->rec, rrow, &h->src, srow};
        b.itp_cur = j;
        if ((s = do_step(h, b, g ? SF_MODE_GRAD : SF_MODE_PLAIN, nullptr,
                         g ? snap_slot(snaps, h, n / save_every) : nullptr, st)))
            return s;
        if ((s = side_interp(h, h->src, out, srow, j + 1, st))) return s;
    }
    if ((s = join_side(h, st))) return s;
    if (h->nt % 2 == 0) return swap_halves(h, A, B, st);
    return SF_OK;
}

// ------------------------------------------------------------------ CUDA graphs (SF_OPT_GRAPH)
static void drop_graphs(sf_handle *h)
{
    for (SfGraphCache *G : {&h->gfwd, &h->gadj}) {
        if (G->exec) cudaGraphExecDestroy(G->exec);
        *G = SfGraphCache{};
    }
}

// Run `body(stream)` eagerly, or -- graphs on, same arguments as the previous call -- capture
// it once on the handle's graph stream and replay it there, ordered after and before the
// caller's stream by events (the legacy default stream cannot be captured).
template <class F>
static sf_status with_graph(sf_handle *h, SfGraphCache &G, const void *const k[6], const long long ik[3],
                            cudaStream_t st, F body)
{
    if (!h->use_graph || h->prof || h->nranks > 1) return body(st);
    auto same = [&](const void *const *a, const long long *ai) {
        for (int i = 0; i < 6; ++i)
            if (a[i] != k[i]) return false;
        for (int i = 0; i < 3; ++i)
            if (ai[i] != ik[i]) return false;
        return true;
    };
    if (G.exec && same(G.key, G.ikey)) {
        SF_CUDA_TRY(cudaEventRecord(h->ev_gin, st));
        SF_CUDA_TRY(cudaStreamWaitEvent(h->gstream, h->ev_gin, 0));
        SF_CUDA_TRY(cudaGraphLaunch(G.exec, h->gstream));
        SF_CUDA_TRY(cudaEventRecord(h->ev_gout, h->gstream));
        SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_gout, 0));
        return SF_OK;
    }
    if (!same(G.seen, G.iseen)) {  // first call with these arguments: eager (builds tables)
        for (int i = 0; i < 6; ++i) G.seen[i] = k[i];
        for (int i = 0; i < 3; ++i) G.iseen[i] = ik[i];
        return body(st);
    }
    // second call: capture the whole call on the graph stream, instantiate, replay
    SF_CUDA_TRY(cudaEventRecord(h->ev_gin, st));
    SF_CUDA_TRY(cudaStreamWaitEvent(h->gstream, h->ev_gin, 0));
    SF_CUDA_TRY(cudaStreamBeginCapture(h->gstream, cudaStreamCaptureModeThreadLocal));
    sf_status s = body(h->gstream);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(h->gstream, &g);
    if (s) {
        if (g) cudaGraphDestroy(g);
        return s;
    }
    if (e != cudaSuccess) return sf_set_error(SF_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e2 = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e2 != cudaSuccess) return sf_set_error(SF_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e2));
    if (G.exec) cudaGraphExecDestroy(G.exec);
    G.exec = ex;
    for (int i = 0; i < 6; ++i) G.key[i] = k[i];
    for (int i = 0; i < 3; ++i) G.ikey[i] = ik[i];
    SF_CUDA_TRY(cudaGraphLaunch(G.exec, h->gstream));
    SF_CUDA_TRY(cudaEventRecord(h->ev_gout, h->gstream));
    SF_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_gout, 0));
    return SF_OK;
}

extern "C" sf_status sf_forward(sf_handle *h, const float *wavelet, float *rec, float *u,
                                float *snaps, int save_every, void *stream)
{
    if (!h || !u) return sf_set_error(SF_ERR_INVALID_ARG, "handle or u is NULL");
    const void *k[6] = {wavelet, rec, u, snaps, stream, nullptr};
    const long long ik[3] = {save_every, h->nt, 0};
    return with_graph(h, h->gfwd, k, ik, S(stream), [&](cudaStream_t s2) {
        return forward_body(h, wavelet, rec, u, snaps, save_every, s2);
    });
}

extern "C" sf_status sf_adjoint(sf_handle *h, const float *res, float *srca, float *v,
                                const float *snaps, int save_every, float *grad, void *stream)
{
    if (!h || !v) return sf_set_error(SF_ERR_INVALID_ARG, "handle or v is NULL");
    const void *k[6] = {res, srca, v, snaps, grad, stream};
    const long long ik[3] = {save_every, h->nt, 1};
    return with_graph(h, h->gadj, k, ik, S(stream), [&](cudaStream_t s2) {
        return adjoint_body(h, res, srca, v, snaps, save_every, grad, s2);
    });
}

extern "C" sf_status sf_residual(sf_handle *h, const float *d_syn, const float *d_obs, float *res,
                                 double *J, void *stream)
{
    if (!h || !d_syn || !d_obs || !res) return sf_set_error(SF_ERR_INVALID_ARG, "NULL argument");
    cudaStream_t st = S(stream);
    const int64_t n = (int64_t)h->nt * h->rec.np;
    const int nb = 1024;
    {
        ProfScope ps(h, PK_OTHER, st);
        k_residual<<<nb, 256, 0, st>>>(d_syn, d_obs, res, n, h->partial);
    }
    {
        ProfScope ps(h, PK_OTHER, st);
        k_sum_partials<<<1, 32, 0, st>>>(h->partial, nb, h->dJ);
    }
    SF_CUDA_TRY(cudaGetLastError());
    if (J) {
        SF_CUDA_TRY(cudaMemcpyAsync(J, h->dJ, sizeof(double), cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return SF_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

extern "C" size_t sf_gradient_workspace_bytes(const sf_handle *h, int save_every)
{
    if (!h || save_every < 1) return 0;
    const size_t N = (size_t)h->N;
    const size_t nsnap = (size_t)((h->nt - 1) / save_every + 1);
    return align256(snap_es(h) * N * nsnap) + 2 * align256(sizeof(float) * 2 * N) +
           align256(sizeof(float) * (size_t)h->nt * std::max(h->rec.np, 1)) +
           align256(sizeof(float) * (size_t)h->nt * std::max(h->src.np, 1));
}

extern "C" sf_status sf_gradient(sf_handle *h, const float *wavelet, const float *d_obs, float *grad,
                                 double *J, void *ws, size_t ws_bytes, int save_every, void *stream)
{
    if (!h || !grad || !d_obs || !ws) return sf_set_error(SF_ERR_INVALID_ARG, "NULL argument");
    if (save_every < 1) return sf_set_error(SF_ERR_INVALID_ARG, "save_every < 1");
    if (ws_bytes < sf_gradient_workspace_bytes(h, save_every))
        return sf_set_error(SF_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes,
                            sf_gradient_workspace_bytes(h, save_every));
    cudaStream_t st = S(stream);
    const size_t N = (size_t)h->N;
    const size_t nsnap = (size_t)((h->nt - 1) / save_every + 1);
    char *p = static_cast<char *>(ws);
    float *snaps = reinterpret_cast<float *>(p);
    p += align256(snap_es(h) * N * nsnap);
    float *u = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * 2 * N);
    float *v = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * 2 * N);
    float *rec = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * (size_t)h->nt * std::max(h->rec.np, 1));
    float *srca = reinterpret_cast<float *>(p);
    SF_CUDA_TRY(cudaMemsetAsync(u, 0, sizeof(float) * 2 * N, st));
    SF_CUDA_TRY(cudaMemsetAsync(v, 0, sizeof(float) * 2 * N, st));
    SF_CUDA_TRY(cudaMemsetAsync(grad, 0, sizeof(float) * N, st));
    sf_status s;
    if ((s = sf_forward(h, wavelet, rec, u, snaps, save_every, st))) return s;
    if (h->nranks > 1 && h->rec.np > 0) {  // every rank needs the full record (C18)
        if ((s = sf_comm_allreduce_f32(h->comm, rec, (size_t)h->nt * h->rec.np, st, h->rank))) return s;
    }
    if ((s = sf_residual(h, rec, d_obs, rec, J, st))) return s;
    if ((s = sf_adjoint(h, rec, h->src.np > 0 ? srca : nullptr, v, snaps, save_every, grad, st))) return s;
    return SF_OK;
}

// ------------------------------------------------------------------ checkpointed gradient
// Time windows of the handle's loops: sf_forward / sf_adjoint run h->nt samples from the
// state they are given, so a segment [b, b + L] is the same call with nt = L + 1 and the
// sparse-series pointers offset by b rows (wavelet rows b.., residual rows b..).
namespace {
struct NtWindow {
    sf_handle *h;
    int saved;
    NtWindow(sf_handle *h_, int nt) : h(h_), saved(h_->nt) { h->nt = nt; }
    ~NtWindow() { h->nt = saved; }
};
}  // namespace

extern "C" size_t sf_gradient_ckpt_workspace_bytes(const sf_handle *h, int save_every, int segment)
{
    if (!h || save_every < 1 || segment < save_every || segment % save_every) return 0;
    const size_t N = (size_t)h->N;
    const size_t nseg = (size_t)((h->nt - 1 + segment - 1) / segment);
    const size_t nss = (size_t)(segment / save_every + 1);
    const size_t nr = (size_t)std::max(h->rec.np, 1), ns = (size_t)std::max(h->src.np, 1);
    return align256(sizeof(float) * 2 * N * nseg) + align256(snap_es(h) * N * nss) +
           2 * align256(sizeof(float) * 2 * N) + align256(sizeof(float) * (size_t)h->nt * nr) +
           align256(sizeof(float) * (size_t)h->nt * ns) + align256(sizeof(float) * (size_t)(segment + 1) * nr) +
           align256(sizeof(float) * (size_t)(segment + 1) * ns);
}

extern "C" sf_status sf_gradient_ckpt(sf_handle *h, const float *wavelet, const float *d_obs, float *grad,
                                      double *J, void *ws, size_t ws_bytes, int save_every, int segment,
                                      void *stream)
{
    if (!h || !grad || !d_obs || !ws) return sf_set_error(SF_ERR_INVALID_ARG, "NULL argument");
    if (save_every < 1 || segment < save_every || segment % save_every)
        return sf_set_error(SF_ERR_INVALID_ARG, "segment %d is not a positive multiple of save_every %d",
                            segment, save_every);
    const size_t need = sf_gradient_ckpt_workspace_bytes(h, save_every, segment);
    if (ws_bytes < need) return sf_set_error(SF_ERR_WORKSPACE, "workspace %zu < %zu bytes", ws_bytes, need);
    cudaStream_t st = S(stream);
    const size_t N = (size_t)h->N;
    const int nt = h->nt, nrec = h->rec.np, nsrc = h->src.np;
    const int nseg = (nt - 1 + segment - 1) / segment;
    const size_t nr = (size_t)std::max(nrec, 1), ns = (size_t)std::max(nsrc, 1);
    char *p = static_cast<char *>(ws);
    float *ckpt = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * 2 * N * nseg);
    float *snaps = reinterpret_cast<float *>(p);
    p += align256(snap_es(h) * N * (size_t)(segment / save_every + 1));
    float *u = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * 2 * N);
    float *v = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * 2 * N);
    float *rec = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * (size_t)nt * nr);
    float *srca = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * (size_t)nt * ns);
    float *rec_seg = reinterpret_cast<float *>(p);
    p += align256(sizeof(float) * (size_t)(segment + 1) * nr);
    float *srca_seg = reinterpret_cast<float *>(p);
    SF_CUDA_TRY(cudaMemsetAsync(u, 0, sizeof(float) * 2 * N, st));
    SF_CUDA_TRY(cudaMemsetAsync(v, 0, sizeof(float) * 2 * N, st));
    SF_CUDA_TRY(cudaMemsetAsync(grad, 0, sizeof(float) * N, st));
    sf_status s;
    // pass 1: forward over the segments, checkpointing each segment's initial state pair
    for (int k = 0; k < nseg; ++k) {
        const int b = k * segment, len = std::min(segment, nt - 1 - b);
        SF_CUDA_TRY(cudaMemcpyAsync(ckpt + 2 * N * k, u, sizeof(float) * 2 * N, cudaMemcpyDeviceToDevice, st));
        {
            NtWindow win(h, len + 1);
            if ((s = sf_forward(h, wavelet ? wavelet + (size_t)b * nsrc : nullptr, nrec ? rec_seg : nullptr, u,
                                nullptr, 0, st)))
                return s;
        }
        if (nrec) {  // rows 1..len are levels b+1..b+len (row 0 = level b, already recorded)
            const int r0 = k == 0 ? 0 : 1;
            SF_CUDA_TRY(cudaMemcpyAsync(rec + (size_t)(b + r0) * nrec, rec_seg + (size_t)r0 * nrec,
                                        sizeof(float) * (size_t)(len + 1 - r0) * nrec, cudaMemcpyDeviceToDevice, st));
        }
    }
    if (h->nranks > 1 && nrec > 0) {  // every rank needs the full record (C18)
        if ((s = sf_comm_allreduce_f32(h->comm, rec, (size_t)nt * nrec, st, h->rank))) return s;
    }
    if ((s = sf_residual(h, rec, d_obs, rec, J, st))) return s;
    // pass 2: backward over the segments: recompute the segment's forward from its
    // checkpoint with snapshots every save_every, then its adjoint steps with correlation
    for (int k = nseg - 1; k >= 0; --k) {
        const int b = k * segment, len = std::min(segment, nt - 1 - b);
        SF_CUDA_TRY(cudaMemcpyAsync(u, ckpt + 2 * N * k, sizeof(float) * 2 * N, cudaMemcpyDeviceToDevice, st));
        NtWindow win(h, len + 1);
        if ((s = sf_forward(h, wavelet ? wavelet + (size_t)b * nsrc : nullptr, nrec ? rec_seg : nullptr, u,
                            snaps, save_every, st)))
            return s;
        if ((s = sf_adjoint(h, rec + (size_t)b * nrec, nsrc ? srca_seg : nullptr, v, snaps, save_every, grad, st)))
            return s;
        if (nsrc) {  // rows 0..len-1 are levels b..b+len-1 (row len = level b+len, from the later segment)
            const int rows = len + (k == nseg - 1 ? 1 : 0);
            SF_CUDA_TRY(cudaMemcpyAsync(srca + (size_t)b * nsrc, srca_seg, sizeof(float) * (size_t)rows * nsrc,
                                        cudaMemcpyDeviceToDevice, st));
        }
    }
    return SF_OK;
}

// ------------------------------------------------------------------ end-to-end host form
namespace {
struct HostCache {
    std::mutex mu;
    float *m = nullptr, *damp = nullptr, *wav = nullptr, *rec = nullptr, *u = nullptr;
    size_t nm = 0, nd = 0, nw = 0, nr = 0, nu = 0;
    cudaStream_t copy = nullptr;  // record downloads overlapping the next time window
    cudaEvent_t ev = nullptr;
    cudaEvent_t evh = nullptr;    // uploads done (orders sf_create's legacy-stream work)
};
// one cache per device: its buffers, stream and events belong to the device that was
// current when they were created.  The buffers come from the plain (cudaMalloc) /
// (cudaFree), not from the stream-ordered pool the macros above route to: cudaMalloc is
// synchronous, so a buffer is usable on any stream of its device (the caller's stream may
// be non-blocking) as soon as ensure() returns, and cudaFree waits for the device, so a
// buffer still read by earlier work on another stream is never released under it
constexpr int SF_HC_DEVICES = 64;
HostCache g_hcs[SF_HC_DEVICES];

sf_status ensure(float **p, size_t *cap, size_t n)
{
    if (n == 0) return SF_OK;
    if (*cap >= n) return SF_OK;
    if (*p) SF_CUDA_TRY((cudaFree)(*p));
    *p = nullptr;
    *cap = 0;
    SF_CUDA_TRY((cudaMalloc)((void **)p, n * sizeof(float)));
    *cap = n;
    return SF_OK;
}
}  // namespace

extern "C" sf_status sf_forward_once(const sf_desc *hd, const float *wavelet_host, float *rec_host,
                                     float *u_final_host, void *stream)
{
    return sf_forward_host(hd, wavelet_host, rec_host, u_final_host, stream);
}

extern "C" sf_status sf_forward_host(const sf_desc *hd, const float *wavelet_host, float *rec_host,
                                     float *u_final_host, void *stream)
{
    sf_status s = validate_desc(hd);
    if (s) return s;
    cudaStream_t st = S(stream);
    int dev = 0;
    SF_CUDA_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= SF_HC_DEVICES) return sf_set_error(SF_ERR_INVALID_ARG, "device %d", dev);
    HostCache &g_hc = g_hcs[dev];
    std::lock_guard<std::mutex> lk(g_hc.mu);
    size_t N = 1;
    for (int a = 0; a < hd->ndim; ++a) N *= (size_t)hd->shape[a];
    const size_t nw = (size_t)hd->nt * hd->nsrc, nr = (size_t)hd->nt * hd->nrec;
    if ((s = ensure(&g_hc.m, &g_hc.nm, N))) return s;
    if (hd->damp && (s = ensure(&g_hc.damp, &g_hc.nd, N))) return s;
    if ((s = ensure(&g_hc.wav, &g_hc.nw, nw))) return s;
    if ((s = ensure(&g_hc.rec, &g_hc.nr, nr))) return s;
    if ((s = ensure(&g_hc.u, &g_hc.nu, 2 * N))) return s;
    SF_CUDA_TRY(cudaMemcpyAsync(g_hc.m, hd->m, N * sizeof(float), cudaMemcpyHostToDevice, st));
    if (hd->damp)
        SF_CUDA_TRY(cudaMemcpyAsync(g_hc.damp, hd->damp, N * sizeof(float), cudaMemcpyHostToDevice, st));
    if (nw) SF_CUDA_TRY(cudaMemcpyAsync(g_hc.wav, wavelet_host, nw * sizeof(float), cudaMemcpyHostToDevice, st));
    SF_CUDA_TRY(cudaMemsetAsync(g_hc.u, 0, 2 * N * sizeof(float), st));
    // sf_create's device work runs on the legacy stream: order it after the uploads by an
    // event instead of a host sync, so that its host-side table building overlaps them
    if (!g_hc.evh) SF_CUDA_TRY(cudaEventCreateWithFlags(&g_hc.evh, cudaEventDisableTiming));
    SF_CUDA_TRY(cudaEventRecord(g_hc.evh, st));
    SF_CUDA_TRY(cudaStreamWaitEvent(cudaStreamLegacy, g_hc.evh, 0));
    sf_desc dd = *hd;
    dd.m = g_hc.m;
    dd.damp = hd->damp ? g_hc.damp : nullptr;
    sf_handle *h = nullptr;
    if ((s = sf_create(&dd, &h))) return s;
    // the forward in a few time windows (the same loop: sf_forward from the state it is
    // given, wavelet / record rows offset): each window's finished record rows go to the
    // host on a copy stream while the next window computes -- only the last window's
    // download stays exposed
    if (!g_hc.copy) {
        SF_CUDA_TRY(cudaStreamCreateWithFlags(&g_hc.copy, cudaStreamNonBlocking));
        SF_CUDA_TRY(cudaEventCreateWithFlags(&g_hc.ev, cudaEventDisableTiming));
    }
    const int nwin = (nr && rec_host && hd->nt > 64) ? 4 : 1;
    const int steps = hd->nt - 1;
    int64_t row0 = 0;  // first record row not yet downloaded
    for (int w = 0, b = 0; w < nwin && !s; ++w) {
        const int len = (w == nwin - 1) ? steps - b : steps / nwin;
        {
            NtWindow win(h, len + 1);
            s = sf_forward(h, nw ? g_hc.wav + (size_t)b * hd->nsrc : nullptr,
                           nr ? g_hc.rec + (size_t)b * hd->nrec : nullptr, g_hc.u, nullptr, 0, st);
        }
        if (s) break;
        b += len;
        if (nr && rec_host) {  // rows [row0, b) are final (row b is rewritten, identically, next window)
            const int64_t row1 = (w == nwin - 1) ? hd->nt : b;
            SF_CUDA_TRY(cudaEventRecord(g_hc.ev, st));
            SF_CUDA_TRY(cudaStreamWaitEvent(g_hc.copy, g_hc.ev, 0));
            cudaError_t e = cudaMemcpyAsync(rec_host + row0 * hd->nrec, g_hc.rec + row0 * hd->nrec,
                                            sizeof(float) * (size_t)(row1 - row0) * hd->nrec,
                                            cudaMemcpyDeviceToHost, g_hc.copy);
            if (e != cudaSuccess) s = sf_set_error(SF_ERR_CUDA, "rec download: %s", cudaGetErrorString(e));
            row0 = row1;
        }
    }
    if (!s && nr && rec_host) {
        cudaError_t e = cudaStreamSynchronize(g_hc.copy);
        if (e != cudaSuccess) s = sf_set_error(SF_ERR_CUDA, "rec download: %s", cudaGetErrorString(e));
    }
    if (!s && u_final_host) {
        cudaError_t e = cudaMemcpyAsync(u_final_host, g_hc.u, 2 * N * sizeof(float), cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = sf_set_error(SF_ERR_CUDA, "u download: %s", cudaGetErrorString(e));
    }
    if (!s) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) s = sf_set_error(SF_ERR_CUDA, "sync: %s", cudaGetErrorString(e));
    }
    sf_destroy(h);
    return s;
}
