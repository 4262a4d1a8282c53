// stencil_tma.cuh -- sm_100a 2.5D streaming stencil step, TMA-fed, register-rotated,
// persistent (one CTA per SM, each walking (tile, x-chunk) items).
//
// Hot kernel of the path (memory-bandwidth bound).  A tile
// is BY = 7 VY (32 / LZ) rows (y) x TZ = LZ VZ columns (z) -- LZ = 32: 14 x 128 tiles; LZ = 8:
// 56 x 32 "narrow" tiles for a z remainder (SF_OPT_ZSPLIT); a CTA walks its (tile, x-chunk) items --
// each a run of planes of one tile column streamed along x (the outermost, slab axis) --
// keeping its TMA pipeline running across items.  Per plane p of a segment:
//   * the producer warp's elected lane issues TMA (cp.async.bulk.tensor) loads:
//       - u^n plane p with its (y, z) halo into a DU-deep u ring: box (TZ + 2 HZ) x (BY + 2R);
//         the TMA out-of-bounds zero fill IS the zero ghost halo (reading C6);
//       - old / c3 / beta (+ snapshot / gradient in GRAD mode) of output plane q = p - R
//         into a DC-deep coefficient ring (with separable damping, DM = SF_DAMP_SEP, beta
//         is regenerated from three 1D profiles instead: 16 B/pt instead of 20);
//     completion via mbarrier transaction counts (full), slot reuse via one consumer
//     arrive per warp (empty), each preceded by a generic -> async proxy fence (the slot's
//     LDS reads vs the TMA refill: write-after-read across proxies);
//   * each consumer warp (VY rows, VZ consecutive z per lane) pushes its own u values of
//     plane p into a register queue of depth 2R+1 (compile-time rotated by unrolling the
//     plane loop by 2R+1: no register moves), then finishes output plane q = p - R:
//       in-plane  P = sum_k w_k (((y-k + y+k) + (z-k + z+k)) - 4u)  from the u tile of plane q
//                 (still in the ring: DU >= R + 1; each y row is loaded once for all VY rows),
//       x term    X = sum_k w_k ((u_{q-k} + u_{q+k}) - 2u)           from the register queue,
//       update    out = u + beta (u - old) + c3 (P + X),  stored in place over `old`
//     (plus the snapshot copy / fused gradient correlation; small source sets injected by
//     the owning lane before the store).
// HBM traffic per point (compulsory): read u^n, old, c3 (+beta), write out: 16 B (20 B
// with damping); each segment re-reads 2R warm-up planes of u^n.  Shared-memory traffic
// per point (the measured limiter of the previous one-row design): y rows (2R/VY + 1) x 4 B,
// z halo 2 HZ/VZ x 4 B, coefficients 4 B each, + the TMA fills -- no partial-sum ring.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <type_traits>
#include <utility>
#include "stencil_common.cuh"

#ifndef SF_DC_MIN
#define SF_DC_MIN 3
#endif
#ifndef SF_DC_MIN_HI
#define SF_DC_MIN_HI 2
#endif
#ifndef SF_WS_PREG
#define SF_WS_PREG 24
#endif
#ifndef SF_WS_CREG
#define SF_WS_CREG 240
#endif
#ifndef SF_MBAR_SUSPEND_NS
#define SF_MBAR_SUSPEND_NS 0x100000
#endif

// Debug builds (-DSF_DEBUG_BOUNDS): every shared-memory load is checked against its ring
// slot and every global store against its buffer; a violation traps (compute-sanitizer is
// not available on the test pool).
#ifdef SF_DEBUG_BOUNDS
#define SF_CHK(p, lo, hi)                                                                   \
    do {                                                                                   \
        if ((const float *)(p) < (const float *)(lo) || (const float *)(p) + 4 > (const float *)(hi)) \
            __trap();                                                                      \
    } while (0)
#else
#define SF_CHK(p, lo, hi) \
    do {                  \
    } while (0)
#endif

namespace sftma {


__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// try_wait with a suspend-time hint: a waiting warp sleeps until the phase completes (or
// the hint expires) instead of spinning, leaving the issue slots to the other warps
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity), "r"(SF_MBAR_SUSPEND_NS)
            : "memory");
    }
}

// Orders this thread's earlier generic-proxy shared-memory reads (LDS) before later
// async-proxy writes to the same bytes (the producer's TMA refill after the release): a
// write-after-read across proxies, which the mbarrier release alone does not order.
// Measured: releasing a u slot right after its loads gave wrong values in 4 of 12 runs
// without the fence, 0 of 32 with it.  Every consumer release is fenced, and the output
// plane's releases come after the loaded values are consumed, so the fence has no loads
// left to wait for (configs[1] +1 %, configs[4] -0.4 % time vs no fence).
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                          uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void tma_load4(uint32_t dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                          int c3, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

// L2 prefetch of a TMA box (no shared memory, no completion tracking)
__device__ __forceinline__ void tma_prefetch3(const CUtensorMap *tm, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *tm)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// Tile geometry / shared-memory plan.  VY = 2 rows x VZ = 4 columns per thread: y-neighbour
// loads cost (2R/VY) x 4 B per point and z-halo loads (2 HZ/VZ) x 4 B, so a 2 x 4 block keeps
// shared-memory traffic under ~75 B per point even at r = 8, and its (2r+1) x 8-float
// register queue still fits in 255 registers (<= 244 used at r = 8, no spills).
// 7 consumer warps + 1 producer = 8 warps = 2 per SM sub-partition, which leaves each
// thread the full 255 registers (a ninth warp would put 3 warps on one sub-partition and
// cap every thread at 168 registers).
// Lane layout: LZ lanes along z x (32 / LZ) lane rows along y per warp.  LZ = 32 (default):
// a warp covers VY rows x 128 columns.  LZ = 8 ("narrow" tiles, 32 columns x 56 rows): the z
// remainder of grids whose n2 is not a multiple of 128 (configs[4]: 400 = 3 x 128 + 16),
// where 128-column tiles would be mostly idle lanes.  8 lanes x 16 B = one 128-B shared-
// memory wavefront per row, so the lane rows never share a bank phase (conflict-free).
// LAY = 1 ("wide", tuning vy = 3, r >= 5): 2 z per lane and 11 consumer warps -- 4 points per
// thread halve the register queue (2r+1 planes x points) so that 12 warps (3 per SM sub-
// partition) fit the register file: more warps to hide the FP latency that bounds the
// 7-warp layout at high order.  Tiles 22 x 64.
// LAY = 2 ("ws", tuning vy = 4): 8 consumer warps (2 per SM sub-partition, 16 x 128 tiles) and
// a producer WARPGROUP that hands its registers to the consumers (setmaxnreg): the launch
// holds 12 warps at 168 registers; the producer warpgroup shrinks to SF_WS_PREG (one warp
// issues the TMA loads, three exit), the consumers grow to SF_WS_CREG.  The 7-warp layout
// leaves the producer's sub-partition with one consumer warp: the eighth fills it.
template <int R, int VY, int LZ = 32, int LAY = 0>
struct Geo {
    static constexpr int VZ = LAY == 1 ? 2 : 4;
    static constexpr int NW = LAY == 1 ? 11 : LAY == 2 ? 8 : 7;  // consumer warps
    static constexpr int LY = 32 / LZ;                  // lane rows per warp
    static constexpr int BY = NW * LY * VY;             // rows per tile
    static constexpr int TZ = LZ * VZ;                  // columns per tile
    static constexpr int HZ = ((R + 3) / 4) * 4;        // z halo rounded up to 16 B
};

template <int R, int VY, int DM, int MODE, int LZ = 32, int LAY = 0>
struct Cfg {
    static constexpr bool DAMP = (DM == SF_DAMP_ARRAY);  // beta array streamed
    using G = Geo<R, VY, LZ, LAY>;
    static constexpr int VZ = G::VZ, NW = G::NW, BY = G::BY, TZ = G::TZ, HZ = G::HZ;
    static constexpr int W = TZ + 2 * HZ;               // smem row pitch of the u tile
    static constexpr int H = BY + 2 * R;                // rows of the u tile
    static constexpr int Q = 2 * R + 1;                 // register queue depth
    static constexpr int UST = ((W * H * 4 + 127) / 128) * 128;   // u ring stage bytes
    static constexpr int PL = TZ * BY * 4;              // one halo-free plane
    static constexpr int NPL = 2 + (DAMP ? 1 : 0) + (MODE == SF_MODE_GRAD ? 2 : 0);
    static constexpr int CST = NPL * PL;                // coefficient ring stage bytes
    static constexpr int BUDGET = 226 * 1024;
    // ring depths: the u ring must hold planes q..p (R + 1) plus the producer's lead, the
    // coefficient ring DC output planes.  Leads are balanced: DU up to R + 5 while the
    // coefficient ring keeps SF_DC_MIN stages, then the rest to the coefficients (up to 4;
    // below SF_DC_MIN only when even DU = R + 2 leaves no more, e.g. r = 8 GRAD + damping)
    // r >= 7: two coefficient stages are enough and the freed stage deepens the u ring's
    // lead from 1 to 2 planes (configs[3]: -1.1 %, A/B)
    static constexpr int DC_MIN = R >= 7 ? SF_DC_MIN_HI : SF_DC_MIN;
    static constexpr int DU_WANT = R + 5;
    static constexpr int DU_FIT = (BUDGET - DC_MIN * CST) / UST;
    static constexpr int DU = DU_FIT >= DU_WANT ? DU_WANT : (DU_FIT >= R + 2 ? DU_FIT : R + 2);
    static constexpr int DC_FIT = (BUDGET - DU * UST) / CST;
    static constexpr int DC = DC_FIT >= 4 ? 4 : DC_FIT;
    static constexpr int SMEM = DU * UST + DC * CST + 128;  // + alignment slack
    // NW consumer warps + 1 TMA producer warp (LAY = 2: + a producer warpgroup of 4)
    static constexpr int PWARPS = LAY == 2 ? 4 : 1;
    static constexpr int THREADS = 32 * (NW + PWARPS);
    static_assert(DC >= 1, "coefficient ring does not fit shared memory");
    static_assert(DU >= R + 2, "u ring does not fit shared memory");
};

// VZ consecutive floats <-> VZ/2 fp32x2 pair registers (LDS/STG .64 / .128)
template <int VZ>
__device__ __forceinline__ void ldp(const float *p, f2_t *v)
{
    if (VZ == 4) {
        const ulonglong2 t = *reinterpret_cast<const ulonglong2 *>(p);
        v[0] = t.x;
        v[1] = t.y;
    } else {
        v[0] = *reinterpret_cast<const unsigned long long *>(p);
    }
}
template <int VZ>
__device__ __forceinline__ void stp(float *p, const f2_t *v)
{
    if (VZ == 4) *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(v[0], v[1]);
    else *reinterpret_cast<unsigned long long *>(p) = v[0];
}
// predicated 16-/8-byte global store (no divergent branch around edge tiles)
template <int VZ>
__device__ __forceinline__ void stp_if(float *p, const f2_t *v, bool pred)
{
    if (VZ == 4)
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t"
                     "@q st.global.v2.b64 [%0], {%1, %2};\n\t}" ::"l"(p), "l"(v[0]), "l"(v[1]), "r"((uint32_t)pred)
                     : "memory");
    else
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t"
                     "@q st.global.b64 [%0], %1;\n\t}" ::"l"(p), "l"(v[0]), "r"((uint32_t)pred)
                     : "memory");
}
// fp16 snapshot store (SF_OPT_SNAP_HALF): p = (float*)snap_out + e addresses element e; the
// VZ values go to element e of the __half array at snap_out (round to nearest even)
template <int VZ>
__device__ __forceinline__ void stsnap_half(float *snap_out, float *p, const f2_t *v)
{
    __half2 *hp = reinterpret_cast<__half2 *>(reinterpret_cast<__half *>(snap_out) + (p - snap_out));
#pragma unroll
    for (int jp = 0; jp < VZ / 2; ++jp) {
        float x, y;
        upk2(v[jp], x, y);
        hp[jp] = __floats2half2_rn(x, y);
    }
}

__device__ __forceinline__ float lo2(f2_t v)
{
    float a, b;
    upk2(v, a, b);
    return a;
}
__device__ __forceinline__ float hi2(f2_t v)
{
    float a, b;
    upk2(v, a, b);
    return b;
}

// fp32x2 form of sf_beta_sep: sxy = sx + sy (both lanes), sz = the lanes' sigma_z
__device__ __forceinline__ f2_t beta_sep2(f2_t sxy, f2_t sz, f2_t hdt2, f2_t one2, f2_t m1)
{
    const f2_t sh = mul2(add2(sxy, sz), hdt2);
    const f2_t den = add2(one2, sh);
    return mul2(fma2(m1, sh, one2), pk2(sf_rcp(lo2(den)), sf_rcp(hi2(den))));
}

// Work split: per tile the planes [xa, xb) then [xa2, xb2) (PT in all), cut into `nchunk`
// chunks of `chunk` planes; item it = (tile it % tiles, chunk it / tiles); CTA b takes items
// b, b + G, b + 2G, ...  Consecutive CTAs work on y/z-neighbouring tiles of the same chunk at
// the same time, so the tiles' shared halo rows are read from HBM once and hit in L2 for the
// neighbour.  A chunk crossing from the first range into the second is two segments.
struct Seg {
    int tile;
    int64_t qa, qb;
};
__device__ __forceinline__ Seg next_seg(int64_t w, int64_t end, int64_t P1, int64_t PT,
                                        const SfStepArgs &a)
{
    Seg s;
    s.tile = (int)(w / PT);
    const int64_t pl = w - (int64_t)s.tile * PT;
    int64_t lim;
    if (pl < P1) {
        s.qa = a.xa + pl;
        lim = P1 - pl;
    } else {
        s.qa = a.xa2 + (pl - P1);
        lim = PT - pl;
    }
    s.qb = s.qa + min(lim, end - w);
    return s;
}

// streaming direction of a segment: +1 (ascending x), or -1 for the last chunk of a tile in
// the one-launch slab schedule (SfStepArgs::bidir; needs two or more chunks per tile)
__device__ __forceinline__ int seg_dir(const SfStepArgs &a, int it, int tiles, int nchunk, int64_t w1,
                                       int64_t PT)
{
    return (a.bidir && nchunk > 1 && it / tiles == nchunk - 1 && w1 == (int64_t)(it % tiles + 1) * PT) ? -1 : 1;
}

// BIDIR: 0 plain; 1 one-launch slab schedule (downward last chunk, boundary signals); 2 the
// same + peer stores of the boundary planes (SF_OPT_P2P) -- separate instances, so that
// neither the plain kernel nor the NCCL form pays for code it does not run
template <int R, int VY, int DM, int MODE, int LZ = 32, int BIDIR = 0, int LAY = 0>
__global__ void __launch_bounds__(Cfg<R, VY, DM, MODE, LZ, LAY>::THREADS, 1)
k_tma3d(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_old,
        const __grid_constant__ CUtensorMap tm_c3, const __grid_constant__ CUtensorMap tm_beta,
        const __grid_constant__ CUtensorMap tm_snap, const __grid_constant__ CUtensorMap tm_grad,
        const SfStepArgs a, const int snap_slot, const int chunk, const int nchunk)
{
    using C = Cfg<R, VY, DM, MODE, LZ, LAY>;
    constexpr bool DAMP = C::DAMP;
    constexpr int VZ = C::VZ, NJ = VZ / 2, NW = C::NW, BY = C::BY, TZ = C::TZ, HZ = C::HZ;
    constexpr int Q = C::Q, W = C::W, DU = C::DU, DC = C::DC;
    // merged Laplacian form (sf_merged3: one chain over the three axes per radius, 7 instead
    // of 8 FP operations) at r >= 5 outside the gradient's GRAD mode (stencil_common.cuh)
    constexpr bool MRG = sf_merged_form(R, MODE);
    const int PD = a.l2_prefetch;  // planes of L2 prefetch beyond the smem ring (0 = off)
    // slot release by the consumers: one arrive per warp (lane 0, after __syncwarp).  Per-
    // thread arrives (tried for r >= 5, 1.6 % faster on configs[3]) produced rare wrong values
    // when small blocks of another kernel (the side-stream records) shared the SM.
    constexpr int ARRIVERS = C::NW;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    // keep the address space visible to the compiler (LDS, not generic LD)
    unsigned char *smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    unsigned char *cring = smem + DU * C::UST;
    __shared__ __align__(8) uint64_t bars[2 * DU + 2 * DC];
    const uint32_t ufull = smem_u32(bars), uempty = ufull + 8 * DU;
    const uint32_t cfull = uempty + 8 * DU, cempty = cfull + 8 * DC;

    const int lane = threadIdx.x, wy = threadIdx.y;
    const int64_t P1 = a.xb - a.xa, PT = P1 + (a.xb2 - a.xa2);
    // tiles cover the columns [zbase, n2t) (a split launch: the 128-column tiles, then the
    // narrow remainder tiles); neighbours beyond that range are still read (real halo)
    const int ntz = (int)((a.n2t - a.zbase + TZ - 1) / TZ);
    const int tiles = ntz * (int)((a.n1 + BY - 1) / BY);
    // nchunk == 0: balanced contiguous split -- CTA b walks the planes [b T / G, (b + 1) T / G)
    // of the tile-major sequence of all T = tiles x PT (tile, plane) units (one "item" per CTA,
    // cut into segments at tile boundaries): every CTA gets the same number of planes whatever
    // the tile count, at the price of neighbouring tiles drifting apart in x (their shared halo
    // rows then come from HBM twice); otherwise items = (tile, x-chunk) dealt round-robin.
    const bool bal = nchunk == 0;
    const int64_t TT = (int64_t)tiles * PT;
    const int items = bal ? (int)gridDim.x : tiles * nchunk;
    if ((int)blockIdx.x >= items) return;  // uniform over the CTA
    auto item_w0 = [&](int it) -> int64_t {
        return bal ? TT * it / gridDim.x : (int64_t)(it % tiles) * PT + (int64_t)(it / tiles) * chunk;
    };
    auto item_w1 = [&](int it) -> int64_t {
        return bal ? TT * (it + 1) / gridDim.x : min((int64_t)(it % tiles) * PT + (int64_t)(it / tiles + 1) * chunk,
                                                      (int64_t)(it % tiles + 1) * PT);
    };

    if (wy == 0 && lane == 0) {
#pragma unroll 1
        for (int s = 0; s < DU; ++s) {
            mbar_init(ufull + 8 * s, 1);
            mbar_init(uempty + 8 * s, ARRIVERS);
        }
#pragma unroll 1
        for (int s = 0; s < DC; ++s) {
            mbar_init(cfull + 8 * s, 1);
            mbar_init(cempty + 8 * s, ARRIVERS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    sf_pdl_wait();  // (PDL) the prologue above overlapped the previous kernel's tail

    if (LAY == 2) {
        // register hand-over between the warpgroups (12 warps x 168 at launch): producer
        // warpgroup 24 x 128, consumers 240 x 256 threads = 64 512 <= 65 536
        if (wy >= NW) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(SF_WS_PREG));
        else asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SF_WS_CREG));
    }
    if (wy >= NW) {
        // ------------------------------------------------ producer warp (TMA issue)
        if (wy == NW && lane == 0) {
            prefetch_tmap(&tm_cur);
            prefetch_tmap(&tm_old);
            prefetch_tmap(&tm_c3);
            if (DAMP) prefetch_tmap(&tm_beta);
            const uint32_t ubase = smem_u32(smem), cbase = smem_u32(cring);
            int us = 0, cs = 0;
            uint32_t uph = 0, cph = 0;
            int64_t gu = 0, gc = 0;  // ring uses so far
            for (int it = blockIdx.x; it < items; it += gridDim.x)
            for (int64_t w = item_w0(it), w1 = item_w1(it); w < w1;) {
                const Seg sg = next_seg(w, w1, P1, PT, a);
                // (BIDIR instances only: the one-launch slab schedule; elsewhere dir == 1 folds)
                const int dir = BIDIR ? seg_dir(a, it, tiles, nchunk, w1, PT) : 1;
                w += sg.qb - sg.qa;
                const int z0 = (int)a.zbase + (sg.tile % ntz) * TZ, y0 = (sg.tile / ntz) * BY;
                const int NP = (int)(sg.qb - sg.qa) + 2 * R;
                for (int i = 0; i < NP; ++i) {
                    // plane of u^n / output plane (downward segments start at qb - 1 + R)
                    const int p = dir > 0 ? (int)(sg.qa - R) + i : (int)(sg.qb - 1 + R) - i;
                    const int q = p - dir * R;
                    if (gu >= DU) mbar_wait(uempty + 8 * us, uph ^ 1u);
                    mbar_expect_tx(ufull + 8 * us, W * C::H * 4);  // full box, OOB zero-filled
                    tma_load3(ubase + us * C::UST, &tm_cur, z0 - HZ, y0 - R, p, ufull + 8 * us);
                    ++gu;
                    if (++us == DU) {
                        us = 0;
                        uph ^= 1u;
                    }
                    if (i >= 2 * R) {
                        if (gc >= DC) mbar_wait(cempty + 8 * cs, cph ^ 1u);
                        const uint32_t fb = cfull + 8 * cs;
                        // fp16 snapshots: that plane of the stage carries half the bytes
                        mbar_expect_tx(fb, C::CST - ((MODE == SF_MODE_GRAD && a.snap_half) ? C::PL / 2 : 0));
                        uint32_t pl = cbase + cs * C::CST;
                        tma_load3(pl, &tm_old, z0, y0, q, fb);
                        pl += C::PL;
                        tma_load3(pl, &tm_c3, z0, y0, q, fb);
                        pl += C::PL;
                        if (DAMP) {
                            tma_load3(pl, &tm_beta, z0, y0, q, fb);
                            pl += C::PL;
                        }
                        if (MODE == SF_MODE_GRAD) {
                            tma_load4(pl, &tm_snap, z0, y0, q, snap_slot, fb);
                            pl += C::PL;
                            tma_load3(pl, &tm_grad, z0, y0, q, fb);
                        }
                        ++gc;
                        if (++cs == DC) {
                            cs = 0;
                            cph ^= 1u;
                        }
                    }
                    // warm L2 PD planes ahead of the smem rings
                    if (PD > 0 && i + PD < NP) {
                        const int pp = p + dir * PD, qq = q + dir * PD;
                        tma_prefetch3(&tm_cur, z0 - HZ, y0 - R, pp);
                        if (i + PD >= 2 * R) {
                            tma_prefetch3(&tm_old, z0, y0, qq);
                            tma_prefetch3(&tm_c3, z0, y0, qq);
                            if (DAMP) tma_prefetch3(&tm_beta, z0, y0, qq);
                        }
                    }
                }
            }
        }
        return;
    }

    // ---------------------------------------------------- consumer warps
    f2_t V[Q][VY][NJ];  // own u at planes (fp32 pairs), slot = iteration index mod Q
    static_assert(Q <= 17, "slot switch covers r <= 8");
    constexpr int LY = C::G::LY;
    const int lz = lane % LZ, ly = lane / LZ;        // lane position in the warp's block
    const int rr = VY * (wy * LY + ly);              // first own row in the tile
    const int rown = R + rr;                         // first own row in the u tile
    const float *ubase = reinterpret_cast<const float *>(smem);
    const float *cbase = reinterpret_cast<const float *>(cring);
    constexpr int UF = C::UST / 4, CF = C::CST / 4, PF = C::PL / 4;  // strides in floats
    const int own_off = rown * W + HZ + VZ * lz;        // own values in a u tile
    const int po = rr * TZ + VZ * lz;                   // own values (row 0) in a plane
    int us = 0, uo = DU - R, cs = 0;                    // uo: u slot of plane q = p - R
    uint32_t uph = 0, cph = 0;
    const int n2 = (int)a.n2;
    const int64_t plane = a.n1 * a.n2;
    // packed constants
    f2_t Wk[R + 1];
#pragma unroll
    for (int k = 1; k <= R; ++k) Wk[k] = pk2(a.w.w[k], a.w.w[k]);
    Wk[0] = 0ull;
    const f2_t M4 = pk2(-4.f, -4.f), M2 = pk2(-2.f, -2.f), M1 = pk2(-1.f, -1.f), M6 = pk2(-6.f, -6.f);
    const f2_t NG = pk2(-a.gscale, -a.gscale), ONE2 = pk2(1.f, 1.f);
    const f2_t HDT2 = pk2(a.hdt, a.hdt);
    constexpr int QINF = 0x7fffffff;

    for (int it = blockIdx.x; it < items; it += gridDim.x)
    for (int64_t w = item_w0(it), w1 = item_w1(it); w < w1;) {
        const Seg sg = next_seg(w, w1, P1, PT, a);
        const int dir = BIDIR ? seg_dir(a, it, tiles, nchunk, w1, PT) : 1;
        w += sg.qb - sg.qa;
        const int z0 = (int)a.zbase + (sg.tile % ntz) * TZ, y0 = (sg.tile / ntz) * BY;
        const int zg = z0 + VZ * lz;
        const int yg = y0 + rr;
        const bool zact = zg < a.n2;
        // separable damping: profiles of the own rows / columns (clamped reads at ragged edges)
        float SY[VY];
        f2_t SZ[NJ], BYZ[VY][NJ];
        if (DM == SF_DAMP_SEP) {
#pragma unroll
            for (int j = 0; j < VY; ++j) SY[j] = __ldg(a.sigy + min(yg + j, (int)a.n1 - 1));
            const int zc = min(zg, (int)a.n2 - VZ);
#pragma unroll
            for (int jp = 0; jp < NJ; ++jp) SZ[jp] = pk2(__ldg(a.sigz + zc + 2 * jp), __ldg(a.sigz + zc + 2 * jp + 1));
#pragma unroll
            for (int j = 0; j < VY; ++j) {
                const float s0 = __fadd_rn(0.0f, SY[j]);
#pragma unroll
                for (int jp = 0; jp < NJ; ++jp) BYZ[j][jp] = beta_sep2(pk2(s0, s0), SZ[jp], HDT2, ONE2, M1);
            }
        }
        bool act[VY];
#pragma unroll
        for (int j = 0; j < VY; ++j) act[j] = zact && (yg + j < a.n1);
        const int qa = (int)sg.qa, qb = (int)sg.qb;
        const int NP = (qb - qa) + 2 * R;
        const int64_t dplane = dir * plane;
        float *optr = a.out + (int64_t)(dir > 0 ? qa : qb - 1) * plane + (int64_t)yg * a.n2 + zg;
        const int p0 = dir > 0 ? qa - R : qb - 1 + R;  // plane of u^n at iteration 0
        // boundary signals (one-launch slab schedule): the iteration after which this segment
        // has stored all of [xa, xa + r) (left) / [xb - r, xb) (right), else -1; checked once
        // per unrolled group of iterations (a check inside the unrolled body costs scheduling)
        int fiL = (BIDIR && a.sig && dir > 0 && qa == (int)a.xa) ? min((int)a.xa + R, qb) - 1 - qa + 2 * R : -1;
        int fiR = (BIDIR && a.sig && qb == (int)a.xb) ? (dir < 0 ? (qb - 1 - max((int)a.xb - R, qa)) + 2 * R : NP - 1) : -1;
        // snapshot row pointer (element offsets as the output; with fp16 snapshots it only
        // carries the element index, stsnap_half rebases it onto the __half array)
        float *sptr = (MODE == SF_MODE_SAVE) ? a.snap_out + (optr - a.out) : nullptr;
        float *gptr = (MODE == SF_MODE_GRAD) ? a.grad + (optr - a.out) : nullptr;
        // fused injection: this warp's cursor (warp-uniform), first entry at q >= qa
        // (downward segments walk the list backwards from the last entry at q < qb)
        int ci = 0, cb = 0, ce = 0, cq = QINF;
        if (MODE != SF_MODE_GRAD && a.inj_beg) {
            const int wl = sg.tile * NW + wy;
            cb = ci = a.inj_beg[wl];
            ce = a.inj_beg[wl + 1];
            if (dir > 0) {
                while (ci < ce && a.inj_q[ci] < qa) ++ci;
                cq = ci < ce ? a.inj_q[ci] : QINF;
            } else {
                ci = ce - 1;
                while (ci >= cb && a.inj_q[ci] >= qb) --ci;
                cq = ci >= cb ? a.inj_q[ci] : QINF;
            }
        }

        // The x-direction register queue needs compile-time slots; only that small part
        // (load plane p into its slot, x term of plane q) is replicated per slot through a
        // switch -- everything else exists once, which keeps the loop in the instruction
        // cache at r = 8 (a plane loop unrolled 2r+1 times thrashes it).
        // For r <= 4 the whole loop body is unrolled 2r+1 times instead (slot = unrolled
        // index, the switch folds away): small enough for the instruction cache, and the
        // stage/slot bookkeeping becomes compile-time.
        constexpr int UNR = (R <= 4) ? Q : 1;
        int sl = 0;  // queue slot of plane p: iteration index mod Q
#pragma unroll 1
        for (int base = 0; base < NP; base += UNR) {
#pragma unroll
        for (int s2 = 0; s2 < UNR; ++s2) {
                    const int i = base + s2;
                    if (i >= NP) break;
                    if (UNR == Q) sl = s2;
                    const int p = p0 + dir * i;
                    const bool outp = (i >= 2 * R);
                    // separable damping: sigma_x of the output plane q = p - R (issued early)
                    const float sxq = (DM == SF_DAMP_SEP && outp) ? __ldg(a.sigx + (p - dir * R)) : 0.0f;
                    // ---- (1) in-plane partial of output plane q = p - R: its u tile is
                    // resident (arrived R planes ago), so this overlaps the wait for plane p
                    f2_t Pin[VY][NJ], Uq[VY][NJ];
                    // in-plane terms of output plane q from its u tile; xs(j, jp, k) adds the x pair
                    // (merged form) or nothing (per-axis form: the x term is a separate chain)
                    auto inplane = [&](const float *uq, auto xs) {
                        // y rows rown - R .. rown + VY - 1 + R (own rows included)
                        f2_t Y[VY + 2 * R][NJ];
#pragma unroll
                        for (int t = 0; t < VY + 2 * R; ++t) {
                            SF_CHK(uq + own_off + (t - R) * W, uq, uq + W * C::H);
                            ldp<VZ>(uq + own_off + (t - R) * W, Y[t]);
                        }
#pragma unroll
                        for (int j = 0; j < VY; ++j)
#pragma unroll
                            for (int jp = 0; jp < NJ; ++jp) Uq[j][jp] = Y[R + j][jp];
                        // z halos of the own rows: floats [-HZ, 0) and [VZ, VZ + HZ)
                        f2_t ZL[VY][HZ / 2], ZR[VY][HZ / 2];
#pragma unroll
                        for (int j = 0; j < VY; ++j) {
#pragma unroll
                            for (int c = 0; c < HZ / VZ; ++c) {
                                SF_CHK(uq + own_off + j * W - HZ + VZ * c, uq, uq + W * C::H);
                                SF_CHK(uq + own_off + j * W + VZ + VZ * c, uq, uq + W * C::H);
                                ldp<VZ>(uq + own_off + j * W - HZ + VZ * c, ZL[j] + NJ * c);
                                ldp<VZ>(uq + own_off + j * W + VZ + VZ * c, ZR[j] + NJ * c);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < VY; ++j) {
                            // float at z offset e (relative to the own first column) of row j
                            auto F = [&](int e) -> float {
                                if (e < 0) {
                                    const int f = e + HZ;
                                    return (f & 1) ? hi2(ZL[j][f >> 1]) : lo2(ZL[j][f >> 1]);
                                }
                                if (e >= VZ) {
                                    const int f = e - VZ;
                                    return (f & 1) ? hi2(ZR[j][f >> 1]) : lo2(ZR[j][f >> 1]);
                                }
                                return (e & 1) ? hi2(Uq[j][e >> 1]) : lo2(Uq[j][e >> 1]);
                            };
                            // aligned pair starting at even z offset e
                            auto PZ = [&](int e) -> f2_t {
                                if (e < 0) return ZL[j][(e + HZ) >> 1];
                                if (e >= VZ) return ZR[j][(e - VZ) >> 1];
                                return Uq[j][e >> 1];
                            };
#pragma unroll
                            for (int jp = 0; jp < NJ; ++jp) {
                                const f2_t u = Uq[j][jp];
                                // radius ascending (== sf_inplane3 / sf_merged3 per lane)
                                f2_t P = 0ull;
#pragma unroll
                                for (int k = 1; k <= R; ++k) {
                                    const f2_t ys = add2(Y[R + j - k][jp], Y[R + j + k][jp]);
                                    const int em = 2 * jp - k, ep = 2 * jp + k;
                                    f2_t zs;
                                    if (k & 1)  // odd radius: unaligned pairs, two scalar adds
                                        zs = pk2(__fadd_rn(F(em), F(ep)), __fadd_rn(F(em + 1), F(ep + 1)));
                                    else
                                        zs = add2(PZ(em), PZ(ep));
                                    if constexpr (MRG)
                                        P = fma2(Wk[k], fma2(M6, u, add2(add2(ys, zs), xs(j, jp, k))), P);
                                    else
                                        P = fma2(Wk[k], fma2(M4, u, add2(ys, zs)), P);
                                }
                                Pin[j][jp] = P;
                            }
                        }
                    };
                    // ---- (1) in-plane partial of output plane q = p - R: its u tile is
                    // resident (arrived R planes ago), so this overlaps the wait for plane p
                    // (merged form: inside the slot code below, after the wait)
                    if (!MRG && outp) inplane(ubase + uo * UF, [](int, int, int) { return 0ull; });
                    // ---- (2) plane p of u^n into queue slot sl; x term of plane q (slot sl - R)
                    mbar_wait(ufull + 8 * us, uph);
                    const float *ut = ubase + us * UF;
                    f2_t X[VY][NJ];
                                        auto slot = [&](auto ic) {
                        constexpr int S = decltype(ic)::value;
                        constexpr int SQ = (S - R + Q) % Q;
#pragma unroll
                        for (int j = 0; j < VY; ++j) {
                            SF_CHK(ut + own_off + j * W, ut, ut + W * C::H);
                            ldp<VZ>(ut + own_off + j * W, V[S][j]);
                        }
                        if (MRG && outp) {
                            // merged form: one chain over the three axes per radius
                            inplane(ubase + uo * UF, [&](int j, int jp, int k) {
                                return add2(V[(SQ - k + Q) % Q][j][jp], V[(SQ + k) % Q][j][jp]);
                            });
                        } else if (outp) {
#pragma unroll
                            for (int j = 0; j < VY; ++j)
#pragma unroll
                                for (int jp = 0; jp < NJ; ++jp) {
                                    f2_t x = 0ull;
#pragma unroll
                                    for (int k = 1; k <= R; ++k)
                                        x = fma2(Wk[k], sf_xterm_x2(V[(SQ - k + Q) % Q][j][jp], V[(SQ + k) % Q][j][jp], V[SQ][j][jp], M2), x);
                                    X[j][jp] = x;
                                }
                        }
                    };
                    switch (sl) {
#define SF_SLOT(S_) \
    case S_:        \
        if constexpr (S_ < Q) slot(std::integral_constant<int, S_>{}); \
        break;
                        SF_SLOT(0) SF_SLOT(1) SF_SLOT(2) SF_SLOT(3) SF_SLOT(4) SF_SLOT(5) SF_SLOT(6)
                        SF_SLOT(7) SF_SLOT(8) SF_SLOT(9) SF_SLOT(10) SF_SLOT(11) SF_SLOT(12) SF_SLOT(13)
                        SF_SLOT(14) SF_SLOT(15) SF_SLOT(16)
#undef SF_SLOT
                    }
                    if (UNR != Q && ++sl == Q) sl = 0;
                    if (p < qa || p >= qb) {  // never an output plane: release the slot now
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(uempty + 8 * us);
                    }
                    if (outp) {
                        // ---- (3) finish output plane q: update, store ----
                        mbar_wait(cfull + 8 * cs, cph);
                        const float *cp = cbase + cs * CF + po;
                        f2_t ov[VY][NJ], cv[VY][NJ], bv[VY][NJ], sv[VY][NJ], gv[VY][NJ];
#pragma unroll
                        for (int j = 0; j < VY; ++j) {
                            SF_CHK(cp + j * TZ, cbase + cs * CF, cbase + cs * CF + C::NPL * PF);
                            SF_CHK(cp + PF + j * TZ, cbase + cs * CF, cbase + cs * CF + C::NPL * PF);
                            ldp<VZ>(cp + j * TZ, ov[j]);
                            ldp<VZ>(cp + PF + j * TZ, cv[j]);
                            int nxt = 2;
                            if (DAMP) {
                                ldp<VZ>(cp + 2 * PF + j * TZ, bv[j]);
                                nxt = 3;
                            } else if (DM == SF_DAMP_SEP) {
                                // beta regenerated from the separable profiles (== sf_beta_sep);
                                // planes with sigma_x = 0 (warp-uniform) reuse the per-segment
                                // beta(0, sigma_y, sigma_z) -- the same bits, as 0 + sy == sy
                                if (sxq == 0.0f) {
#pragma unroll
                                    for (int jp = 0; jp < NJ; ++jp) bv[j][jp] = BYZ[j][jp];
                                } else {
                                    const f2_t sxy = pk2(__fadd_rn(sxq, SY[j]), __fadd_rn(sxq, SY[j]));
#pragma unroll
                                    for (int jp = 0; jp < NJ; ++jp) bv[j][jp] = beta_sep2(sxy, SZ[jp], HDT2, ONE2, M1);
                                }
                            } else {
#pragma unroll
                                for (int jp = 0; jp < NJ; ++jp) bv[j][jp] = ONE2;
                            }
                            if (MODE == SF_MODE_GRAD) {
                                if (a.snap_half) {  // fp16 plane: VZ halves per lane, widened exactly
                                    const __half2 *hp = reinterpret_cast<const __half2 *>(
                                        reinterpret_cast<const __half *>(cp - po + nxt * PF) + (po + j * TZ));
#pragma unroll
                                    for (int jp = 0; jp < NJ; ++jp) {
                                        const float2 f = __half22float2(hp[jp]);
                                        sv[j][jp] = pk2(f.x, f.y);
                                    }
                                } else {
                                    ldp<VZ>(cp + nxt * PF + j * TZ, sv[j]);
                                }
                                ldp<VZ>(cp + (nxt + 1) * PF + j * TZ, gv[j]);
                            }
                        }
                        // done with the u tile of plane q and the coefficient stage
                        const int q = p - dir * R;
                        f2_t res2[VY][NJ], gres2[VY][NJ];
#pragma unroll
                        for (int j = 0; j < VY; ++j) {
#pragma unroll
                            for (int jp = 0; jp < NJ; ++jp) {
                                const f2_t u = Uq[j][jp];
                                const f2_t lap = MRG ? Pin[j][jp] : add2(Pin[j][jp], X[j][jp]);
                                // out = u + beta (u - old) + c3 lap   (== sf_update per lane)
                                const f2_t d = fma2(M1, ov[j][jp], u);
                                res2[j][jp] = fma2(cv[j][jp], lap, fma2(bv[j][jp], d, u));
                                if (MODE == SF_MODE_GRAD) {
                                    // S = (beta - 1) d + c3 lap ; g -= gscale * snap * S
                                    const f2_t S2 = fma2(add2(bv[j][jp], M1), d, mul2(cv[j][jp], lap));
                                    gres2[j][jp] = fma2(NG, mul2(sv[j][jp], S2), gv[j][jp]);
                                }
                            }
                        }
                        // done with the u tile of plane q and the coefficient stage: released
                        // after their values are consumed (the fence then has no loads to wait for)
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(uempty + 8 * uo);
                            mbar_arrive(cempty + 8 * cs);
                        }
                        if (++cs == DC) {
                            cs = 0;
                            cph ^= 1u;
                        }
                        if (MODE != SF_MODE_GRAD && cq == q) {
                            // fused injection, rare path: res[t] += sum_e coef_e vals[pt_e]
                            // (the fp32 operations of k_inject, bitwise); lj = ((jy 32 + lane) 4 + jz)
                            float res[VY][VZ];
#pragma unroll
                            for (int j = 0; j < VY; ++j)
#pragma unroll
                                for (int jp = 0; jp < NJ; ++jp) upk2(res2[j][jp], res[j][2 * jp], res[j][2 * jp + 1]);
                            do {
                                const int lj = a.inj_lj[ci];
                                if (((lj >> 2) & 31) == lane) {
                                    const int t = a.inj_t[ci];
                                    float dd = 0.f;
#pragma unroll 1
                                    for (int e = a.inj_rowptr[t]; e < a.inj_rowptr[t + 1]; ++e)
                                        dd = __fmaf_rn(a.inj_coef[e], a.inj_vals[a.inj_pt[e]], dd);
                                    const int jy = lj >> 7, jz = lj & 3;
#pragma unroll
                                    for (int j = 0; j < VY; ++j)
#pragma unroll
                                        for (int jj = 0; jj < VZ; ++jj)
                                            res[j][jj] = (jy == j && jz == jj) ? __fadd_rn(res[j][jj], dd) : res[j][jj];
                                }
                                if (dir > 0) {
                                    ++ci;
                                    cq = ci < ce ? a.inj_q[ci] : QINF;
                                } else {
                                    --ci;
                                    cq = ci >= cb ? a.inj_q[ci] : QINF;
                                }
                            } while (cq == q);
#pragma unroll
                            for (int j = 0; j < VY; ++j)
#pragma unroll
                                for (int jp = 0; jp < NJ; ++jp) res2[j][jp] = pk2(res[j][2 * jp], res[j][2 * jp + 1]);
                        }
                        if (UNR == 1) {
                            // rolled loop (r >= 5): predicated stores, no divergent branches
                            // (measured 5 % faster on configs[3])
#pragma unroll
                            for (int j = 0; j < VY; ++j) {
                                if (act[j]) SF_CHK(optr + j * n2, a.out, a.out + a.n0b * plane);
                                stp_if<VZ>(optr + j * n2, res2[j], act[j]);
                                if (MODE == SF_MODE_SAVE) {
                                    if (a.snap_half) {
                                        if (act[j]) stsnap_half<VZ>(a.snap_out, sptr + j * n2, res2[j]);
                                    } else {
                                        stp_if<VZ>(sptr + j * n2, res2[j], act[j]);
                                    }
                                }
                                if (MODE == SF_MODE_GRAD) stp_if<VZ>(gptr + j * n2, gres2[j], act[j]);
                            }
                        } else {
                            // unrolled loop (r <= 4): plain branchy stores -- the predicated
                            // form measured 8 % slower here (scheduling of the unrolled body)
                            if (zact) {
#pragma unroll
                                for (int j = 0; j < VY; ++j) {
                                    if (yg + j < a.n1) {
                                        SF_CHK(optr + j * a.n2, a.out, a.out + a.n0b * plane);
                                        stp<VZ>(optr + j * a.n2, res2[j]);
                                        if (MODE == SF_MODE_SAVE) {
                                            if (a.snap_half) stsnap_half<VZ>(a.snap_out, sptr + j * a.n2, res2[j]);
                                            else stp<VZ>(sptr + j * a.n2, res2[j]);
                                        }
                                        if (MODE == SF_MODE_GRAD) stp<VZ>(gptr + j * a.n2, gres2[j]);
                                    }
                                }
                            }
                        }
                        if (BIDIR == 2 && ((q >= a.mq[0] && q < a.mq[1]) || (q >= a.mq[2] && q < a.mq[3]))) {
                            // peer-store halo exchange (SF_OPT_P2P): a boundary plane
                            // is also stored straight into the neighbour's halo of the same level
                            // (peer-mapped buffer at byte offset md from its own address)
                            const int64_t db = (q < a.mq[1]) ? a.md[0] : a.md[1];
#pragma unroll
                            for (int j = 0; j < VY; ++j)
                                if (act[j]) stp<VZ>(sf_mirror(optr + j * a.n2, db), res2[j]);
                        }
                        optr += dplane;
                        if (MODE == SF_MODE_SAVE) sptr += dplane;
                        if (MODE == SF_MODE_GRAD) gptr += dplane;

                    }
                    if (++us == DU) {
                        us = 0;
                        uph ^= 1u;
                    }
                    if (++uo == DU) uo = 0;
        }
            // one-launch schedule: a boundary range of this tile is stored -> every consumer
            // thread fences its stores, the consumer warps meet, one thread signals
            const int done = base + UNR;  // iterations finished (or more: the last group)
            const bool fl = BIDIR && fiL >= 0 && done > fiL, fr = BIDIR && fiR >= 0 && done > fiR;
            if (BIDIR && (fl || fr)) {
                __threadfence();
                asm volatile("bar.sync 1, %0;" ::"r"(NW * 32) : "memory");
                if (wy == 0 && lane == 0) {
                    if (fl) atomicAdd(a.sig + 0, 1u);
                    if (fr) atomicAdd(a.sig + 1, 1u);
                }
                if (fl) fiL = -1;
                if (fr) fiR = -1;
            }
        }
    }
}

}  // namespace sftma
