// stencil_tma.cuh -- sm_100a 2.5D streaming stencil step, TMA-fed, register-rotated.
//
// Hot kernel of the path (memory-bandwidth bound):
// each CTA owns a (y, z) tile of BY rows x 128 columns and streams along x (the
// outermost, slab axis) over a chunk of planes.  Per plane p:
//   * one elected thread issues TMA (cp.async.bulk.tensor) loads into an S-stage
//     shared-memory ring, completion tracked by mbarrier transaction counts:
//       - u^n plane p with its (y, z) halo: box (128 + 2 HZ) x (BY + 2R); the TMA
//         out-of-bounds zero fill IS the zero ghost halo (reading C6),
//       - old / c3 / beta (and snapshot / gradient in GRAD mode) of output plane q = p - R;
//   * every thread (4 consecutive z of one y row) reads its z-row and 2R y-neighbour
//     rows as float4 (conflict-free), forms the in-plane partial P_p at arrival and
//     pushes u_p and P_p into register queues of depth 2R+1 (compile-time rotated by
//     unrolling the plane loop by 2R+1: no register moves);
//   * output plane q = p - R is finished from the queues: X = sum_k w_k((u_{q-k}+u_{q+k})-2u_q),
//     Lap = P_q + X, out = u + beta (u - old) + c3 Lap, stored with STG.128 in place
//     over `old` (plus the snapshot copy / fused gradient correlation).
// HBM traffic per point (compulsory): read u^n, old, c3 (+beta) and write out:
// 16 B (20 B with damping); x-chunk warm-up re-reads 2R planes of u^n per chunk.
#pragma once
#include <cuda.h>
#include "stencil_common.cuh"

namespace sftma {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                          uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load4(void *dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                          int c3, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
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

__device__ __forceinline__ void stg4(float *p, float4 v)
{
    *reinterpret_cast<float4 *>(p) = v;
}

template <int R, int BY, int VZ, bool DAMP, int MODE>
struct Cfg {
    static constexpr int TZ = 32 * VZ;                   // z columns per CTA (32 lanes x VZ)
    static constexpr int HZ = ((R + 3) / 4) * 4;         // z halo rounded up to 4 floats
    static constexpr int W = TZ + 2 * HZ;                // smem row pitch of the u^n tile
    static constexpr int H = BY + 2 * R;                 // rows of the u^n tile
    static constexpr int Q = 2 * R + 1;                  // register queue depth
    static constexpr int CUR_BYTES = ((W * H * 4 + 127) / 128) * 128;
    static constexpr int PL_BYTES = TZ * BY * 4;         // one plane without halo
    static constexpr int NPL = 2 + (DAMP ? 1 : 0) + (MODE == SF_MODE_GRAD ? 2 : 0);
    static constexpr int STAGE_BYTES = CUR_BYTES + NPL * PL_BYTES;
    static constexpr int PRING = R;                      // in-plane partials kept for R planes
                                                          // (slot read for plane p-R, then rewritten with p)
    static constexpr int PRING_BYTES = PRING * PL_BYTES;
    static constexpr int S_MAX = (220 * 1024 - PRING_BYTES) / STAGE_BYTES;
    // pipeline depth: 4 stages for r <= 4 (measured equal to 5 on configs[1]; keeps two
    // BY = 8 CTAs per SM), 5 for r >= 5 (4 % faster on configs[3])
    static constexpr int S_WANT = R >= 5 ? 5 : 4;
    static constexpr int S = S_MAX >= S_WANT ? S_WANT : S_MAX;
    static constexpr int SMEM = S * STAGE_BYTES + PRING_BYTES + 128;  // + alignment slack
    static constexpr int THREADS = 32 * (BY + 1);         // BY consumer warps + 1 TMA producer warp
    static_assert(S >= 2, "stage does not fit shared memory");
    static_assert(VZ == 2 || VZ == 4, "VZ");
};

// VZ consecutive floats <-> VZ/2 fp32x2 pair registers (LDS/STS/STG .64 / .128)
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

// VZ consecutive floats <-> registers (LDS.64 / LDS.128, STG.64 / STG.128)
template <int VZ>
__device__ __forceinline__ void ldv(const float *p, float *v)
{
    if (VZ == 4) {
        const float4 t = *reinterpret_cast<const float4 *>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
        const float2 t = *reinterpret_cast<const float2 *>(p);
        v[0] = t.x; v[1] = t.y;
    }
}
template <int VZ>
__device__ __forceinline__ void stv(float *p, const float *v)
{
    if (VZ == 4) *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
}

// One CTA = BY consumer warps (one y row each, VZ consecutive z per lane) + 1 producer
// warp whose elected lane issues every TMA load.  Per stage: `full` (TMA transaction
// bytes) and `empty` (one arrive per consumer warp) mbarriers.
template <int R, int BY, int VZ, bool DAMP, int MODE>
__global__ void __launch_bounds__(32 * (BY + 1), (BY == 8 && R <= 4) ? 2 : 1)
k_tma3d(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_old,
        const __grid_constant__ CUtensorMap tm_c3, const __grid_constant__ CUtensorMap tm_beta,
        const __grid_constant__ CUtensorMap tm_snap, const __grid_constant__ CUtensorMap tm_grad,
        const SfStepArgs a, const int snap_slot, const int chunk)
{
    using C = Cfg<R, BY, VZ, DAMP, MODE>;
    constexpr int NJ = VZ / 2;  // fp32x2 pairs per lane
    constexpr int Q = C::Q, TZ = C::TZ, HZ = C::HZ, W = C::W, S = C::S, PR = C::PRING;
    const int PD = a.l2_prefetch;  // planes of L2 prefetch beyond the smem ring (0 = off)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // keep the address space visible to the compiler (LDS, not generic LD): align by
    // offsetting the shared array itself
    unsigned char *smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    float *pring = reinterpret_cast<float *>(smem + S * C::STAGE_BYTES);
    __shared__ __align__(8) uint64_t full[S];   // TMA bytes landed in stage s
    __shared__ __align__(8) uint64_t empty[S];  // every consumer warp finished reading stage s

    const int lane = threadIdx.x, wy = threadIdx.y;
    const int z0 = blockIdx.x * TZ, y0 = blockIdx.y * BY;
    // chunk -> planes [qa, qb): chunks of the first range, then of the optional second
    int64_t zc = blockIdx.z, ra = a.xa, rb = a.xb;
    {
        const int64_t nch1 = (a.xb - a.xa + chunk - 1) / chunk;
        if (zc >= nch1) {
            zc -= nch1;
            ra = a.xa2;
            rb = a.xb2;
        }
    }
    const int64_t qa = ra + zc * chunk;
    const int64_t qb = min(qa + (int64_t)chunk, rb);
    if (qa >= qb) return;  // uniform over the CTA
    const int NP = (int)(qb - qa) + 2 * R;

    if (wy == 0 && lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], BY);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    if (wy == BY) {
        // ------------------------------------------------ producer warp (TMA issue)
        if (lane == 0) {
            prefetch_tmap(&tm_cur);
            prefetch_tmap(&tm_old);
            prefetch_tmap(&tm_c3);
            int st = 0;
            uint32_t ph = 0;
            for (int i = 0; i < NP; ++i) {
                if (i >= S) mbar_wait(&empty[st], ph ^ 1u);
                unsigned char *base = smem + st * C::STAGE_BYTES;
                const int p = (int)(qa - R) + i;   // plane of u^n
                const int q = p - R;               // output plane
                const bool outp = (i >= 2 * R);
                uint32_t bytes = W * C::H * 4;    // full box; out-of-bounds part zero-filled
                if (outp) bytes += C::NPL * C::PL_BYTES;
                mbar_expect_tx(&full[st], bytes);
                tma_load3(base, &tm_cur, z0 - HZ, y0 - R, p, &full[st]);
                if (outp) {
                    unsigned char *pl = base + C::CUR_BYTES;
                    tma_load3(pl, &tm_old, z0, y0, q, &full[st]);
                    pl += C::PL_BYTES;
                    tma_load3(pl, &tm_c3, z0, y0, q, &full[st]);
                    pl += C::PL_BYTES;
                    if (DAMP) {
                        tma_load3(pl, &tm_beta, z0, y0, q, &full[st]);
                        pl += C::PL_BYTES;
                    }
                    if (MODE == SF_MODE_GRAD) {
                        tma_load4(pl, &tm_snap, z0, y0, q, snap_slot, &full[st]);
                        pl += C::PL_BYTES;
                        tma_load3(pl, &tm_grad, z0, y0, q, &full[st]);
                    }
                }
                // warm L2 PD planes ahead of the smem ring: the smem stages then fill from
                // L2 and the ring depth no longer has to cover the full HBM latency
                if (PD > 0 && i + PD < NP) {
                    const int pp = p + PD, qq = q + PD;
                    tma_prefetch3(&tm_cur, z0 - HZ, y0 - R, pp);
                    if (i + PD >= 2 * R) {
                        tma_prefetch3(&tm_old, z0, y0, qq);
                        tma_prefetch3(&tm_c3, z0, y0, qq);
                        if (DAMP) tma_prefetch3(&tm_beta, z0, y0, qq);
                    }
                }
                if (++st == S) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }

    // ---------------------------------------------------- consumer warps
    f2_t V[Q][NJ];  // u at planes (fp32 pairs), slot = iteration index mod Q
    const int rown = R + wy;
    const int zg = z0 + VZ * lane;
    const int yg = y0 + wy;
    const bool active = (zg < a.n2) && (yg < a.n1);
    const int64_t plane = a.n1 * a.n2;
    const int64_t rowoff = (int64_t)yg * a.n2 + zg;
    const int po = wy * TZ + VZ * lane;  // this thread's VZ floats in a halo-free plane
    float *myP = pring + po;            // private ring of in-plane partials (stride PL floats)
    int st = 0, pw = 0;
    uint32_t ph = 0;
    // packed constants: weights {w_k, w_k}, -4, -2, -1, -gscale
    f2_t Wk[R + 1];
#pragma unroll
    for (int k = 1; k <= R; ++k) Wk[k] = pk2(a.w.w[k], a.w.w[k]);
    Wk[0] = 0ull;
    const f2_t M4 = pk2(-4.f, -4.f), M2 = pk2(-2.f, -2.f), M1 = pk2(-1.f, -1.f);
    const f2_t NG = pk2(-a.gscale, -a.gscale), ONE2 = pk2(1.f, 1.f);
    // fused sparse work: this warp's cursors (warp-uniform), first entries at q >= qa
    constexpr int QINF = 0x7fffffff;
    int ci = 0, ce = 0, cq = QINF;
    {
        const int wl = (blockIdx.y * gridDim.x + blockIdx.x) * BY + wy;
        if (a.inj_beg) {
            ci = a.inj_beg[wl];
            ce = a.inj_beg[wl + 1];
            while (ci < ce && a.inj_q[ci] < qa) ++ci;
            cq = ci < ce ? a.inj_q[ci] : QINF;
        }
    }

    for (int base = 0; base < NP; base += Q) {
#pragma unroll
        for (int s = 0; s < Q; ++s) {
            const int i = base + s;
            if (i < NP) {
                mbar_wait(&full[st], ph);
                const unsigned char *sb = smem + st * C::STAGE_BYTES;
                const float *cs = reinterpret_cast<const float *>(sb);
                // z row of this thread as aligned fp32 pairs: floats [VZ lane, VZ lane + 2 HZ + VZ)
                constexpr int NZP = (2 * HZ + VZ) / 2;
                f2_t zp[NZP];
#pragma unroll
                for (int c = 0; c < (2 * HZ + VZ) / VZ; ++c) ldp<VZ>(cs + rown * W + VZ * lane + VZ * c, zp + NJ * c);
                // odd-offset pairs (floats 2c+1, 2c+2), needed by odd radii
                f2_t zo[NZP - 1];
#pragma unroll
                for (int c = 0; c < NZP - 1; ++c) {
                    float a0, a1, b0, b1;
                    upk2(zp[c], a0, a1);
                    upk2(zp[c + 1], b0, b1);
                    zo[c] = pk2(a1, b0);
                }
#pragma unroll
                for (int jp = 0; jp < NJ; ++jp) V[s][jp] = zp[HZ / 2 + jp];
                // in-plane partial P_p = sum_k w_k ((y-k + y+k) + (z-k + z+k) - 4u), fp32x2
                f2_t pp2[NJ];
#pragma unroll
                for (int jp = 0; jp < NJ; ++jp) pp2[jp] = 0ull;
#pragma unroll
                for (int k = 1; k <= R; ++k) {
                    f2_t ym2[NJ], yp2[NJ];
                    ldp<VZ>(cs + (rown - k) * W + HZ + VZ * lane, ym2);
                    ldp<VZ>(cs + (rown + k) * W + HZ + VZ * lane, yp2);
#pragma unroll
                    for (int jp = 0; jp < NJ; ++jp) {
                        const int fm = HZ + 2 * jp - k, fpp = HZ + 2 * jp + k;  // float index of the pair start
                        const f2_t zm = (k & 1) ? zo[(fm - 1) / 2] : zp[fm / 2];
                        const f2_t zq = (k & 1) ? zo[(fpp - 1) / 2] : zp[fpp / 2];
                        const f2_t t = sf_inplane3_x2(ym2[jp], yp2[jp], zm, zq, V[s][jp], M4);
                        pp2[jp] = fma2(Wk[k], t, pp2[jp]);
                    }
                }
                const bool outp = (i >= 2 * R);
                f2_t ov[NJ], cv[NJ], bv[NJ], sv[NJ], gv[NJ], pq[NJ];
                if (!DAMP) {
#pragma unroll
                    for (int jp = 0; jp < NJ; ++jp) bv[jp] = ONE2;
                }
                if (outp) {
                    const float *pl = reinterpret_cast<const float *>(sb + C::CUR_BYTES);
                    ldp<VZ>(pl + po, ov);
                    ldp<VZ>(pl + TZ * BY + po, cv);
                    int nxt = 2;
                    if (DAMP) {
                        ldp<VZ>(pl + 2 * TZ * BY + po, bv);
                        nxt = 3;
                    }
                    if (MODE == SF_MODE_GRAD) {
                        ldp<VZ>(pl + nxt * TZ * BY + po, sv);
                        ldp<VZ>(pl + (nxt + 1) * TZ * BY + po, gv);
                    }
                }
                // this warp is done with the stage: release it to the producer
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == S) {
                    st = 0;
                    ph ^= 1u;
                }
                // P ring (thread-private slots, R deep): slot pw holds P_{p-R}; read it, then
                // overwrite it with P_p (same thread, program order)
                if (outp) ldp<VZ>(myP + pw * (TZ * BY), pq);
                stp<VZ>(myP + pw * (TZ * BY), pp2);
                if (++pw == PR) pw = 0;
                // ---- finish output plane q = p - R from the register queue ----
                if (outp) {
                    const int sq = (s - R + Q) % Q;  // compile-time after unrolling
                    const int64_t q = qa + (i - 2 * R);
                    f2_t res2[NJ], gres2[NJ];
#pragma unroll
                    for (int jp = 0; jp < NJ; ++jp) {
                        const f2_t u = V[sq][jp];
                        f2_t X = 0ull;
#pragma unroll
                        for (int k = 1; k <= R; ++k)
                            X = fma2(Wk[k], sf_xterm_x2(V[(sq - k + Q) % Q][jp], V[(sq + k) % Q][jp], u, M2), X);
                        const f2_t lap = add2(pq[jp], X);
                        // out = u + beta (u - old) + c3 lap   (== sf_update per lane)
                        const f2_t d = fma2(M1, ov[jp], u);
                        res2[jp] = fma2(cv[jp], lap, fma2(bv[jp], d, u));
                        if (MODE == SF_MODE_GRAD) {
                            // S = (beta - 1) d + c3 lap ; g -= gscale * snap * S   (== sf_d2 / sf_grad)
                            const f2_t S2 = fma2(add2(bv[jp], M1), d, mul2(cv[jp], lap));
                            gres2[jp] = fma2(NG, mul2(sv[jp], S2), gv[jp]);
                        }
                    }
                    if (MODE != SF_MODE_GRAD && cq == (int)q) {  // GRAD steps inject standalone
                        // fused injection, rare path: res[j] += sum_e coef_e vals[pt_e]
                        // (the fp32 operations of k_inject, bitwise)
                        float res[VZ];
#pragma unroll
                        for (int jp = 0; jp < NJ; ++jp) upk2(res2[jp], res[2 * jp], res[2 * jp + 1]);
                        do {
                            const int lj = a.inj_lj[ci];
                            if ((lj >> 2) == lane) {
                                const int t = a.inj_t[ci];
                                float dd = 0.f;
#pragma unroll 1
                                for (int e = a.inj_rowptr[t]; e < a.inj_rowptr[t + 1]; ++e)
                                    dd = __fmaf_rn(a.inj_coef[e], a.inj_vals[a.inj_pt[e]], dd);
                                const int j = lj & 3;
#pragma unroll
                                for (int jj = 0; jj < VZ; ++jj) res[jj] = (j == jj) ? __fadd_rn(res[jj], dd) : res[jj];
                            }
                            ++ci;
                            cq = ci < ce ? a.inj_q[ci] : QINF;
                        } while (cq == (int)q);
#pragma unroll
                        for (int jp = 0; jp < NJ; ++jp) res2[jp] = pk2(res[2 * jp], res[2 * jp + 1]);
                    }
                    if (active) {
                        const int64_t off = q * plane + rowoff;
                        stp<VZ>(a.out + off, res2);
                        if (MODE == SF_MODE_SAVE) stp<VZ>(a.snap_out + off, res2);
                        if (MODE == SF_MODE_GRAD) stp<VZ>(a.grad + off, gres2);
                    }
                }
            }
        }
    }
}

}  // namespace sftma
