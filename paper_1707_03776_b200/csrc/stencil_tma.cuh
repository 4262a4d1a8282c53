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

template <int R, int BY, bool DAMP, int MODE>
struct Cfg {
    static constexpr int TZ = 128;                       // z columns per CTA (32 lanes x 4)
    static constexpr int HZ = ((R + 3) / 4) * 4;         // z halo rounded up to 4 floats
    static constexpr int W = TZ + 2 * HZ;                // smem row pitch of the u^n tile
    static constexpr int H = BY + 2 * R;                 // rows of the u^n tile
    static constexpr int Q = 2 * R + 1;                  // register queue depth
    static constexpr int CUR_BYTES = ((W * H * 4 + 127) / 128) * 128;
    static constexpr int PL_BYTES = TZ * BY * 4;         // one plane without halo
    static constexpr int NPL = 2 + (DAMP ? 1 : 0) + (MODE == SF_MODE_GRAD ? 2 : 0);
    static constexpr int STAGE_BYTES = CUR_BYTES + NPL * PL_BYTES;
    static constexpr int PRING = R + 1;                  // in-plane partials kept for R planes
    static constexpr int PRING_BYTES = PRING * PL_BYTES;
    static constexpr int S_MAX = (220 * 1024 - PRING_BYTES) / STAGE_BYTES;
    static constexpr int S = S_MAX >= 4 ? 4 : S_MAX;      // pipeline depth
    static constexpr int SMEM = S * STAGE_BYTES + PRING_BYTES + 128;  // + alignment slack
    static constexpr int THREADS = 32 * (BY + 1);         // BY consumer warps + 1 TMA producer warp
    static_assert(S >= 2, "stage does not fit shared memory");
};

// One CTA = BY consumer warps (one y row each, 4 z per lane) + 1 producer warp whose
// elected lane issues every TMA load.  Per stage: `full` (TMA transaction bytes) and
// `empty` (one arrive per consumer warp) mbarriers.
template <int R, int BY, bool DAMP, int MODE>
__global__ void __launch_bounds__(32 * (BY + 1), (BY == 8 && R <= 4) ? 2 : 1)
k_tma3d(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_old,
        const __grid_constant__ CUtensorMap tm_c3, const __grid_constant__ CUtensorMap tm_beta,
        const __grid_constant__ CUtensorMap tm_snap, const __grid_constant__ CUtensorMap tm_grad,
        const SfStepArgs a, const int snap_slot, const int chunk)
{
    using C = Cfg<R, BY, DAMP, MODE>;
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
    const int64_t qa = a.xa + (int64_t)blockIdx.z * chunk;
    const int64_t qb = min(qa + (int64_t)chunk, a.xb);
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
    float V[Q][4];  // u at planes, slot = iteration index mod Q
    const int rown = R + wy;
    const int zg = z0 + 4 * lane;
    const int yg = y0 + wy;
    const bool active = (zg < a.n2) && (yg < a.n1);
    const int64_t plane = a.n1 * a.n2;
    const int64_t rowoff = (int64_t)yg * a.n2 + zg;
    const int po = wy * TZ + 4 * lane;   // this thread's float4 in a halo-free plane
    float *myP = pring + po;            // private ring of in-plane partials (stride PL floats)
    int st = 0, pw = 0;
    uint32_t ph = 0;
    // packed constants: weights {w_k, w_k}, -4, -2, -1, -gscale
    f2_t Wk[R + 1];
#pragma unroll
    for (int k = 1; k <= R; ++k) Wk[k] = pk2(a.w.w[k], a.w.w[k]);
    Wk[0] = 0ull;
    const f2_t M4 = pk2(-4.f, -4.f), M2 = pk2(-2.f, -2.f), M1 = pk2(-1.f, -1.f);
    const f2_t NG = pk2(-a.gscale, -a.gscale);
    // fused sparse work: this warp's cursors (warp-uniform), first entries at q >= qa
    constexpr int QINF = 0x7fffffff;
    int ci = 0, ce = 0, cq = QINF, pi = 0, pe = 0, pq_ = QINF;
    {
        const int wl = (blockIdx.y * gridDim.x + blockIdx.x) * BY + wy;
        if (a.inj_beg) {
            ci = a.inj_beg[wl];
            ce = a.inj_beg[wl + 1];
            while (ci < ce && a.inj_q[ci] < qa) ++ci;
            cq = ci < ce ? a.inj_q[ci] : QINF;
        }
        if (a.itp_beg) {
            pi = a.itp_beg[wl];
            pe = a.itp_beg[wl + 1];
            while (pi < pe && a.itp_q[pi] < qa) ++pi;
            pq_ = pi < pe ? a.itp_q[pi] : QINF;
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
                // z row of this thread: columns [4 lane, 4 lane + 2 HZ + 4)
                float zr[2 * HZ + 4];
#pragma unroll
                for (int c = 0; c < (2 * HZ + 4) / 4; ++c) {
                    const float4 t = *reinterpret_cast<const float4 *>(cs + rown * W + 4 * lane + 4 * c);
                    zr[4 * c + 0] = t.x;
                    zr[4 * c + 1] = t.y;
                    zr[4 * c + 2] = t.z;
                    zr[4 * c + 3] = t.w;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) V[s][j] = zr[HZ + j];
                // in-plane partial P_p = sum_k w_k ((y-k + y+k) + (z-k + z+k) - 4u), as
                // two fp32x2 lanes (points j, j+1)
                f2_t pp2[2] = {0ull, 0ull};
#pragma unroll
                for (int k = 1; k <= R; ++k) {
                    const float4 m4 = *reinterpret_cast<const float4 *>(cs + (rown - k) * W + HZ + 4 * lane);
                    const float4 p4 = *reinterpret_cast<const float4 *>(cs + (rown + k) * W + HZ + 4 * lane);
                    const f2_t ym2[2] = {pk2(m4.x, m4.y), pk2(m4.z, m4.w)};
                    const f2_t yp2[2] = {pk2(p4.x, p4.y), pk2(p4.z, p4.w)};
#pragma unroll
                    for (int jp = 0; jp < 2; ++jp) {
                        const int j = 2 * jp;
                        const f2_t t = sf_inplane3_x2(ym2[jp], yp2[jp], pk2(zr[HZ + j - k], zr[HZ + j + 1 - k]),
                                                      pk2(zr[HZ + j + k], zr[HZ + j + 1 + k]),
                                                      pk2(zr[HZ + j], zr[HZ + j + 1]), M4);
                        pp2[jp] = fma2(Wk[k], t, pp2[jp]);
                    }
                }
                float pp[4];
                upk2(pp2[0], pp[0], pp[1]);
                upk2(pp2[1], pp[2], pp[3]);
                const bool outp = (i >= 2 * R);
                float ov[4], cv[4], bv[4] = {1.f, 1.f, 1.f, 1.f}, sv[4], gv[4], pq[4];
                if (outp) {
                    const float *pl = reinterpret_cast<const float *>(sb + C::CUR_BYTES);
                    const float4 o4 = *reinterpret_cast<const float4 *>(pl + po);
                    const float4 c4 = *reinterpret_cast<const float4 *>(pl + TZ * BY + po);
                    ov[0] = o4.x; ov[1] = o4.y; ov[2] = o4.z; ov[3] = o4.w;
                    cv[0] = c4.x; cv[1] = c4.y; cv[2] = c4.z; cv[3] = c4.w;
                    int nxt = 2;
                    if (DAMP) {
                        const float4 b4 = *reinterpret_cast<const float4 *>(pl + 2 * TZ * BY + po);
                        bv[0] = b4.x; bv[1] = b4.y; bv[2] = b4.z; bv[3] = b4.w;
                        nxt = 3;
                    }
                    if (MODE == SF_MODE_GRAD) {
                        const float4 s4 = *reinterpret_cast<const float4 *>(pl + nxt * TZ * BY + po);
                        const float4 g4 = *reinterpret_cast<const float4 *>(pl + (nxt + 1) * TZ * BY + po);
                        sv[0] = s4.x; sv[1] = s4.y; sv[2] = s4.z; sv[3] = s4.w;
                        gv[0] = g4.x; gv[1] = g4.y; gv[2] = g4.z; gv[3] = g4.w;
                    }
                }
                // this warp is done with the stage: release it to the producer
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == S) {
                    st = 0;
                    ph ^= 1u;
                }
                // P ring (thread-private slots): read P_{p-R} (slot pw+1), write P_p (slot pw)
                int pr = pw + 1;
                if (pr == PR) pr = 0;
                if (outp) {
                    const float4 t = *reinterpret_cast<const float4 *>(myP + pr * (TZ * BY));
                    pq[0] = t.x; pq[1] = t.y; pq[2] = t.z; pq[3] = t.w;
                }
                *reinterpret_cast<float4 *>(myP + pw * (TZ * BY)) = make_float4(pp[0], pp[1], pp[2], pp[3]);
                pw = pr;
                // ---- finish output plane q = p - R from the register queue ----
                if (outp) {
                    const int sq = (s - R + Q) % Q;  // compile-time after unrolling
                    const int64_t q = qa + (i - 2 * R);
                    float res[4], gres[4];
#pragma unroll
                    for (int jp = 0; jp < 2; ++jp) {
                        const int j = 2 * jp;
                        const f2_t u = pk2(V[sq][j], V[sq][j + 1]);
                        f2_t X = 0ull;
#pragma unroll
                        for (int k = 1; k <= R; ++k) {
                            const int sm = (sq - k + Q) % Q, sp = (sq + k) % Q;
                            X = fma2(Wk[k], sf_xterm_x2(pk2(V[sm][j], V[sm][j + 1]), pk2(V[sp][j], V[sp][j + 1]), u, M2),
                                     X);
                        }
                        const f2_t lap = add2(pk2(pq[j], pq[j + 1]), X);
                        // out = u + beta (u - old) + c3 lap   (== sf_update per lane)
                        const f2_t d = fma2(M1, pk2(ov[j], ov[j + 1]), u);
                        const f2_t b2 = pk2(bv[j], bv[j + 1]), c2 = pk2(cv[j], cv[j + 1]);
                        const f2_t o = fma2(c2, lap, fma2(b2, d, u));
                        upk2(o, res[j], res[j + 1]);
                        if (MODE == SF_MODE_GRAD) {
                            // S = (beta - 1) d + c3 lap ; g -= gscale * snap * S   (== sf_d2 / sf_grad)
                            const f2_t S2 = fma2(add2(b2, M1), d, mul2(c2, lap));
                            const f2_t g2 = fma2(NG, mul2(pk2(sv[j], sv[j + 1]), S2), pk2(gv[j], gv[j + 1]));
                            upk2(g2, gres[j], gres[j + 1]);
                        }
                    }
                    if (cq == (int)q) {
                        // fused injection: res[j] += sum_e coef_e vals[pt_e]
                        // (the fp32 operations of k_inject, bitwise)
                        do {
                            const int lj = a.inj_lj[ci];
                            if ((lj >> 2) == lane) {
                                const int t = a.inj_t[ci];
                                float d = 0.f;
#pragma unroll 1
                                for (int e = a.inj_rowptr[t]; e < a.inj_rowptr[t + 1]; ++e)
                                    d = __fmaf_rn(a.inj_coef[e], a.inj_vals[a.inj_pt[e]], d);
                                const int j = lj & 3;
                                res[0] = (j == 0) ? __fadd_rn(res[0], d) : res[0];
                                res[1] = (j == 1) ? __fadd_rn(res[1], d) : res[1];
                                res[2] = (j == 2) ? __fadd_rn(res[2], d) : res[2];
                                res[3] = (j == 3) ? __fadd_rn(res[3], d) : res[3];
                                if (MODE == SF_MODE_GRAD) {
                                    gres[0] = (j == 0) ? __fmaf_rn(-a.gscale, __fmul_rn(sv[0], d), gres[0]) : gres[0];
                                    gres[1] = (j == 1) ? __fmaf_rn(-a.gscale, __fmul_rn(sv[1], d), gres[1]) : gres[1];
                                    gres[2] = (j == 2) ? __fmaf_rn(-a.gscale, __fmul_rn(sv[2], d), gres[2]) : gres[2];
                                    gres[3] = (j == 3) ? __fmaf_rn(-a.gscale, __fmul_rn(sv[3], d), gres[3]) : gres[3];
                                }
                            }
                            ++ci;
                            cq = ci < ce ? a.inj_q[ci] : QINF;
                        } while (cq == (int)q);
                    }
                    if (pq_ == (int)q) {
                        // fused interpolation of points owned by one lane
                        do {
                            if (a.itp_lane[pi] == lane) {
                                const int kc = a.itp_k[pi];
                                float acc = 0.f;
#pragma unroll 1
                                for (int c = 0; c < kc; ++c) {
                                    const int j = a.itp_j[4 * pi + c];
                                    const float v = j == 0 ? res[0] : j == 1 ? res[1] : j == 2 ? res[2] : res[3];
                                    acc = __fmaf_rn(a.itp_w[4 * pi + c], v, acc);
                                }
                                a.itp_out[a.itp_p[pi]] = acc;
                            }
                            ++pi;
                            pq_ = pi < pe ? a.itp_q[pi] : QINF;
                        } while (pq_ == (int)q);
                    }
                    if (active) {
                        const int64_t off = q * plane + rowoff;
                        stg4(a.out + off, make_float4(res[0], res[1], res[2], res[3]));
                        if (MODE == SF_MODE_SAVE)
                            stg4(a.snap_out + off, make_float4(res[0], res[1], res[2], res[3]));
                        if (MODE == SF_MODE_GRAD)
                            stg4(a.grad + off, make_float4(gres[0], gres[1], gres[2], gres[3]));
                    }
                }
            }
        }
    }

}

}  // namespace sftma
