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
    static constexpr int S_MAX = (220 * 1024) / STAGE_BYTES;
    static constexpr int S = S_MAX >= 4 ? 4 : S_MAX;      // pipeline depth
    static constexpr int SMEM = S * STAGE_BYTES + 128;    // + alignment slack
    static_assert(S >= 2, "stage does not fit shared memory");
};

template <int R, int BY, bool DAMP, int MODE>
__global__ void __launch_bounds__(32 * BY, 1)
k_tma3d(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_old,
        const __grid_constant__ CUtensorMap tm_c3, const __grid_constant__ CUtensorMap tm_beta,
        const __grid_constant__ CUtensorMap tm_snap, const __grid_constant__ CUtensorMap tm_grad,
        const SfStepArgs a, const int snap_slot, const int chunk)
{
    using C = Cfg<R, BY, DAMP, MODE>;
    constexpr int Q = C::Q, TZ = C::TZ, HZ = C::HZ, W = C::W, S = C::S;
    extern __shared__ unsigned char smem_raw[];
    unsigned char *smem = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    __shared__ __align__(8) uint64_t full[S];

    const int lane = threadIdx.x, wy = threadIdx.y, tid = wy * 32 + lane;
    const int z0 = blockIdx.x * TZ, y0 = blockIdx.y * BY;
    const int64_t qa = a.xa + (int64_t)blockIdx.z * chunk;
    const int64_t qb = min(qa + (int64_t)chunk, a.xb);
    if (qa >= qb) return;  // uniform over the CTA
    const int NP = (int)(qb - qa) + 2 * R;

    if (tid == 0) {
        prefetch_tmap(&tm_cur);
        prefetch_tmap(&tm_old);
#pragma unroll
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    // producer: plane p = qa - R + i, output plane q = p - R
    auto issue = [&](int i) {
        const int st = i % S;
        unsigned char *base = smem + st * C::STAGE_BYTES;
        const int64_t p = qa - R + i;
        const int64_t q = p - R;
        const bool outp = (q >= qa);
        uint32_t bytes = W * C::H * 4;  // full box, OOB part zero-filled
        if (outp) bytes += C::NPL * C::PL_BYTES;
        mbar_expect_tx(&full[st], bytes);
        tma_load3(base, &tm_cur, z0 - HZ, y0 - R, (int)p, &full[st]);
        if (outp) {
            unsigned char *pl = base + C::CUR_BYTES;
            tma_load3(pl, &tm_old, z0, y0, (int)q, &full[st]);
            pl += C::PL_BYTES;
            tma_load3(pl, &tm_c3, z0, y0, (int)q, &full[st]);
            pl += C::PL_BYTES;
            if (DAMP) {
                tma_load3(pl, &tm_beta, z0, y0, (int)q, &full[st]);
                pl += C::PL_BYTES;
            }
            if (MODE == SF_MODE_GRAD) {
                tma_load4(pl, &tm_snap, z0, y0, (int)q, snap_slot, &full[st]);
                pl += C::PL_BYTES;
                tma_load3(pl, &tm_grad, z0, y0, (int)q, &full[st]);
            }
        }
    };
    if (tid == 0) {
        for (int i = 0; i < S && i < NP; ++i) issue(i);
    }

    float V[Q][4];  // u at planes, slot = plane index mod Q (relative to qa - R)
    float P[Q][4];  // in-plane partial Laplacian, same slots
    const int rown = R + wy;
    const int zg = z0 + 4 * lane;
    const int yg = y0 + wy;
    const bool active = (zg < a.n2) && (yg < a.n1);
    const int64_t plane = a.n1 * a.n2;
    const int64_t rowoff = (int64_t)yg * a.n2 + zg;

    for (int base = 0; base < NP; base += Q) {
#pragma unroll
        for (int s = 0; s < Q; ++s) {
            const int i = base + s;
            if (i < NP) {
                const int st = i % S;
                mbar_wait(&full[st], (uint32_t)((i / S) & 1));
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
                float pp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int k = 1; k <= R; ++k) {
                    const float4 ym = *reinterpret_cast<const float4 *>(cs + (rown - k) * W + HZ + 4 * lane);
                    const float4 yp = *reinterpret_cast<const float4 *>(cs + (rown + k) * W + HZ + 4 * lane);
                    const float ymv[4] = {ym.x, ym.y, ym.z, ym.w};
                    const float ypv[4] = {yp.x, yp.y, yp.z, yp.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        pp[j] = __fmaf_rn(a.w.w[k],
                                          sf_inplane3(ymv[j], ypv[j], zr[HZ + j - k], zr[HZ + j + k],
                                                      zr[HZ + j]),
                                          pp[j]);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) P[s][j] = pp[j];

                if (i >= 2 * R) {
                    const int sq = (s - R + Q) % Q;  // compile-time after unrolling
                    const int64_t q = qa + (i - 2 * R);
                    const float *pl = reinterpret_cast<const float *>(sb + C::CUR_BYTES);
                    const int po = wy * TZ + 4 * lane;
                    const float4 o4 = *reinterpret_cast<const float4 *>(pl + po);
                    const float4 c4 = *reinterpret_cast<const float4 *>(pl + TZ * BY + po);
                    float4 b4 = make_float4(1.f, 1.f, 1.f, 1.f);
                    int nxt = 2;
                    if (DAMP) {
                        b4 = *reinterpret_cast<const float4 *>(pl + 2 * TZ * BY + po);
                        nxt = 3;
                    }
                    const float ov[4] = {o4.x, o4.y, o4.z, o4.w};
                    const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
                    const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
                    float res[4], gres[4];
                    float sv[4] = {0.f, 0.f, 0.f, 0.f}, gv[4] = {0.f, 0.f, 0.f, 0.f};
                    if (MODE == SF_MODE_GRAD) {
                        const float4 s4 = *reinterpret_cast<const float4 *>(pl + nxt * TZ * BY + po);
                        const float4 g4 = *reinterpret_cast<const float4 *>(pl + (nxt + 1) * TZ * BY + po);
                        sv[0] = s4.x; sv[1] = s4.y; sv[2] = s4.z; sv[3] = s4.w;
                        gv[0] = g4.x; gv[1] = g4.y; gv[2] = g4.z; gv[3] = g4.w;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float u = V[sq][j];
                        float X = 0.f;
#pragma unroll
                        for (int k = 1; k <= R; ++k)
                            X = __fmaf_rn(a.w.w[k], sf_xterm(V[(sq - k + Q) % Q][j], V[(sq + k) % Q][j], u), X);
                        const float lap = __fadd_rn(P[sq][j], X);
                        res[j] = sf_update(u, ov[j], bv[j], cv[j], lap);
                        if (MODE == SF_MODE_GRAD)
                            gres[j] = sf_grad(gv[j], a.gscale, sv[j], sf_d2(u, ov[j], bv[j], cv[j], lap));
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
                __syncthreads();
                if (tid == 0 && i + S < NP) issue(i + S);
            }
        }
    }
}

}  // namespace sftma
