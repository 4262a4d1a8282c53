// stencil_tb2.cuh -- temporal blocking: TWO time steps per HBM pass, r <= 4,
// 3D, plain forward steps (SF_OPT_TBLOCK).
//
// The paper's DLE loop blocking and its runtime block-size tuning are cache
// blocking of one step; the GPU analogue that can beat the single-step HBM roofline is
// blocking in TIME: u^{n+1} and u^{n+2} are both formed from one read of u^{n-1}, u^n, c3
// (and beta), so the compulsory traffic falls from 20 B to 24 B per TWO point updates
// (12 B/update; 10 B without the beta array).  The price is redundant work: step 2 at a
// point needs step 1 on a radius-r neighbourhood, so each CTA computes step 1 on its tile
// grown by r rows (y) and 4 columns (z) on each side -- (8 + 2r) x 128 step-1 points for
// 8 x 120 step-2 points, 1.42x the step-1 work at r = 4 -- and re-streams 4r warm-up planes
// per x-chunk instead of 2r.
//
// Per CTA (8 warps, no producer warp: thread 0 issues the TMA loads after the block barrier
// that frees their slot), per plane p of u^n along x (the streamed axis):
//   * TMA: u^n plane p with a (2r, 8)-deep (y, z) halo into a (r + 2)-deep ring (zero OOB
//     fill = the zero ghost halo, reading C6); old u^{n-1}, c3 (, beta) of step-1 plane
//     q1 = p - r over the grown tile into a 2-3 stage ring;
//   * step 1 at q1 (grown tile; warp w owns rows w + r and, for w < 2r, one halo row; 4
//     columns per lane): the per-point arithmetic of every other variant (stencil_common.cuh,
//     fp32x2), x term from a (2r+1)-deep register queue, source injection of step n by the
//     owning lane; the result goes to a (2r+2)-deep shared ring of step-1 planes and -- the
//     tile's own rows and columns -- to u^{n+1} in HBM;
//   * block barrier;
//   * step 2 at q2 = p - 2r (own tile rows): neighbours from the step-1 ring, old = u^n from
//     the register queue, c3 / beta re-read through L2, injection of step n + 1, store u^{n+2}.
// Out-of-grid step-1 points come out as +0 by themselves (u, old, c3, beta all zero-filled),
// which is the zero ghost halo step 2 must see.  Every value is formed by the same operations
// in the same order as the single-step kernels: bitwise equal to two single steps
// (tests/test_gpu_parity.py::test_tblock_bitwise).  The outputs go to two other buffers (the
// neighbours' grown tiles still read u^{n-1} and u^n): the host rotates four buffers.
#pragma once
#include "launch.cuh"
#include "stencil_tma.cuh"


namespace sftb {

constexpr int TY = 8;      // step-2 rows per tile (one per warp)
constexpr int TZ = 120;    // step-2 columns per tile (lanes 1..30)
constexpr int EZ = 128;    // step-1 columns (32 lanes x 4)
constexpr int MZ = 4;      // z margin of the grown tile (>= r, keeps 16-byte alignment)

template <int R, bool DAMP>
struct TbCfg {
    static_assert(R >= 1 && R <= 4, "two-step kernel: r <= 4");
    static constexpr int EY = TY + 2 * R;           // step-1 rows
    static constexpr int UH = EY + 2 * R;           // u^n box rows
    static constexpr int UW = EZ + 2 * MZ;          // u^n box columns
    static constexpr int Q = 2 * R + 1;             // register queue depth
    static constexpr int L = 2;                     // TMA lead of the u ring (planes)
    static constexpr int DU = R + L;                // u ring: planes q1 .. p + L - 1
    static constexpr int UST = ((UW * UH * 4 + 127) / 128) * 128;
    static constexpr int PL = EZ * EY * 4;          // one grown-tile plane
    static constexpr int NPL = DAMP ? 3 : 2;
    static constexpr int CST = NPL * PL;
    static constexpr int DV = 2 * R + 2;            // step-1 ring (2r + 1 read, 1 being written)
    static constexpr int BUDGET = 226 * 1024;
    static constexpr int DC = (DU * UST + 3 * CST + DV * PL <= BUDGET) ? 3 : 2;
    static constexpr int SMEM = DU * UST + DC * CST + DV * PL + 128;
    static_assert(DU * UST + DC * CST + DV * PL <= BUDGET, "two-step kernel does not fit shared memory");
};

template <int R, bool DAMP>
__global__ void __launch_bounds__(256, 1)
k_tb2(const __grid_constant__ CUtensorMap tm_cur, const __grid_constant__ CUtensorMap tm_old,
      const __grid_constant__ CUtensorMap tm_c3, const __grid_constant__ CUtensorMap tm_beta, const TbArgs a)
{
    using namespace sftma;
    using C = TbCfg<R, DAMP>;
    constexpr int UW = C::UW, Q = C::Q, DU = C::DU, DC = C::DC, DV = C::DV, L = C::L;
    constexpr int UF = C::UST / 4, CF = C::CST / 4, PF = C::PL / 4;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char *smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    float *uring = reinterpret_cast<float *>(smem);
    float *cring = uring + DU * UF;
    float *vring = cring + DC * CF;
    __shared__ __align__(8) uint64_t bars[DU + DC];
    const uint32_t ufull = smem_u32(bars), cfull = ufull + 8 * DU;

    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int ntz = (a.n2 + TZ - 1) / TZ, tiles = ntz * ((a.n1 + TY - 1) / TY);
    const int items = tiles * a.nchunk;
    if ((int)blockIdx.x >= items) return;
    if (threadIdx.x == 0) {
        for (int s = 0; s < DU; ++s) mbar_init(ufull + 8 * s, 1);
        for (int s = 0; s < DC; ++s) mbar_init(cfull + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        prefetch_tmap(&tm_cur);
        prefetch_tmap(&tm_old);
        prefetch_tmap(&tm_c3);
        if (DAMP) prefetch_tmap(&tm_beta);
    }
    __syncthreads();

    // own rows of the grown tile: eA = wq + R (tile row wq), eB = a halo row for wq < 2R
    const int eA = wq + R;
    const bool has2 = wq < 2 * R;
    const int eB = wq < R ? wq : wq + TY;   // (unused when !has2)
    const bool ctr = lane >= 1 && lane <= 30;  // step-2 lanes (tile columns)
    f2_t Wk[R + 1];
#pragma unroll
    for (int k = 1; k <= R; ++k) Wk[k] = pk2(a.w.w[k], a.w.w[k]);
    Wk[0] = 0ull;
    const f2_t M4 = pk2(-4.f, -4.f), M2 = pk2(-2.f, -2.f), M1 = pk2(-1.f, -1.f), ONE2 = pk2(1.f, 1.f);
    const f2_t M6 = pk2(-6.f, -6.f);
    constexpr bool MRG = sf_merged_form(R, SF_MODE_PLAIN);  // as the single-step forward
    const int64_t plane = (int64_t)a.n1 * a.n2;
    const uint32_t ub = smem_u32(uring), cb = smem_u32(cring);
    f2_t V[Q][2][2];   // own u^n values (rows eA, eB; 2 pairs) at the last Q planes
    uint32_t gu = 0, gc = 0;  // ring uses before the current item

    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int tile = it % tiles, ck = it / tiles;
        const int qa = ck * a.chunk, qb = min(a.n0, qa + a.chunk);
        const int z0 = (tile % ntz) * TZ, y0 = (tile / ntz) * TY;
        const int NP = qb - qa + 4 * R, p0 = qa - 2 * R;
        auto issue_u = [&](int i) {
            const uint32_t g = gu + i, s = g % DU;
            mbar_expect_tx(ufull + 8 * s, UW * C::UH * 4);
            tma_load3(ub + s * C::UST, &tm_cur, z0 - 2 * MZ, y0 - 2 * R, p0 + i, ufull + 8 * s);
        };
        auto issue_c = [&](int i) {  // step-1 plane of iteration i (>= 2R)
            const uint32_t g = gc + (i - 2 * R), s = g % DC;
            const int q1 = p0 + i - R;
            mbar_expect_tx(cfull + 8 * s, C::CST);
            uint32_t d = cb + s * C::CST;
            tma_load3(d, &tm_old, z0 - MZ, y0 - R, q1, cfull + 8 * s);
            tma_load3(d + C::PL, &tm_c3, z0 - MZ, y0 - R, q1, cfull + 8 * s);
            if (DAMP) tma_load3(d + 2 * C::PL, &tm_beta, z0 - MZ, y0 - R, q1, cfull + 8 * s);
        };
        // the previous item's reads of every ring slot are done before the refills
        fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 0; i < L && i < NP; ++i) issue_u(i);
            for (int i = 2 * R; i < NP && i < 2 * R + DC; ++i) issue_c(i);
        }
        // own positions
        const int zA = z0 - MZ + 4 * lane;               // first own column (grid)
        const int yA = y0 + wq;                          // tile row (grid) of eA
        const bool st_ok = ctr && zA < a.n2 && yA < a.n1;  // owns stored tile points
        float *o1p = a.o1 + (int64_t)yA * a.n2 + zA;
        float *o2p = a.o2 + (int64_t)yA * a.n2 + zA;
        const float *c3p = a.c3 + (int64_t)yA * a.n2 + zA;
        const float *bep = DAMP ? a.beta + (int64_t)yA * a.n2 + zA : nullptr;
        // injection cursors (CTA-uniform): first entries at planes >= qa - R (step 1), >= qa (step 2)
        int c1 = 0, c2 = 0, ce = 0;
        if (a.beg) {
            c1 = a.beg[tile];
            ce = a.beg[tile + 1];
            while (c1 < ce && a.e_q[c1] < qa - R) ++c1;
            c2 = c1;
            while (c2 < ce && a.e_q[c2] < qa) ++c2;
        }

#pragma unroll 1
        for (int base = 0; base < NP; base += Q) {
#pragma unroll
            for (int s2 = 0; s2 < Q; ++s2) {
                const int i = base + s2;
                if (i >= NP) break;
                const int p = p0 + i, q1 = p - R, q2 = p - 2 * R;
                const bool st1 = i >= 2 * R, st2 = i >= 4 * R;
                // step 2's c3 / beta (tile row, 4 columns) through L2, issued early
                f2_t c3v[2], bev[2];
                if (st2 && st_ok) {
                    ldp<4>(c3p + (int64_t)q2 * plane, c3v);
                    if (DAMP) ldp<4>(bep + (int64_t)q2 * plane, bev);
                }
                // ---- plane p of u^n into queue slot s2
                {
                    const uint32_t g = gu + i;
                    mbar_wait(ufull + 8 * (g % DU), (g / DU) & 1u);
                    const float *ut = uring + (g % DU) * UF;
                    ldp<4>(ut + (eA + R) * UW + MZ + 4 * lane, V[s2][0]);
                    if (has2) ldp<4>(ut + (eB + R) * UW + MZ + 4 * lane, V[s2][1]);
                }
                // ---- step 1 at q1 (grown tile)
                if (st1) {
                    const uint32_t gq = gu + i - R;  // u slot of plane q1
                    const float *uq = uring + (gq % DU) * UF;
                    const uint32_t gcs = gc + (i - 2 * R);
                    mbar_wait(cfull + 8 * (gcs % DC), (gcs / DC) & 1u);
                    const float *cp = cring + (gcs % DC) * CF;
                    const int SQ = (s2 - R + Q) % Q;  // queue slot of q1 (folds: the loop is unrolled)
                    f2_t res[2][2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        if (j == 1 && !has2) break;
                        const int e = j ? eB : eA;
                        const float *row = uq + (e + R) * UW + MZ + 4 * lane;  // own 4 values of q1
                        f2_t Y[2 * R + 1][2];
#pragma unroll
                        for (int t = 0; t <= 2 * R; ++t) ldp<4>(row + (t - R) * UW, Y[t]);
                        f2_t ZL[2], ZR[2];
                        ldp<4>(row - 4, ZL);
                        ldp<4>(row + 4, ZR);
                        auto F = [&](int o) -> float {  // float at z offset o of the own row
                            const f2_t v = o < 0 ? ZL[(o + 4) >> 1] : o >= 4 ? ZR[(o - 4) >> 1] : Y[R][o >> 1];
                            return (o & 1) ? hi2(v) : lo2(v);
                        };
                        auto PZ = [&](int o) -> f2_t {  // aligned pair at even offset o
                            return o < 0 ? ZL[(o + 4) >> 1] : o >= 4 ? ZR[(o - 4) >> 1] : Y[R][o >> 1];
                        };
                        const float *co = cp + e * EZ + 4 * lane;
                        f2_t ov[2], cv[2], bv[2];
                        ldp<4>(co, ov);
                        ldp<4>(co + PF, cv);
                        if (DAMP) ldp<4>(co + 2 * PF, bv);
                        else bv[0] = bv[1] = ONE2;
#pragma unroll
                        for (int jp = 0; jp < 2; ++jp) {
                            const f2_t u = V[SQ][j][jp];
                            f2_t P = 0ull;
#pragma unroll
                            for (int k = 1; k <= R; ++k) {
                                const f2_t ys = add2(Y[R - k][jp], Y[R + k][jp]);
                                const int em = 2 * jp - k, ep = 2 * jp + k;
                                f2_t zs;
                                if (k & 1) zs = pk2(__fadd_rn(F(em), F(ep)), __fadd_rn(F(em + 1), F(ep + 1)));
                                else zs = add2(PZ(em), PZ(ep));
                                if constexpr (MRG)  // merged form (== sf_merged3 per lane)
                                    P = fma2(Wk[k], fma2(M6, u, add2(add2(ys, zs), add2(V[(SQ - k + Q) % Q][j][jp], V[(SQ + k) % Q][j][jp]))), P);
                                else
                                    P = fma2(Wk[k], fma2(M4, u, add2(ys, zs)), P);
                            }
                            f2_t X = 0ull;
                            if constexpr (!MRG) {
#pragma unroll
                                for (int k = 1; k <= R; ++k)
                                    X = fma2(Wk[k], sf_xterm_x2(V[(SQ - k + Q) % Q][j][jp], V[(SQ + k) % Q][j][jp], u, M2), X);
                            }
                            const f2_t lap = MRG ? P : add2(P, X);
                            const f2_t d = fma2(M1, ov[jp], u);
                            res[j][jp] = fma2(cv[jp], lap, fma2(bv[jp], d, u));
                        }
                    }
                    // injection of step n (the fp32 operations of k_inject)
                    if (a.vals1) {
                        while (c1 < ce && a.e_q[c1] == q1) {
                            const int ep = a.e_p[c1], ey = ep >> 7, ec = ep & 127;
                            if (ec >> 2 == lane && (ey == eA || (has2 && ey == eB))) {
                                const int t = a.e_t[c1];
                                float dd = 0.f;
                                for (int e = a.rowptr[t]; e < a.rowptr[t + 1]; ++e)
                                    dd = __fmaf_rn(a.coef[e], a.vals1[a.pt[e]], dd);
                                const int j = ey == eA ? 0 : 1, jj = ec & 3;
#pragma unroll
                                for (int j2 = 0; j2 < 2; ++j2)
#pragma unroll
                                    for (int jp = 0; jp < 2; ++jp) {
                                        float lo, hi;
                                        upk2(res[j2][jp], lo, hi);
                                        if (j2 == j && jj == 2 * jp) lo = __fadd_rn(lo, dd);
                                        if (j2 == j && jj == 2 * jp + 1) hi = __fadd_rn(hi, dd);
                                        res[j2][jp] = pk2(lo, hi);
                                    }
                            }
                            ++c1;
                        }
                    }
                    float *vs = vring + (i % DV) * PF + 4 * lane;
                    stp<4>(vs + eA * EZ, res[0]);
                    if (has2) stp<4>(vs + eB * EZ, res[1]);
                    if (st_ok && q1 >= qa && q1 < qb) stp<4>(o1p + (int64_t)q1 * plane, res[0]);
                }
                // the ring slots read above may be refilled; step 1 of q1 is visible to all
                fence_proxy_async_smem();
                __syncthreads();
                if (threadIdx.x == 0) {
                    if (i + L < NP) issue_u(i + L);
                    if (st1 && i + DC < NP) issue_c(i + DC);
                }
                // ---- step 2 at q2 (tile rows), neighbours from the step-1 ring
                if (st2 && ctr) {
                    const float *vq = vring + ((i - R) % DV) * PF + eA * EZ + 4 * lane;  // step 1 of q2
                    f2_t Y[2 * R + 1][2];
#pragma unroll
                    for (int t = 0; t <= 2 * R; ++t) ldp<4>(vq + (t - R) * EZ, Y[t]);
                    f2_t ZL[2], ZR[2];
                    ldp<4>(vq - 4, ZL);
                    ldp<4>(vq + 4, ZR);
                    auto F = [&](int o) -> float {
                        const f2_t v = o < 0 ? ZL[(o + 4) >> 1] : o >= 4 ? ZR[(o - 4) >> 1] : Y[R][o >> 1];
                        return (o & 1) ? hi2(v) : lo2(v);
                    };
                    auto PZ = [&](int o) -> f2_t {
                        return o < 0 ? ZL[(o + 4) >> 1] : o >= 4 ? ZR[(o - 4) >> 1] : Y[R][o >> 1];
                    };
                    f2_t XM[R + 1][2], XP[R + 1][2];
#pragma unroll
                    for (int k = 1; k <= R; ++k) {
                        ldp<4>(vring + ((i - R - k) % DV) * PF + eA * EZ + 4 * lane, XM[k]);
                        ldp<4>(vring + ((i - R + k) % DV) * PF + eA * EZ + 4 * lane, XP[k]);
                    }
                    const int SO = (s2 + 1) % Q;  // queue slot of q2 = p - 2R: u^n, step 2's old
                    f2_t res[2];
#pragma unroll
                    for (int jp = 0; jp < 2; ++jp) {
                        const f2_t u = Y[R][jp];
                        f2_t P = 0ull;
#pragma unroll
                        for (int k = 1; k <= R; ++k) {
                            const f2_t ys = add2(Y[R - k][jp], Y[R + k][jp]);
                            const int em = 2 * jp - k, ep = 2 * jp + k;
                            f2_t zs;
                            if (k & 1) zs = pk2(__fadd_rn(F(em), F(ep)), __fadd_rn(F(em + 1), F(ep + 1)));
                            else zs = add2(PZ(em), PZ(ep));
                            if constexpr (MRG)
                                P = fma2(Wk[k], fma2(M6, u, add2(add2(ys, zs), add2(XM[k][jp], XP[k][jp]))), P);
                            else
                                P = fma2(Wk[k], fma2(M4, u, add2(ys, zs)), P);
                        }
                        f2_t X = 0ull;
                        if constexpr (!MRG) {
#pragma unroll
                            for (int k = 1; k <= R; ++k) X = fma2(Wk[k], sf_xterm_x2(XM[k][jp], XP[k][jp], u, M2), X);
                        }
                        const f2_t lap = MRG ? P : add2(P, X);
                        const f2_t d = fma2(M1, V[SO][0][jp], u);
                        const f2_t bb = DAMP ? bev[jp] : ONE2;
                        res[jp] = fma2(c3v[jp], lap, fma2(bb, d, u));
                    }
                    if (a.vals2) {
                        while (c2 < ce && a.e_q[c2] == q2) {
                            const int ep = a.e_p[c2], ey = ep >> 7, ec = ep & 127;
                            if (ec >> 2 == lane && ey == eA) {
                                const int t = a.e_t[c2];
                                float dd = 0.f;
                                for (int e = a.rowptr[t]; e < a.rowptr[t + 1]; ++e)
                                    dd = __fmaf_rn(a.coef[e], a.vals2[a.pt[e]], dd);
                                const int jj = ec & 3;
#pragma unroll
                                for (int jp = 0; jp < 2; ++jp) {
                                    float lo, hi;
                                    upk2(res[jp], lo, hi);
                                    if (jj == 2 * jp) lo = __fadd_rn(lo, dd);
                                    if (jj == 2 * jp + 1) hi = __fadd_rn(hi, dd);
                                    res[jp] = pk2(lo, hi);
                                }
                            }
                            ++c2;
                        }
                    }
                    if (st_ok) stp<4>(o2p + (int64_t)q2 * plane, res);
                } else if (st2 && a.vals2) {
                    while (c2 < ce && a.e_q[c2] == q2) ++c2;  // keep the cursor in step
                }
            }
        }
        gu += NP;
        gc += NP - 2 * R;
    }
}

}  // namespace sftb
