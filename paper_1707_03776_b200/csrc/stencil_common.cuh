// stencil_common.cuh -- per-point arithmetic shared by every stencil kernel variant.
//
// One fixed evaluation order for every variant (generic thread-per-point, TMA 2.5D
// streaming, slab boundary/interior launches), so that all variants -- and the
// multi-GPU slab run vs the 1-GPU run -- produce identical bits (reading C18).
//
// Laplacian in the per-radius difference form (reading C15):
//   P  = sum_{k=1..r} w_k * ( ((y_-k + y_+k) + (z_-k + z_+k)) - 4 u )   (3D; 2D: (z_-k + z_+k) - 2u)
//   X  = sum_{k=1..r} w_k * ( (x_-k + x_+k) - 2 u )
//   Lap = P + X,  w_k = fp32(w_k^exact / h^2)
// so that a constant field is annihilated exactly (4u and 2u are exact) and the fp32
// weights never need to sum to zero.  3D, r >= 5, outside the gradient's GRAD mode: the
// MERGED form (sf_merged3 below) -- one chain over the three axes per radius,
//   L  = sum_{k=1..r} w_k * fma(-6, u, ((y_-k + y_+k) + (z_-k + z_+k)) + (x_-k + x_+k))
// 7 instead of 8 FP operations per radius (the kernel is FP-issue bound at high order:
// configs[4] -7 %), still exact on a constant field: the FMA forms 6u exactly inside.  (At
// r = 4 it gained 1 % under the power cap but doubled the configs[2] full-size gradient error,
// 3.8e-5 -> 7.0e-5: SF_MERGED_RMIN stays 5.)  (An
// earlier chain that subtracted a separately rounded fl(6u) doubled the fp32 error --
// configs[2] gradient 1.9e-4 vs 3.8e-5; the gradient's in-kernel
// S = out - 2u + old is the most sensitive use of L, so GRAD mode keeps the per-axis form.)
// Update (the
// paper's solve(), with a
// centred u.dt, reading C1), beta/c3 hoisted per point at setup:
//   out = u + beta (u - old) + c3 * Lap
// Gradient term formed in-register (reading C13/C14; north_star "g += v u_tt"):
//   S = out - 2u + old (before injection) = (beta - 1)(u - old) + c3 * Lap
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define SF_MAXR 8

struct SfWeights {
    float w[SF_MAXR + 1];   // w[k], k = 1..r, already divided by h^2 (w[0] unused)
};

enum SfMode { SF_MODE_PLAIN = 0, SF_MODE_SAVE = 1, SF_MODE_GRAD = 2 };
// damping representation: none (beta = 1), hoisted beta array, separable profiles
enum SfDampMode { SF_DAMP_NONE = 0, SF_DAMP_ARRAY = 1, SF_DAMP_SEP = 2 };

// Programmatic dependent launch (SF_OPT_PDL): a kernel launched with the programmatic-
// serialisation attribute may start while the previous kernel of the stream drains; it waits
// here, before its first global-memory access, until that kernel has completed and its
// writes are visible.  A no-op when the kernel was launched without the attribute.
__device__ __forceinline__ void sf_pdl_wait()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// in-plane term at radius k for 3D: ((ym + yp) + (zm + zp)) - 4u, as one fma
__device__ __forceinline__ float sf_inplane3(float ym, float yp, float zm, float zp, float u)
{
    float s = __fadd_rn(__fadd_rn(ym, yp), __fadd_rn(zm, zp));
    return __fmaf_rn(-4.0f, u, s);
}

// in-plane term at radius k for 2D (only z in-plane): (zm + zp) - 2u
__device__ __forceinline__ float sf_inplane2(float zm, float zp, float u)
{
    return __fmaf_rn(-2.0f, u, __fadd_rn(zm, zp));
}

// Merged form (SF_MERGED): t_k = (((y-k + y+k) + (z-k + z+k)) + (x-k + x+k)) - 6u, one FMA with
// the exact product 6u (no separately rounded fl(6u)), L = sum_k w_k t_k: 7 instead of 8 FP
// operations per radius, still exact on a constant field.
#ifndef SF_MERGED
#define SF_MERGED 1
#endif
#ifndef SF_MERGED_GRAD
#define SF_MERGED_GRAD 0
#endif
#ifndef SF_MERGED_RMIN
#define SF_MERGED_RMIN 5
#endif
__host__ __device__ constexpr bool sf_merged_form(int r, int mode)
{
    return SF_MERGED && r >= SF_MERGED_RMIN && (SF_MERGED_GRAD || mode != SF_MODE_GRAD);
}
__device__ __forceinline__ float sf_merged3(float ym, float yp, float zm, float zp, float xm, float xp, float u)
{
    float s = __fadd_rn(__fadd_rn(__fadd_rn(ym, yp), __fadd_rn(zm, zp)), __fadd_rn(xm, xp));
    return __fmaf_rn(-6.0f, u, s);
}

// x term at radius k: (xm + xp) - 2u
__device__ __forceinline__ float sf_xterm(float xm, float xp, float u)
{
    return __fmaf_rn(-2.0f, u, __fadd_rn(xm, xp));
}

// out = u + beta (u - old) + c3 * lap
__device__ __forceinline__ float sf_update(float u, float old, float beta, float c3, float lap)
{
    float d = __fsub_rn(u, old);
    float o = __fmaf_rn(beta, d, u);
    return __fmaf_rn(c3, lap, o);
}

// S = (beta - 1)(u - old) + c3 * lap
__device__ __forceinline__ float sf_d2(float u, float old, float beta, float c3, float lap)
{
    float d = __fsub_rn(u, old);
    return __fmaf_rn(__fsub_rn(beta, 1.0f), d, __fmul_rn(c3, lap));
}

// grad -= gscale * snap * S
__device__ __forceinline__ float sf_grad(float g, float gscale, float snap, float S)
{
    return __fmaf_rn(-gscale, __fmul_rn(snap, S), g);
}

// ---- packed fp32x2 forms (sm_100a FADD2 / FFMA2 / FMUL2): two lanes of exactly the
// scalar IEEE round-to-nearest operations above, so results are bitwise identical to
// the scalar path while the FP issue count halves.
typedef unsigned long long f2_t;

__device__ __forceinline__ f2_t pk2(float lo, float hi)
{
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk2(f2_t v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b)
{
    f2_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b)
{
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c)
{
    f2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// ((ym + yp) + (zm + zp)) - 4u  (== sf_inplane3 per lane)
__device__ __forceinline__ f2_t sf_inplane3_x2(f2_t ym, f2_t yp, f2_t zm, f2_t zp, f2_t u, f2_t m4)
{
    return fma2(m4, u, add2(add2(ym, yp), add2(zm, zp)));
}
// (xm + xp) - 2u  (== sf_xterm per lane)
__device__ __forceinline__ f2_t sf_xterm_x2(f2_t xm, f2_t xp, f2_t u, f2_t m2)
{
    return fma2(m2, u, add2(xm, xp));
}

// beta regenerated from separable damping profiles (sf_desc.sigma, reading C7):
//   s = ((sx + sy) + sz) * (dt/2),  beta = (1 - s) * rcp(1 + s)
// rcp.approx.ftz (one MUFU op, rel. error < 2^-22) instead of an IEEE division; every
// variant uses this one function (or its lane-wise identical fp32x2 form), so they agree
// bitwise.  The argument 1 + s lies in [1, 2) (s = sigma dt/2 < 1 for any stable damping),
// so flush-to-zero never applies (the non-ftz form adds seven range-fixup instructions).
__device__ __forceinline__ float sf_rcp(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sf_beta_sep(float sx, float sy, float sz, float hdt)
{
    const float s = __fmul_rn(__fadd_rn(__fadd_rn(sx, sy), sz), hdt);
    return __fmul_rn(__fsub_rn(1.0f, s), sf_rcp(__fadd_rn(1.0f, s)));
}

// byte offset of a peer-store mirror (SfStepArgs::md): the same element in the neighbour's buffer
__device__ __forceinline__ float *sf_mirror(float *p, int64_t db)
{
    return reinterpret_cast<float *>(reinterpret_cast<char *>(p) + db);
}

// Kernel parameter block shared by all stencil variants.
struct SfStepArgs {
    const float *cur;      // u^n (read, with neighbours)
    float *out;            // old level on input (u^{n-1}), new level on output (in place)
    const float *c3;       // hoisted dt^2 / A
    const float *beta;     // hoisted (m - eta dt/2) / A, or NULL (== 1, or separable below)
    const float *sigx, *sigy, *sigz;  // separable damping profiles of the buffer (or NULL)
    float hdt;             // dt / 2 (fp32) for sf_beta_sep
    float *snap_out;       // SAVE: snapshot slot to write (== out values), else NULL
    const float *snap_in;  // GRAD: u^n snapshot slot
    int snap_half;         // snapshots stored as fp16 (SF_OPT_SNAP_HALF): snap_out / snap_in
                           // then point to __half data (element offsets unchanged)
    float *grad;           // GRAD: gradient accumulator
    float gscale;          // GRAD: k / dt^2
    int64_t n0b, n1, n2;   // buffer extents (n0b includes slab halo planes)
    int64_t xa, xb;        // planes [xa, xb) of the buffer to compute
    int64_t xa2, xb2;      // optional second range [xa2, xb2) in the same launch (xa2 == xb2: none)
    int64_t zbase, n2t;    // TMA kernel: its tiles cover the columns [zbase, n2t) (0, n2: all)
    SfWeights w;
    // Peer-store halo exchange (SF_OPT_P2P): an output plane q in [mq[0], mq[1])
    // is also stored at byte offset md[0] from its own address (the left neighbour's right
    // halo, a peer-mapped pointer), q in [mq[2], mq[3]) at md[1] (the right neighbour's
    // left halo).  Empty ranges: no mirror.
    int64_t mq[4];
    int64_t md[2];
    int l2_prefetch;       // TMA kernel: L2 prefetch distance in planes (0 = off)
    // Fused injection of small point sets in the TMA kernel (NULL inj_beg = none).  Lists
    // are per (tile, consumer warp): entries [beg[tile * NW + w], beg[tile * NW + w + 1])
    // sorted by output plane q; every entry is owned by one lane, which applies it to its
    // registers before the store: inj_q, inj_lj ((row * 32 + lane) * 4 + z),
    // inj_t (row of the CSR inj_rowptr / inj_pt / inj_coef, values inj_vals[pt]) ->
    // out[t] += sum coef vals.  (Records are interpolated by a separate kernel.)
    const int *inj_beg, *inj_q, *inj_lj, *inj_t, *inj_rowptr, *inj_pt;
    const float *inj_coef, *inj_vals;
    // One-launch slab schedule (TMA kernel): bidir = 1 streams the LAST x-chunk of every tile
    // downward (from xb - 1), so that both boundary ranges [xa, xa + r) and [xb - r, xb) are
    // finished r output planes into the launch; sig != NULL: after a CTA has stored all of a
    // boundary range of its tile, it fences and adds 1 to sig[0] (left) / sig[1] (right), so
    // that a stream waiting on the counter (cuStreamWaitValue32) can start the halo exchange
    // while the same launch computes the interior.
    int bidir;
    unsigned int *sig;
};
