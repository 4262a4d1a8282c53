/*
 * sf.h -- C-ABI of the B200-native acoustic finite-difference propagator (libsf.so).
 *
 * The hot path of the seismic example of Lange et al., "Optimised finite difference
 * computation from symbolic equations" (Devito, SciPy 2017; PAPER.md = the paper's
 * text, cited P:line):
 *
 *   forward:  m u_tt - Lap u + eta u_t = q
 *            u.forward = solve(m*u.dt2 - u.laplace + eta*u.dt, u.forward)
 *            src.inject(field=u, expr=src*dt**2/m)
 *            rec.interpolate(expr=u)
 *   adjoint:  same stencil run backwards in time (time_axis=Backward),
 *            eta sign flipped, receivers injected, sources interpolated.
 *   gradient (BASELINE north_star, not in the paper): g += v * u_tt correlation of
 *            the adjoint wavefield with saved / subsampled forward wavefields.
 *
 * Discretisation (DESIGN.md §3 readings C1-C20):
 *   A = m + eta dt/2, beta = (m - eta dt/2)/A, c3 = dt^2/A,
 *   out = cur + beta (cur - old) + c3 * L_h cur,  L_h = centred order-`space_order`
 *   Laplacian with a zero ghost halo (C6); forward (cur, old) = (u^n, u^{n-1}) -> u^{n+1},
 *   adjoint (cur, old) = (v^n, v^{n+1}) -> v^{n-1}.  Injection after the stencil into the
 *   new level with scale dt^2/m (C3, C9); records sample the level just completed (C4).
 *   Gradient: g -= k * u^n * (v^{n+1} - 2 v^n + v^{n-1}) / dt^2 for n % k == 0 (C13, C14).
 *
 * Conventions for every call:
 *   - Grid arrays: device-resident, caller-owned, contiguous fp32, row-major
 *     [n0][n1][n2] = [x][y][z] (2D: [x][z]), last axis fastest, exactly N points.
 *   - Sparse time series: device fp32, time-major [nt][npoint] (C12).
 *   - Coordinates: HOST fp64 [npoint][ndim], metres from computational index 0;
 *     a point outside [0, (n-1) h] on any axis is SF_ERR_OUT_OF_DOMAIN (never clipped).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); every call is
 *     ordered on it and returns without synchronising unless stated.
 *   - Ownership: the library never frees caller memory.  A handle owns its setup
 *     tables and its coefficient arrays (beta, c3: 1-2 x N floats), allocated from the
 *     device's stream-ordered memory pool (retained for reuse) and freed by sf_destroy.
 *   - Errors: every call validates before launching anything and returns an
 *     sf_status; nothing is thrown across the ABI.  sf_last_error() gives a message
 *     (thread-local).  A handle is not thread-safe.
 */
#ifndef SF_H
#define SF_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SF_API __attribute__((visibility("default")))
#else
#define SF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SF_OK = 0,
    SF_ERR_INVALID_ARG = 1,   /* NULL required pointer, nt < 2, dt <= 0, h <= 0, min m <= 0 */
    SF_ERR_SHAPE = 2,         /* an extent < 2, or a slab with fewer than r local planes     */
    SF_ERR_ORDER = 3,         /* space_order odd, < 2 or > 16                                */
    SF_ERR_CFL = 4,           /* dt * vmax / h > 2 / sqrt(ndim * sum|w|)                      */
    SF_ERR_OUT_OF_DOMAIN = 5, /* sparse point outside the grid                               */
    SF_ERR_WORKSPACE = 6,     /* workspace too small                                         */
    SF_ERR_CUDA = 7,          /* CUDA runtime / driver error                                 */
    SF_ERR_NCCL = 8           /* NCCL error                                                  */
} sf_status;

typedef struct {
    int ndim;                 /* 2 or 3                                                      */
    int64_t shape[3];         /* computational grid (GLOBAL grid when distributed)            */
    double h;                 /* isotropic spacing [m]                                       */
    int space_order;          /* even, 2..16 (r = space_order/2 halo)                         */
    int nt;                   /* samples t_n = n dt, n = 0..nt-1 (nt-1 updates)                */
    double dt;                /* [s]                                                          */
    const float *m;           /* device [N] square slowness s^2/m^2, > 0 (local slab when     */
                              /* distributed: [n0_loc + 2r][n1][n2], halo planes unused)      */
    const float *damp;        /* device [N] eta >= 0, or NULL (== 0 everywhere)                */
    int nsrc;                 /* number of sources (forward injection, adjoint interpolation) */
    const double *src_coords; /* host [nsrc][ndim]                                            */
    int nrec;                 /* number of receivers                                          */
    const double *rec_coords; /* host [nrec][ndim]                                            */
    const float *sigma[3];    /* optional SEPARABLE damping (reading C7: eta = m sigma with    */
                              /* sigma = sum over axes of a 1D profile): host [shape[a]]      */
                              /* profiles sigma_a >= 0 [1/s] of the GLOBAL grid, a < ndim, all */
                              /* given or all NULL; with them `damp` must be NULL.  The kernel */
                              /* then regenerates beta = (1 - s)/(1 + s), s = sigma dt/2, from */
                              /* the profiles instead of streaming a beta array: 16 instead of */
                              /* 20 bytes per point-update.  eta is evaluated once (at the m  */
                              /* given); gradients are d J / d m at that fixed eta (C13).      */
} sf_desc;

typedef struct sf_handle sf_handle;

/* Centred 2nd-derivative FD weights of order space_order:
 * w[0] = centre, w[k] = weight at offsets +-k, k = 1..r, in units of 1/h^2. */
SF_API sf_status sf_fd_weights(int space_order, double *w /* host [r+1] */);

/* Validate (shape, order, CFL, domain), build interpolation / injection tables and the
 * hoisted coefficient arrays beta and c3 on the device.  Synchronises the device once. */
SF_API sf_status sf_create(const sf_desc *d, sf_handle **out);
/* Synchronises the device (work on any stream may still use the handle), then returns
 * the handle's device memory to the pool.  NULL is a no-op. */
SF_API void sf_destroy(sf_handle *h);

/* Forward propagation.
 *   wavelet [nt][nsrc]   source signatures (may be NULL iff nsrc == 0)
 *   rec     [nt][nrec]   OUT: rec[n] = P u^n (rec[0] = P u^0); may be NULL iff nrec == 0
 *   u       [2][N]       IN (u^{-1}, u^0) (zeros for a fresh run), OUT (u^{nt-2}, u^{nt-1})
 *   snaps   [nt_snap][N] or NULL: OUT u^n for n % save_every == 0, slot n/save_every,
 *                        nt_snap = (nt-1)/save_every + 1 (slot 0 = u^0)
 *   save_every           >= 1 when snaps != NULL                                      */
SF_API sf_status sf_forward(sf_handle *h, const float *wavelet, float *rec, float *u, float *snaps,
                     int save_every, void *stream);

/* Adjoint propagation.
 *   res  [nt][nrec]   injected at the receivers (scale dt^2/m)
 *   srca [nt][nsrc]   OUT: srca[n] = P_s v^n (srca[nt-1] = P_s v^{nt-1}); may be NULL iff nsrc == 0
 *   v    [2][N]       IN (v^{nt}, v^{nt-1}) (zeros), OUT (v^1, v^0)
 *   snaps, save_every as written by sf_forward; with grad != NULL the correlation
 *   grad -= k u^n (v^{n+1} - 2 v^n + v^{n-1}) / dt^2 (n % k == 0, n >= 1) is ACCUMULATED
 *   into grad [N] (fused into the stencil kernel).  snaps/grad NULL: no gradient.     */
SF_API sf_status sf_adjoint(sf_handle *h, const float *res, float *srca, float *v, const float *snaps,
                     int save_every, float *grad, void *stream);

/* res = d_syn - d_obs ([nt][nrec]) and *J = 1/2 sum res^2 accumulated in fp64 in a fixed
 * order (deterministic).  J is a HOST pointer; the call synchronises `stream`.        */
SF_API sf_status sf_residual(sf_handle *h, const float *d_syn, const float *d_obs, float *res,
                      double *J, void *stream);

/* Full FWI gradient at the handle's m: forward with snapshots every save_every steps,
 * residual against d_obs, adjoint with fused correlation.  grad [N] is OVERWRITTEN;
 * *J (host) = 1/2 ||d_syn - d_obs||^2.  ws: device workspace of
 * sf_gradient_workspace_bytes() bytes (caller-owned). Synchronises `stream` (for J). */
SF_API size_t sf_gradient_workspace_bytes(const sf_handle *h, int save_every);
SF_API sf_status sf_gradient(sf_handle *h, const float *wavelet, const float *d_obs, float *grad,
                      double *J, void *ws, size_t ws_bytes, int save_every, void *stream);

/* Memory-bounded form of sf_gradient: checkpoint-recompute.  The forward
 * stores only the state pair (u^{b-1}, u^b) at every segment start b = 0, S, 2S, ...
 * (segment = S time steps, a positive multiple of save_every); the backward sweep
 * recomputes each segment's forward from its checkpoint, keeping that segment's
 * snapshots only, and runs its adjoint steps.  Workspace ~ (2 ceil((nt-1)/S) + S/save_every
 * + 5) N floats instead of ((nt-1)/save_every + 5) N; one extra forward propagation.
 * The kernels are deterministic, so grad and *J are BITWISE equal to sf_gradient's.
 * SF_ERR_INVALID_ARG if segment is not a positive multiple of save_every. */
SF_API size_t sf_gradient_ckpt_workspace_bytes(const sf_handle *h, int save_every, int segment);
SF_API sf_status sf_gradient_ckpt(sf_handle *h, const float *wavelet, const float *d_obs, float *grad,
                                  double *J, void *ws, size_t ws_bytes, int save_every, int segment,
                                  void *stream);

/* Flat end-to-end form with HOST buffers (desc->m / desc->damp are HOST pointers here):
 * uploads m, damp and the wavelet, creates a handle, runs sf_forward from a zero state,
 * downloads rec [nt][nrec] and (optionally) u_final [2][N] = (u^{nt-2}, u^{nt-1}).
 * Uses a library-owned device cache reused across calls with the same sizes.
 * Synchronises `stream`. */
SF_API sf_status sf_forward_host(const sf_desc *host_desc, const float *wavelet_host, float *rec_host,
                          float *u_final_host, void *stream);
/* SURVEY 8(b)'s name for the same flat form (sf_create + sf_forward + sf_destroy). */
SF_API sf_status sf_forward_once(const sf_desc *host_desc, const float *wavelet_host, float *rec_host,
                          float *u_final_host, void *stream);

/* Profiling: when on, the library records CUDA events around every (SF_OPT_PROF_EVERY:
 * every n-th) stencil launch on the launch stream; sf_get_profile synchronises and returns the summed stencil-kernel
 * time, the number of stencil launches and of all kernel launches since the last reset. */
SF_API sf_status sf_set_profiling(sf_handle *h, int on);
SF_API sf_status sf_get_profile(sf_handle *h, double *stencil_ms, long long *stencil_launches,
                         long long *all_launches, int reset);

/* Per-kind launch times: ms_by_kind[4] / launches_by_kind[4] = {stencil, inject,
 * interpolate, other (swap, residual)}; synchronises like sf_get_profile. */
SF_API sf_status sf_get_profile_detail(sf_handle *h, double *ms_by_kind, long long *launches_by_kind,
                                       int reset);

/* Tuning: kernel variant (0 auto, 1 generic thread-per-point, 2 TMA 2.5D streaming),
 * TMA layout `vy` (0 auto = 2: 2 rows x 4 z per thread, 7 consumer warps, 14 x 128 tiles;
 * 1: one row per thread, 7-row tiles; 3, space order >= 10: 2 rows x 2 z per thread, 11
 * consumer warps, 22 x 64 tiles -- otherwise read as 2; 4: warp-specialised, 8 consumer warps
 * x 2 rows x 4 z, 16 x 128 tiles, a producer warpgroup handing its registers to the
 * consumers) for every step mode (clears the GRAD-mode layout sf_autotune sets), and the number of
 * persistent TMA CTAs `ctas` (0 auto = one per SM; the (tile, plane) work is split into
 * `ctas` equal runs; every setting gives the same bits).  SF_ERR_INVALID_ARG for other
 * values. */
SF_API sf_status sf_set_tuning(sf_handle *h, int variant, int vy, int ctas);
/* Options (sf_set_option): */
#define SF_OPT_L2_PREFETCH 1   /* TMA kernel: L2 prefetch distance in planes (default 0 = off; 8 was
                                  measured 8 % slower on configs[1] with the final kernel)         */
#define SF_OPT_SPLIT 2         /* 1: boundary planes first, then interior (always on in slab mode;
                                  on one GPU it only reorders work: results are bitwise identical) */
#define SF_OPT_FUSE_MAX 3      /* largest point set injected inside the stencil kernel (default
                                  256); larger sets use the standalone injection kernel          */
#define SF_OPT_COMM_SMS 4      /* split schedule: SMs the persistent interior launch leaves free
                                  for the concurrent halo exchange (NCCL kernels) and the side-
                                  stream records (default 8 in slab mode, 0 on one GPU; 0..64)   */
#define SF_OPT_GRAPH 5         /* 1: replay whole sf_forward / sf_adjoint calls as CUDA graphs:
                                  the second call with the same arguments (pointers, save_every,
                                  stream, nt) is captured once and then replayed on an internal
                                  stream ordered after / before `stream` by events -- for small,
                                  launch-bound grids.  Off while profiling and in slab mode;
                                  tuning or option changes drop the cached graphs. (default 0)  */
#define SF_OPT_SNAP_HALF 7     /* 1: every snapshot array (sf_forward / sf_adjoint `snaps`, the
                                  gradient workspaces) holds IEEE fp16 values, 2 bytes each:
                                  u^n rounded to nearest even when saved, widened exactly when
                                  correlated (reading C23; relative error <= 2^-11 per value in
                                  the normal range, values beyond 65504 overflow).  Half the
                                  snapshot memory and bytes.  The TMA kernel then needs
                                  n2 % 8 == 0 (else the generic kernel runs).  (default 0)       */
#define SF_OPT_P2P 8           /* slab handles: 1 replaces the per-step NCCL send/recv with
                                  peer stores -- the boundary-plane kernel (and the injection
                                  there) writes each owned boundary plane straight into the
                                  neighbour's halo of the same level, then bumps a counter in the
                                  neighbour's memory with a stream-ordered write; each rank's
                                  stream waits on its counters (cuStreamWaitValue32) before the
                                  halo is read.  Buffers are exchanged per call: local groups
                                  share pointers, NCCL ranks CUDA IPC handles (all-gathered over
                                  NCCL; the state buffer `u`/`v` must come from cudaMalloc, e.g.
                                  torch's caching allocator).  Every rank must own > 2r planes
                                  (SF_ERR_SHAPE).  Bitwise equal to the NCCL exchange.  Across
                                  processes the counter waits are blocking stream operations:
                                  run with CUDA_DEVICE_MAX_CONNECTIONS >= 16 so none can stall an
                                  unrelated stream sharing its hardware queue; in-process rank
                                  threads (local group) order with events instead. (default 0) */
#define SF_OPT_ZSPLIT 9        /* 3D TMA kernel, space order >= 10: 1 (default) runs a z remainder
                                  of n2 = 128 k + rem, 0 < rem <= 64, as a second launch of narrow
                                  56 x 32 tiles (the 128-column tiles there would be mostly idle
                                  lanes); sources are then injected by the standalone kernel.
                                  Bitwise the same.  (Lower orders run at the HBM roofline, where
                                  the extra launch costs more than the idle lanes.)             */
#define SF_OPT_ONE_LAUNCH 11   /* split schedule (slab handles; SF_OPT_SPLIT on one GPU): 1 (default)
                                  runs each step as ONE persistent TMA launch when the injection
                                  of the step happens inside it (fused source lists) -- the last x-chunk of every tile streams downward,
                                  each CTA fences and bumps a device counter when it has stored a
                                  boundary range, the comm stream waits on the counters
                                  (cuStreamWaitValue32) and runs the NCCL send/recv while the
                                  launch computes the interior.  Otherwise (or 0) the two-launch
                                  split (boundary launch on a high-priority stream, interior
                                  launch).  2: the one-launch schedule also on one GPU (the
                                  exchange becomes a copy into sf_debug_probe's buffer).  In-
                                  process local groups and SF_OPT_P2P keep the two-launch
                                  schedule.  Bitwise the same results.                          */
#define SF_OPT_PDL 12          /* 1 (default): launch the standalone injection kernel, and the stencil
                                  launch that follows it, with programmatic stream serialisation
                                  (PDL): the kernel's launch and prologue overlap the previous
                                  kernel's tail and it waits (griddepcontrol.wait) for that
                                  kernel's writes before its first global access (adjoints with a
                                  receiver set: +1-2 %).  Stencil -> stencil stays plain (no gain:
                                  a persistent launch cannot co-reside with the previous one).
                                  Bitwise the same results.  0: plain launches.                 */
#define SF_OPT_PROF_EVERY 13   /* profiling (sf_set_profiling): time every n-th launch of each kind
                                  (default 1 = every launch); sf_get_profile* scale the timed sum by
                                  launches / timed launches.  An event pair between two kernels
                                  costs 1-3 % of a step and defeats PDL.                          */
#define SF_OPT_LOOP2D 14       /* 1 (default): a small 2D grid (configs[0]: 141 x 141; up to ~200 k
                                  points) runs the whole sf_forward / sf_adjoint time loop (no
                                  snapshots, no gradient) in ONE launch of a 16-CTA cluster: each
                                  CTA holds a slab of rows (both levels, c3, beta) in shared
                                  memory, reads the neighbouring rows through distributed shared
                                  memory, and cluster barriers order stencil, injection and
                                  records step by step (launch-bound otherwise).  Bitwise the
                                  per-step kernels.  0: one launch per step.                     */
#define SF_OPT_BALANCE 16      /* TMA kernel work split: 0 (default) chunked, 1 balanced.
                                  Chunked: (tile, x-chunk) items dealt round-robin to the
                                  persistent CTAs (y/z-neighbouring tiles in step: their shared
                                  halo rows hit in L2), the chunk count minimising rounds x
                                  (chunk + 2r).  Balanced: CTA b streams the contiguous planes
                                  [b T / G, (b + 1) T / G) of all T (tile, plane) units (equal
                                  shares whatever the tile count; neighbours drift apart, halo
                                  rows re-read from HBM).  Sets the split of every step mode;
                                  sf_autotune chooses per mode.  Same bits.                      */
#define SF_OPT_TBLOCK 15       /* temporal blocking, default 0: 1 runs sf_forward without
                                  snapshots two time steps per launch (3D, space order <= 8, one
                                  GPU, no separable profiles, n_z % 4 == 0; SF_ERR_INVALID_ARG
                                  otherwise): each CTA computes step 1 on its tile grown by r
                                  rows / 4 columns per side and step 2 on the tile from one read
                                  of u^{n-1}, u^n, c3, beta (24 B per two updates instead of 40),
                                  bitwise equal to two single steps.  Allocates a second state
                                  pair (2 N floats) when set; an odd step count ends with one
                                  single step.  Measured slower than the single-step kernel on
                                  B200, hence off by default.              */
SF_API sf_status sf_set_option(sf_handle *h, int option, int value);
/* Setup-time tuning (the counterpart of the paper's runtime block-size auto-tuning,
 * P:729-731): times `steps` plain stencil steps (no sparse work) of every feasible launch
 * configuration -- TMA kernel with 14- or 7-row tiles, with or without the narrow remainder
 * tiles (space order >= 10), the thread-per-point kernel -- on the caller's scratch state u
 * ([2][Nloc] device floats, overwritten), keeps the fastest in the handle and returns it in
 * chosen[3] = {variant, vy, zsplit} (may be NULL) and its time per step in *ms (may be NULL).
 * At space order >= 10 every TMA candidate is timed with both work splits (SF_OPT_BALANCE).
 * With the TMA kernel it then times the 7- and 8-warp layouts (vy 2, 4; x both splits at
 * space order >= 10) in GRAD mode (the gradient's adjoint: snapshot and gradient planes
 * streamed beside the stencil; scratch values) and keeps the fastest for GRAD-mode steps
 * (sf_get_tuning_modes).
 * Every configuration computes the same bits.  Synchronises `stream`. */
SF_API sf_status sf_autotune(sf_handle *h, float *u, int steps, int *chosen, float *ms, void *stream);
/* Test hook of the one-launch schedule on one GPU (SF_OPT_ONE_LAUNCH 2): after each step's
 * counters fire, the comm stream copies the r boundary planes at each end of the new level
 * ([xa, xa + r) then [xb - r, xb), 2 r n1 n2 floats) into `dst` (device; NULL = off);
 * *one_launch_steps (may be NULL) = steps run with the one-launch schedule so far. */
SF_API sf_status sf_debug_probe(sf_handle *h, float *dst, long long *one_launch_steps);

/* Which variant / vy / ctas the next launch will use (after auto selection). */
SF_API sf_status sf_get_tuning(const sf_handle *h, int *variant, int *vy, int *ctas);
/* Per-mode tuning of the TMA kernel (each pointer may be NULL; 0s with the generic kernel):
 * the layout (vy) of GRAD-mode steps and the work split (SF_OPT_BALANCE: 0 chunked, 1
 * balanced) of the plain / SAVE steps and of the GRAD-mode steps, as sf_autotune left them.
 * SF_ERR_INVALID_ARG on a NULL handle. */
SF_API sf_status sf_get_tuning_modes(const sf_handle *h, int *vy_grad, int *balance, int *balance_grad);

/* ---- multi-GPU (slab decomposition along axis 0; one process per GPU, NCCL) ---- */

/* Host-only: the slab owned by `rank`: planes [*x0, *x0 + *n0_loc) of the global axis 0.
 * Needs no GPU.  SF_ERR_SHAPE if a rank would own fewer than r planes.            */
SF_API sf_status sf_slab_plan(int64_t n0, int space_order, int rank, int nranks, int64_t *x0,
                       int64_t *n0_loc);
/* Owner rank of a sparse point for injection corners / records (reading C18): the rank
 * owning plane floor-clamped base index along axis 0.  Host-only.                  */
SF_API sf_status sf_sparse_owner(int64_t n0, int space_order, int nranks, double h, double coord0,
                          int *owner);

/* Host-only: the halo exchange sf_forward / sf_adjoint perform after every step on a
 * rank's local buffer [n0_loc + 2r][...] (planes, counted along axis 0):
 *   plan[0] = first plane sent to rank-1        plan[1] = first plane received from rank-1
 *   plan[2] = first plane sent to rank+1        plan[3] = first plane received from rank+1
 *   plan[4] = planes per message (r); plan[5] = has left neighbour; plan[6] = has right. */
SF_API sf_status sf_slab_halo_plan(int64_t n0, int space_order, int rank, int nranks, int64_t plan[7]);

/* NCCL bootstrap: rank 0 calls sf_nccl_unique_id, broadcasts the 128 bytes (e.g. over
 * torch.distributed), every rank calls sf_nccl_comm_init.  The comm is caller-owned. */
SF_API sf_status sf_nccl_unique_id(char id_out[128]);
SF_API sf_status sf_nccl_comm_init(const char id[128], int nranks, int rank, void **comm_out);
SF_API sf_status sf_nccl_comm_destroy(void *comm);
/* Size and rank of an NCCL communicator (ncclCommCount / ncclCommUserRank), e.g. for a
 * harness to verify the communicator spans every rank.  SF_ERR_NCCL on failure. */
SF_API sf_status sf_nccl_comm_info(void *comm, int *nranks, int *rank);
/* Asynchronous-error poll (ncclCommGetAsyncError, non-blocking): SF_ERR_NCCL with the NCCL
 * message if the communicator has failed (a peer died, a link fault, ...).  The library also
 * polls after every NCCL enqueue it makes (halo exchange, record / gradient all-reduce), so a
 * failed exchange surfaces as SF_ERR_NCCL from the next sf_forward / sf_adjoint /
 * sf_gradient / sf_allreduce_gradient call instead of a hang being the only symptom.
 * An in-process group (sf_local_group_create) always reports SF_OK. */
SF_API sf_status sf_nccl_check(void *comm);

/* In-process transport (testing the slab path on ONE device): ranks are threads of one
 * process, each with its own handle and stream; a group created here is passed as the
 * `comm` of sf_create_slab / sf_allreduce_gradient instead of an NCCL communicator.  The
 * exchange moves the same planes as the NCCL path with cudaMemcpyAsync, ordered by CUDA
 * events and a host barrier per step (no kernel ever waits on another rank's kernel).
 * Every rank of the group must call the same sequence of library calls. */
SF_API sf_status sf_local_group_create(int nranks, void **group_out);
SF_API sf_status sf_local_group_destroy(void *group);

/* Slab handle: `global` holds the GLOBAL shape and sparse geometry; global->m/damp
 * point to the LOCAL slab arrays [n0_loc + 2r][n1][n2] (halo planes unused).  All
 * wavefield arrays passed to sf_forward/sf_adjoint are then local [n0_loc + 2r][n1][n2]
 * (u: [2][...]); records/srca are full [nt][npoint] arrays in which each rank writes the
 * rows of the points it owns (others are zeroed) -- sum them over ranks.  The halo of
 * r planes is exchanged every step with ncclSend/ncclRecv over NVLink (`comm` from
 * sf_nccl_comm_init), or with device copies when `comm` is a local group (above). */
SF_API sf_status sf_create_slab(const sf_desc *global, void *comm, int rank, int nranks,
                         sf_handle **out);
/* In-place fp32 sum of grad [Nloc] and fp64 sum of *J (host) over the communicator
 * (multi-shot FWI, one shot per GPU).  `rank` is the caller's rank in `comm` (used by the
 * in-process transport; NCCL knows it).  Synchronises `stream`. */
SF_API sf_status sf_allreduce_gradient(sf_handle *h, void *comm, float *grad, size_t count,
                                       double *J, int rank, void *stream);

/* ---- the paper's other example workloads, 2D fp32, layout [n0][n1] ---- */

/* Linear convection, Eq. 2: nt steps of
 *   u_ij <- u_ij - c dt/dx (u_ij - u_{i-1,j}) - c dt/dy (u_ij - u_{i,j-1})
 * on the interior; edge points keep their values (reading C21).  u: device [n0][n1],
 * in = initial, out = final.  Grids up to 25 600 points run in one CTA (both levels in
 * shared memory, no launch per step; work may be NULL); larger grids need `work`
 * (device [n0][n1] scratch) and launch one kernel per step.  Asynchronous on `stream`. */
SF_API sf_status sf_convection2d(float *u, float *work, int64_t n0, int64_t n1, double c, double dt,
                                 double dx, double dy, int nt, void *stream);

/* Laplace equation by Jacobi sweeps, Eq. 4, boundary rows as in the listing
 * (p[x,0]=0, p[x,n1-1]=bc[x], p[0,y]=p[1,y], p[n0-1,y]=p[n0-2,y]), l1 rule of
 * P:433-447 (reading C22): sweeps until l1 = sum(|p|-|pn|)/sum(|pn|) <= tol or max_iter.
 * p: device [n0][n1], in = initial buffer, out = the last computed p; bc: device [n0];
 * work: device [n0][n1] scratch (may be NULL for grids up to 4 096 points, which run in
 * one CTA; larger grids run one cooperative kernel over all SMs).  The l1 test never
 * leaves the device.  *iters / *l1 (host) receive the sweep count and the last l1.
 * Synchronises `stream`. */
SF_API sf_status sf_laplace2d(float *p, float *work, const float *bc, int64_t n0, int64_t n1, double dx,
                              double dy, double tol, int max_iter, int *iters, double *l1, void *stream);

SF_API const char *sf_last_error(void);
SF_API int sf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SF_H */
