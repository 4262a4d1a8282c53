// sf_internal.h -- handle layout and helpers shared by the host translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/sf.h"
#include "launch.cuh"

// Injection targets grouped by (tile, consumer warp) of the TMA kernel (fused injection).
struct SfInjTiles {
    int by = 0;          // rows per thread (VY) the lists were built for (0 = not built)
    int *beg = nullptr;  // [ntiles * by + 1]
    int *q = nullptr, *lj = nullptr, *t = nullptr;
};

// Sparse point set on the device (one for sources, one for receivers).
struct SfSparse {
    int np = 0;          // points
    int nc = 0;          // corners per point (2^ndim)
    // interpolation: ELL tables e_idx / e_w below (nonzero corners in corner order)
    int *i_owned = nullptr;  // slab mode: 1 if this rank writes the record row
    // injection: CSR by target grid point
    int ntgt = 0;
    int nent = 0;
    int64_t *j_tgt = nullptr;
    int *j_rowptr = nullptr;
    int *j_pt = nullptr;
    float *j_coef = nullptr;  // W dt^2 / m[target]
    // ELL (slot-major) copies used by the standalone kernels
    int ik = 0;               // interpolation slots per point (max nonzero corners)
    int64_t *e_idx = nullptr;
    float *e_w = nullptr;
    int jk = 0;               // injection slots per target (0: use CSR)
    int *ej_pt = nullptr;
    float *ej_coef = nullptr;
    // split launches: target rows in the boundary planes / in the interior
    int *jl_bnd = nullptr, *jl_int = nullptr;
    int n_bnd = -1, n_int = 0;
    std::vector<int64_t> h_tgt;  // host copy of the target offsets
    SfInjTiles tiles;
};

// One cached CUDA graph of a whole sf_forward / sf_adjoint call (SF_OPT_GRAPH): the
// arguments it was captured with, and the arguments of the last eager call (a call is
// captured the second time the same arguments come, after the first one has built every
// lazily created table).
struct SfGraphCache {
    const void *key[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    long long ikey[3] = {0, 0, 0};
    const void *seen[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    long long iseen[3] = {-1, -1, -1};
    cudaGraphExec_t exec = nullptr;
};

struct sf_handle {
    int ndim = 3;
    int64_t gshape[3] = {1, 1, 1};  // global computational grid
    int64_t nb[3] = {1, 1, 1};      // local buffer extents (axis 0 includes slab halos)
    int64_t N = 0;                  // points in the local buffer
    int64_t xa = 0, xb = 0;         // computed planes of the buffer
    double h = 0, dt = 0;
    int so = 0, r = 0, nt = 0;
    SfWeights w{};
    float *c3 = nullptr;
    float *beta = nullptr;
    bool damp = false;              // hoisted beta array (sf_desc.damp given)
    bool sep = false;               // separable damping profiles (sf_desc.sigma given)
    float *sig[3] = {nullptr, nullptr, nullptr};  // local profiles: buffer planes, y, z
    SfSparse src, rec;
    double *partial = nullptr;  // residual partial sums
    double *dJ = nullptr;
    // tuning
    int variant = SF_VAR_AUTO, vy = 0, ctas = 0;
    int vy_grad = 0;                // TMA layout of GRAD-mode steps (0: as vy; set by sf_autotune)
    int balance = 0;                // TMA work split (SF_OPT_BALANCE): 0 chunked, 1 balanced
    int balance_grad = -1;          // ... of GRAD-mode steps (-1: as balance; set by sf_autotune)
    int l2_prefetch = 0;            // TMA L2 prefetch distance (planes, 0 = off); env SF_L2_PREFETCH
    // slab decomposition
    int rank = 0, nranks = 1;
    void *comm = nullptr;
    int64_t x0 = 0, n0_loc = 0;
    // profiling
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_kind;       // kind of event pair i (stencil / inject / interp / other)
    size_t ev_used = 0;
    long long n_kind[4] = {0, 0, 0, 0};
    long long n_samp[4] = {0, 0, 0, 0};  // launches actually timed per kind
    int prof_every = 1;                   // SF_OPT_PROF_EVERY
    long long n_all = 0;
    int sms = 148;                  // multiprocessors of the device (set at create)
    // side stream for records (overlap with the next stencil step)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_itp[2] = {nullptr, nullptr};
    bool itp_pending[2] = {false, false};
    // boundary-first split launches (always in slab mode; optional on one GPU)
    bool split = false;
    cudaStream_t comm_stream = nullptr, hi_stream = nullptr;
    cudaEvent_t ev_pre = nullptr, ev_bnd = nullptr, ev_xch = nullptr;
    int fuse_max = 256;
    int comm_sms = -1;              // SMs left free by the split interior launch (-1: auto)
    // CUDA graphs of whole time loops (SF_OPT_GRAPH), run on gstream between two events
    bool use_graph = false;
    bool snap_half = false;         // snapshots stored as fp16 (SF_OPT_SNAP_HALF, reading C23)
    SfGraphCache gfwd, gadj;
    cudaStream_t gstream = nullptr;
    cudaEvent_t ev_gin = nullptr, ev_gout = nullptr;
    // peer-store halo exchange (SF_OPT_P2P): the boundary-plane kernel stores the
    // owned boundary planes straight into the neighbours' halos (peer-mapped pointers) and
    // signals with a stream-ordered counter write; the neighbour's stream waits on the value
    bool zsplit = true;               // SF_OPT_ZSPLIT: narrow tiles for a z remainder <= 64
    // one-launch slab schedule (SF_OPT_ONE_LAUNCH): the stencil launch signals its finished
    // boundary ranges on device counters; the comm stream waits on them, then exchanges
    bool loop2d = true;               // SF_OPT_LOOP2D: small 2D grids run the whole time loop in one CTA
    bool pdl = true;                  // SF_OPT_PDL: programmatic dependent launches (injection, stencil after it)
    bool prev_inject = false;         // the last kernel launched on the step stream was an injection
    int one_launch = 1;               // 1: in NCCL slab mode when applicable; 2: also on one GPU (emulation)
    unsigned int *sigc = nullptr;     // [2] left / right boundary counters (monotonic)
    uint32_t sig_tgt = 0;             // counter value that marks the current step's boundaries
    int last_tiles = 0;               // tiles of the last bidir launch (signals per side)
    float *probe = nullptr;           // test hook: boundary planes copied here on the comm stream
    long long n_onelaunch = 0;        // steps run with the one-launch schedule
    bool p2p = false;
    uint32_t *p2p_flags = nullptr;    // own device counters: [0] written by the left, [1] by the right neighbour
    uint32_t p2p_seq = 0;             // P2P steps completed (the value the next step writes is seq + 1)
    float *p2p_own[2] = {nullptr, nullptr};                  // own state buffers (A, B) of the current call
    float *p2p_nbr[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [left/right][A/B] of the neighbours
    uint32_t *p2p_nflag[2] = {nullptr, nullptr};             // the neighbours' counters this rank writes
    std::vector<std::pair<std::string, void *>> ipc_open;    // opened IPC handles (NCCL mode), closed at destroy
    // two steps per pass (SF_OPT_TBLOCK, stencil_tb2.cuh): the second buffer pair the
    // forward rotates through, and the per-tile source lists of the two-step kernel
    bool tblock = false;
    float *tb_buf = nullptr;          // [2][N]
    int *tb_beg = nullptr, *tb_q = nullptr, *tb_p = nullptr, *tb_t = nullptr;
    long long n_tb = 0;               // two-step launches so far
};

// error reporting (thread-local message)
sf_status sf_set_error(sf_status s, const char *fmt, ...);
#define SF_CUDA_TRY(call)                                                                  \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return sf_set_error(SF_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                __FILE__, __LINE__);                                       \
    } while (0)

// comm.cu
sf_status sf_comm_halo_exchange(sf_handle *h, float *buf, cudaStream_t st);
// SF_OPT_P2P: publish this rank's state buffers (A, B) and counters, fetch the neighbours'
// (local group: in-process pointers; NCCL: CUDA IPC handles all-gathered over NCCL)
sf_status sf_comm_p2p_setup(sf_handle *h, float *A, float *B, cudaStream_t st);
void sf_comm_p2p_release(sf_handle *h);
bool sf_comm_p2p_local(sf_handle *h);
sf_status sf_comm_p2p_local_step(sf_handle *h, cudaStream_t st, bool left, bool right);
sf_status sf_comm_allreduce_f32(void *comm, float *buf, size_t count, cudaStream_t st, int rank);
sf_status sf_comm_allreduce_f64(void *comm, double *buf, size_t count, cudaStream_t st, int rank);
bool sf_comm_is_local(void *comm);
sf_status sf_comm_check_async(void *comm);
