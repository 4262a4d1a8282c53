// comm.cu -- multi-GPU plumbing over NCCL (NVLink 5 / NVSwitch): slab halo exchange
// and the multi-shot gradient all-reduce (a8).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") so that libsf.so loads on
// hosts without NCCL and reuses the NCCL that torch already loaded (torch wheel,
// 2.28.x) -- only one NCCL per process.  Header: the torch wheel's nccl.h.
//
// Halo exchange of the newest time level, after its stencil + injection (reading C18):
//   send owned planes [r, 2r)              -> left neighbour's right halo [n0_loc + r, n0_loc + 2r)
//   send owned planes [n0_loc, n0_loc + r) -> right neighbour's left halo [0, r)
// Each face is one contiguous r * n1 * n2 block (x is the outermost axis): no packing.
// Global edges keep their zero halo (Dirichlet ghost, reading C6).
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <condition_variable>
#include <mutex>
#include <set>
#include <vector>

#include <nccl.h>

#include "sf_internal.h"

namespace {
struct NcclApi {
    void *lib = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
    decltype(&ncclCommCount) CommCount = nullptr;
    decltype(&ncclCommUserRank) CommUserRank = nullptr;
    bool ok = false;
};

NcclApi &api()
{
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names) {
            a.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (a.lib) break;
        }
        if (!a.lib) return;
#define SF_SYM(f) a.f = reinterpret_cast<decltype(a.f)>(dlsym(a.lib, "nccl" #f))
        SF_SYM(GetUniqueId);
        SF_SYM(CommInitRank);
        SF_SYM(CommDestroy);
        SF_SYM(Send);
        SF_SYM(Recv);
        SF_SYM(GroupStart);
        SF_SYM(GroupEnd);
        SF_SYM(AllReduce);
        SF_SYM(AllGather);
        SF_SYM(GetErrorString);
        SF_SYM(CommGetAsyncError);
        SF_SYM(CommCount);
        SF_SYM(CommUserRank);
#undef SF_SYM
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv &&
               a.GroupStart && a.GroupEnd && a.AllReduce && a.AllGather && a.GetErrorString &&
               a.CommGetAsyncError && a.CommCount && a.CommUserRank;
    });
    return a;
}

sf_status nccl_err(const char *what, ncclResult_t r)
{
    return sf_set_error(SF_ERR_NCCL, "%s: %s", what, api().GetErrorString ? api().GetErrorString(r) : "?");
}
}  // namespace

#define SF_NCCL_TRY(call)                                   \
    do {                                                    \
        ncclResult_t r_ = (call);                           \
        if (r_ != ncclSuccess) return nccl_err(#call, r_);  \
    } while (0)

static sf_status need_nccl()
{
    if (!api().ok) return sf_set_error(SF_ERR_NCCL, "libnccl.so.2 could not be loaded");
    return SF_OK;
}

extern "C" sf_status sf_nccl_unique_id(char id_out[128])
{
    sf_status s = need_nccl();
    if (s) return s;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    SF_NCCL_TRY(api().GetUniqueId(&id));
    memcpy(id_out, &id, 128);
    return SF_OK;
}

extern "C" sf_status sf_nccl_comm_init(const char id[128], int nranks, int rank, void **comm_out)
{
    sf_status s = need_nccl();
    if (s) return s;
    if (!comm_out) return sf_set_error(SF_ERR_INVALID_ARG, "comm_out is NULL");
    ncclUniqueId uid;
    memcpy(&uid, id, 128);
    ncclComm_t c = nullptr;
    SF_NCCL_TRY(api().CommInitRank(&c, nranks, uid, rank));
    *comm_out = c;
    return SF_OK;
}

// Asynchronous NCCL errors (a peer died, a network/NVLink fault, ...) are not returned by
// the enqueue calls: poll the communicator (non-blocking) and surface them as SF_ERR_NCCL.
// Called after every NCCL enqueue of the library; ncclInProgress (a non-blocking
// communicator still initialising) is not an error.
sf_status sf_comm_check_async(void *comm)
{
    if (!comm || sf_comm_is_local(comm) || !api().ok) return SF_OK;
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = api().CommGetAsyncError(static_cast<ncclComm_t>(comm), &ar);
    if (r != ncclSuccess) return nccl_err("ncclCommGetAsyncError", r);
    if (ar != ncclSuccess && ar != ncclInProgress) return nccl_err("asynchronous NCCL error", ar);
    return SF_OK;
}

extern "C" sf_status sf_nccl_check(void *comm)
{
    if (!comm) return sf_set_error(SF_ERR_INVALID_ARG, "comm is NULL");
    return sf_comm_check_async(comm);
}

extern "C" sf_status sf_nccl_comm_info(void *comm, int *nranks, int *rank)
{
    sf_status s = need_nccl();
    if (s) return s;
    if (!comm) return sf_set_error(SF_ERR_INVALID_ARG, "comm is NULL");
    int n = 0, r = 0;
    SF_NCCL_TRY(api().CommCount(static_cast<ncclComm_t>(comm), &n));
    SF_NCCL_TRY(api().CommUserRank(static_cast<ncclComm_t>(comm), &r));
    if (nranks) *nranks = n;
    if (rank) *rank = r;
    return SF_OK;
}

extern "C" sf_status sf_nccl_comm_destroy(void *comm)
{
    sf_status s = need_nccl();
    if (s) return s;
    if (comm) SF_NCCL_TRY(api().CommDestroy(static_cast<ncclComm_t>(comm)));
    return SF_OK;
}

// ------------------------------------------------------------ in-process transport
namespace {
struct LocalGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int count = 0;
    long long gen = 0;
    std::vector<cudaEvent_t> ev, done;
    std::vector<void *> ptr;
    std::vector<void *> p2p;  // [rank][3]: state buffers A, B and the P2P counters
    std::vector<cudaEvent_t> bnd;  // [rank]: the rank's boundary-done event (SF_OPT_P2P)
    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const long long g = gen;
        if (++count == n) {
            count = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
std::mutex g_groups_mu;
std::set<void *> g_groups;

LocalGroup *as_local(void *comm)
{
    std::lock_guard<std::mutex> lk(g_groups_mu);
    return g_groups.count(comm) ? static_cast<LocalGroup *>(comm) : nullptr;
}

template <class T>
__global__ void k_accumulate(T *__restrict__ dst, const T *__restrict__ src, size_t n)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

// sum over the group into every rank's buf: rank 0 accumulates ranks 1.. in rank order,
// the others copy the sum back; events order the streams, barriers order the host calls
template <class T>
sf_status local_allreduce(LocalGroup *G, int rank, T *buf, size_t count, cudaStream_t st)
{
    G->ptr[rank] = buf;
    SF_CUDA_TRY(cudaEventRecord(G->ev[rank], st));
    G->barrier();
    if (rank == 0) {
        for (int q = 1; q < G->n; ++q) {
            SF_CUDA_TRY(cudaStreamWaitEvent(st, G->ev[q], 0));
            k_accumulate<T><<<592, 256, 0, st>>>(buf, static_cast<const T *>(G->ptr[q]), count);
            SF_CUDA_TRY(cudaGetLastError());
        }
        SF_CUDA_TRY(cudaEventRecord(G->done[0], st));
    }
    G->barrier();
    if (rank != 0) {
        SF_CUDA_TRY(cudaStreamWaitEvent(st, G->done[0], 0));
        SF_CUDA_TRY(cudaMemcpyAsync(buf, G->ptr[0], count * sizeof(T), cudaMemcpyDeviceToDevice, st));
        SF_CUDA_TRY(cudaEventRecord(G->done[rank], st));
    }
    G->barrier();
    if (rank == 0)  // rank 0's buffer was read by everyone: order its later writes
        for (int q = 1; q < G->n; ++q) SF_CUDA_TRY(cudaStreamWaitEvent(st, G->done[q], 0));
    G->barrier();
    return SF_OK;
}
}  // namespace

extern "C" sf_status sf_local_group_create(int nranks, void **group_out)
{
    if (nranks < 1 || !group_out) return sf_set_error(SF_ERR_INVALID_ARG, "bad local group (%d)", nranks);
    LocalGroup *G = new LocalGroup();
    G->n = nranks;
    G->ev.resize(nranks);
    G->done.resize(nranks);
    G->ptr.assign(nranks, nullptr);
    G->p2p.assign(3 * (size_t)nranks, nullptr);
    G->bnd.assign(nranks, nullptr);
    for (int q = 0; q < nranks; ++q) {
        SF_CUDA_TRY(cudaEventCreateWithFlags(&G->ev[q], cudaEventDisableTiming));
        SF_CUDA_TRY(cudaEventCreateWithFlags(&G->done[q], cudaEventDisableTiming));
    }
    std::lock_guard<std::mutex> lk(g_groups_mu);
    g_groups.insert(G);
    *group_out = G;
    return SF_OK;
}

extern "C" sf_status sf_local_group_destroy(void *group)
{
    LocalGroup *G = as_local(group);
    if (!G) return sf_set_error(SF_ERR_INVALID_ARG, "not a local group");
    {
        std::lock_guard<std::mutex> lk(g_groups_mu);
        g_groups.erase(group);
    }
    cudaDeviceSynchronize();
    for (int q = 0; q < G->n; ++q) {
        cudaEventDestroy(G->ev[q]);
        cudaEventDestroy(G->done[q]);
    }
    delete G;
    return SF_OK;
}

bool sf_comm_is_local(void *comm) { return as_local(comm) != nullptr; }

// the local form of the halo exchange below: the same planes, copied from the neighbours'
// buffers after their step (event), the neighbours' next writes ordered after the copies
static sf_status local_halo_exchange(sf_handle *h, LocalGroup *G, float *buf, cudaStream_t st)
{
    int64_t plan[7], qp[7];
    sf_status s;
    if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank, h->nranks, plan))) return s;
    const int64_t plane = h->N / h->nb[0];
    const size_t bytes = sizeof(float) * (size_t)plan[4] * (size_t)plane;
    G->ptr[h->rank] = buf;
    SF_CUDA_TRY(cudaEventRecord(G->ev[h->rank], st));
    G->barrier();
    if (plan[5]) {  // left halo <- left neighbour's planes it sends right
        if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank - 1, h->nranks, qp))) return s;
        SF_CUDA_TRY(cudaStreamWaitEvent(st, G->ev[h->rank - 1], 0));
        SF_CUDA_TRY(cudaMemcpyAsync(buf + plan[1] * plane, static_cast<float *>(G->ptr[h->rank - 1]) + qp[2] * plane,
                                    bytes, cudaMemcpyDeviceToDevice, st));
    }
    if (plan[6]) {  // right halo <- right neighbour's planes it sends left
        if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank + 1, h->nranks, qp))) return s;
        SF_CUDA_TRY(cudaStreamWaitEvent(st, G->ev[h->rank + 1], 0));
        SF_CUDA_TRY(cudaMemcpyAsync(buf + plan[3] * plane, static_cast<float *>(G->ptr[h->rank + 1]) + qp[0] * plane,
                                    bytes, cudaMemcpyDeviceToDevice, st));
    }
    SF_CUDA_TRY(cudaEventRecord(G->done[h->rank], st));
    G->barrier();
    if (plan[5]) SF_CUDA_TRY(cudaStreamWaitEvent(st, G->done[h->rank - 1], 0));
    if (plan[6]) SF_CUDA_TRY(cudaStreamWaitEvent(st, G->done[h->rank + 1], 0));
    h->n_all++;
    h->n_kind[3]++;
    return SF_OK;
}

sf_status sf_comm_halo_exchange(sf_handle *h, float *buf, cudaStream_t st)
{
    if (LocalGroup *G = as_local(h->comm)) return local_halo_exchange(h, G, buf, st);
    sf_status s = need_nccl();
    if (s) return s;
    int64_t plan[7];
    if ((s = sf_slab_halo_plan(h->gshape[0], h->so, h->rank, h->nranks, plan))) return s;
    const int64_t plane = h->N / h->nb[0];
    const size_t cnt = (size_t)plan[4] * (size_t)plane;
    ncclComm_t c = static_cast<ncclComm_t>(h->comm);
    SF_NCCL_TRY(api().GroupStart());
    if (plan[5]) {
        SF_NCCL_TRY(api().Send(buf + plan[0] * plane, cnt, ncclFloat, h->rank - 1, c, st));
        SF_NCCL_TRY(api().Recv(buf + plan[1] * plane, cnt, ncclFloat, h->rank - 1, c, st));
    }
    if (plan[6]) {
        SF_NCCL_TRY(api().Send(buf + plan[2] * plane, cnt, ncclFloat, h->rank + 1, c, st));
        SF_NCCL_TRY(api().Recv(buf + plan[3] * plane, cnt, ncclFloat, h->rank + 1, c, st));
    }
    SF_NCCL_TRY(api().GroupEnd());
    h->n_all++;
    h->n_kind[3]++;
    return sf_comm_check_async(h->comm);
}

sf_status sf_comm_allreduce_f32(void *comm, float *buf, size_t count, cudaStream_t st, int rank)
{
    if (LocalGroup *G = as_local(comm)) return local_allreduce<float>(G, rank, buf, count, st);
    sf_status s = need_nccl();
    if (s) return s;
    SF_NCCL_TRY(api().AllReduce(buf, buf, count, ncclFloat, ncclSum, static_cast<ncclComm_t>(comm), st));
    return sf_comm_check_async(comm);
}

sf_status sf_comm_allreduce_f64(void *comm, double *buf, size_t count, cudaStream_t st, int rank)
{
    if (LocalGroup *G = as_local(comm)) return local_allreduce<double>(G, rank, buf, count, st);
    sf_status s = need_nccl();
    if (s) return s;
    SF_NCCL_TRY(api().AllReduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), st));
    return sf_comm_check_async(comm);
}

extern "C" sf_status sf_allreduce_gradient(sf_handle *h, void *comm, float *grad, size_t count,
                                           double *J, int rank, void *stream)
{
    if (!comm || !grad) return sf_set_error(SF_ERR_INVALID_ARG, "NULL argument");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    sf_status s = sf_comm_allreduce_f32(comm, grad, count, st, rank);
    if (s) return s;
    if (J) {
        double *dJ = h ? h->dJ : nullptr;
        bool own = false;
        if (!dJ) {
            SF_CUDA_TRY(cudaMalloc(&dJ, sizeof(double)));
            own = true;
        }
        SF_CUDA_TRY(cudaMemcpyAsync(dJ, J, sizeof(double), cudaMemcpyHostToDevice, st));
        if ((s = sf_comm_allreduce_f64(comm, dJ, 1, st, rank))) return s;
        SF_CUDA_TRY(cudaMemcpyAsync(J, dJ, sizeof(double), cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaStreamSynchronize(st));
        if (own) cudaFree(dJ);
    } else {
        SF_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return SF_OK;
}

// ------------------------------------------------------------ peer-store halo exchange
// (SF_OPT_P2P).  Every call publishes the rank's state buffers (A, B: the two
// time levels it ping-pongs) and its counters; the neighbours' copies become the mirror
// targets of the boundary-plane stencil / injection and of the counter writes.
static sf_status ipc_open(sf_handle *h, const cudaIpcMemHandle_t &hd, void **out)
{
    const std::string key(reinterpret_cast<const char *>(&hd), sizeof hd);
    for (auto &e : h->ipc_open)
        if (e.first == key) {
            *out = e.second;
            return SF_OK;
        }
    void *p = nullptr;
    SF_CUDA_TRY(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
    h->ipc_open.emplace_back(key, p);
    *out = p;
    return SF_OK;
}

sf_status sf_comm_p2p_setup(sf_handle *h, float *A, float *B, cudaStream_t st)
{
    h->p2p_own[0] = A;
    h->p2p_own[1] = B;
    void *mine[3] = {A, B, h->p2p_flags};
    const int nb[2] = {h->rank - 1, h->rank + 1};
    void *theirs[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    if (LocalGroup *G = as_local(h->comm)) {
        for (int k = 0; k < 3; ++k) G->p2p[3 * (size_t)h->rank + k] = mine[k];
        G->bnd[h->rank] = h->ev_bnd;
        SF_CUDA_TRY(cudaEventRecord(G->ev[h->rank], st));
        G->barrier();
        for (int side = 0; side < 2; ++side) {
            const int q = nb[side];
            if (q < 0 || q >= h->nranks) continue;
            for (int k = 0; k < 3; ++k) theirs[side][k] = G->p2p[3 * (size_t)q + k];
            // the neighbour's earlier work on those buffers comes first
            SF_CUDA_TRY(cudaStreamWaitEvent(st, G->ev[q], 0));
        }
        G->barrier();
    } else {
        // separate processes: CUDA IPC handles of the allocations holding A, B and the
        // counters (+ offsets), all-gathered over NCCL; opened once per handle
        sf_status s = need_nccl();
        if (s) return s;
        static PFN_cuMemGetAddressRange_v3020 range = nullptr;
        if (!range) {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                return sf_set_error(SF_ERR_CUDA, "cuMemGetAddressRange unavailable");
            range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
        }
        struct Rec {
            cudaIpcMemHandle_t hd[3];
            int64_t off[3];
        };
        Rec me;
        memset(&me, 0, sizeof me);
        for (int k = 0; k < 3; ++k) {
            CUdeviceptr base = 0;
            size_t sz = 0;
            if (range(&base, &sz, reinterpret_cast<CUdeviceptr>(mine[k])) != CUDA_SUCCESS)
                return sf_set_error(SF_ERR_CUDA, "cuMemGetAddressRange failed");
            SF_CUDA_TRY(cudaIpcGetMemHandle(&me.hd[k], reinterpret_cast<void *>(base)));
            me.off[k] = reinterpret_cast<char *>(mine[k]) - reinterpret_cast<char *>(base);
        }
        std::vector<Rec> all(h->nranks);
        Rec *d = nullptr;
        SF_CUDA_TRY(cudaMalloc(&d, sizeof(Rec) * (h->nranks + 1)));
        SF_CUDA_TRY(cudaMemcpyAsync(d + h->nranks, &me, sizeof(Rec), cudaMemcpyHostToDevice, st));
        SF_NCCL_TRY(api().AllGather(d + h->nranks, d, sizeof(Rec), ncclChar, static_cast<ncclComm_t>(h->comm), st));
        SF_CUDA_TRY(cudaMemcpyAsync(all.data(), d, sizeof(Rec) * h->nranks, cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaStreamSynchronize(st));
        cudaFree(d);
        for (int side = 0; side < 2; ++side) {
            const int q = nb[side];
            if (q < 0 || q >= h->nranks) continue;
            for (int k = 0; k < 3; ++k) {
                void *p = nullptr;
                if ((s = ipc_open(h, all[q].hd[k], &p))) return s;
                theirs[side][k] = static_cast<char *>(p) + all[q].off[k];
            }
        }
    }
    for (int side = 0; side < 2; ++side) {
        h->p2p_nbr[side][0] = static_cast<float *>(theirs[side][0]);
        h->p2p_nbr[side][1] = static_cast<float *>(theirs[side][1]);
        // the left neighbour's counter [1] is written by its right neighbour (this rank), the
        // right neighbour's counter [0] by its left neighbour
        h->p2p_nflag[side] = theirs[side][2] ? static_cast<uint32_t *>(theirs[side][2]) + (side == 0 ? 1 : 0)
                                             : nullptr;
    }
    return SF_OK;
}

void sf_comm_p2p_release(sf_handle *h)
{
    for (auto &e : h->ipc_open) cudaIpcCloseMemHandle(e.second);
    h->ipc_open.clear();
}

// SF_OPT_P2P step ordering inside one process (local group): the rank threads share one
// device context, where a counter wait (cuStreamWaitValue32) enqueued ahead of the
// neighbour's counter write can block that write through a shared hardware queue (seen
// as a hang with 3 ranks x 5 streams > CUDA_DEVICE_MAX_CONNECTIONS = 8).  Events cannot:
// each rank records its boundary-done event, a host barrier makes every record precede
// the neighbours' waits, and a second barrier keeps the next step's record after them.
bool sf_comm_p2p_local(sf_handle *h) { return as_local(h->comm) != nullptr; }

sf_status sf_comm_p2p_local_step(sf_handle *h, cudaStream_t st, bool left, bool right)
{
    LocalGroup *G = as_local(h->comm);
    if (!G) return sf_set_error(SF_ERR_INVALID_ARG, "not a local group");
    G->barrier();
    if (left) SF_CUDA_TRY(cudaStreamWaitEvent(st, G->bnd[h->rank - 1], 0));
    if (right) SF_CUDA_TRY(cudaStreamWaitEvent(st, G->bnd[h->rank + 1], 0));
    G->barrier();
    return SF_OK;
}
