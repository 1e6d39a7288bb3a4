// tca_dist.cu -- mode-1 sharding support:
// shard layout (host), and the two transports a sharded operator uses for
// its two exchange steps per CG iteration:
//   * halo: the 3 boundary mode-1 slabs of p (or of an apply input) to each
//     neighbour (the band of G_1 has half-width 3, R_1 has 2);
//   * allreduce: the fp64 CG scalars <p, q> and <r, r> (Eq. A13/A14 summed
//     over shards).
// NcclTransport: NCCL send/recv + all-reduce on the caller's stream (NVLink /
// NVSwitch on one node); libnccl is loaded lazily with dlopen so the library
// has no link-time NCCL dependency.
// LocalTransport: shards of one process (threads, same or different
// devices) synchronised on the host -- test transport for hosts with fewer
// GPUs than shards; it moves the same bytes with cudaMemcpy.
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "tca_internal.cuh"

namespace tca {

// ---------------------------------------------------------------- layout
tca_status shard_layout(int64_t n1, const double *A1, int64_t m1, int rank, int nranks, int64_t out[4])
{
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TCA_ERR_INVALID_ARG, "bad rank / nranks");
    if (n1 < (int64_t)kHG * nranks)
        return fail(TCA_ERR_SHAPE, "n1 must be >= 3 * nranks (each shard holds at least the halo depth)");
    const int64_t lo = n1 * rank / nranks, hi = n1 * (rank + 1) / nranks;
    // data rows whose basis row touches an owned unknown: support of columns [lo, hi) of A_1
    int64_t dlo = m1, dhi = 0;
    for (int64_t k = 0; k < m1; ++k)
        for (int64_t c = lo; c < hi; ++c)
            if (A1[k * n1 + c] != 0.0) {
                dlo = std::min(dlo, k);
                dhi = std::max(dhi, k + 1);
                break;
            }
    if (dhi <= dlo) { dlo = 0; dhi = 0; }
    out[0] = lo;
    out[1] = hi;
    out[2] = dlo;
    out[3] = dhi;
    return TCA_OK;
}

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {

typedef struct { char internal[128]; } ncclUniqueId_t;
typedef void *ncclComm_t;
enum { ncclSuccess = 0, ncclInProgress = 7 };
enum { ncclFloat64 = 8 };
enum { ncclSum = 0 };

struct NcclApi {
    void *h = nullptr;
    int (*GetUniqueId)(ncclUniqueId_t *) = nullptr;
    int (*CommInitRank)(ncclComm_t *, int, ncclUniqueId_t, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
    int (*CommGetAsyncError)(ncclComm_t, int *) = nullptr;   // optional (error polling)
    int (*CommAbort)(ncclComm_t) = nullptr;                  // optional
    bool ok = false;
};

NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // prefer an already loaded NCCL (e.g. PyTorch's), then the system one
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names) {
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
            if (!api.h) api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        auto sym = [](const char *s) { return dlsym(api.h, s); };
        api.GetUniqueId = (int (*)(ncclUniqueId_t *))sym("ncclGetUniqueId");
        api.CommInitRank = (int (*)(ncclComm_t *, int, ncclUniqueId_t, int))sym("ncclCommInitRank");
        api.CommDestroy = (int (*)(ncclComm_t))sym("ncclCommDestroy");
        api.AllReduce = (int (*)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t))sym("ncclAllReduce");
        api.Send = (int (*)(const void *, size_t, int, int, ncclComm_t, cudaStream_t))sym("ncclSend");
        api.Recv = (int (*)(void *, size_t, int, int, ncclComm_t, cudaStream_t))sym("ncclRecv");
        api.GroupStart = (int (*)())sym("ncclGroupStart");
        api.GroupEnd = (int (*)())sym("ncclGroupEnd");
        api.GetErrorString = (const char *(*)(int))sym("ncclGetErrorString");
        api.CommGetAsyncError = (int (*)(ncclComm_t, int *))sym("ncclCommGetAsyncError");
        api.CommAbort = (int (*)(ncclComm_t))sym("ncclCommAbort");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.Send && api.Recv &&
                 api.GroupStart && api.GroupEnd;
    });
    return api;
}

tca_status nccl_fail(int r, const char *what)
{
    const char *msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    return fail(TCA_ERR_NCCL, std::string(what) + ": " + msg);
}

#define TCA_NCCL_TRY(expr)                                          \
    do {                                                            \
        int r_ = (expr);                                            \
        if (r_ != ncclSuccess) return nccl_fail(r_, #expr);         \
    } while (0)

class NcclTransport final : public Transport {
  public:
    NcclTransport(void *comm, int rank, int nranks) : comm_(comm), rank_(rank), nranks_(nranks) {}
    bool capturable() const override { return true; }   // NCCL collectives and p2p capture into graphs
    bool async_halo() const override { return true; }   // stream-ordered: may run on a side stream
    tca_status allreduce(double *dev, int count, cudaStream_t s) override
    {
        if (aborted_) return fail(TCA_ERR_NCCL, "NCCL communicator aborted after an earlier error");
        TCA_NCCL_TRY(nccl().AllReduce(dev, dev, (size_t)count, ncclFloat64, ncclSum, comm_, s));
        return TCA_OK;
    }
    // Host wait for `s` that does not hang on a dead peer: poll the stream and
    // the communicator's asynchronous error state; on an NCCL error or after
    // TCA_NCCL_TIMEOUT_S seconds (default 1800) the communicator is aborted
    // (its kernels return) and TCA_ERR_NCCL is reported.
    tca_status wait(cudaStream_t s) override
    {
        static const double limit = [] {
            const char *e = getenv("TCA_NCCL_TIMEOUT_S");
            return e ? atof(e) : 1800.0;
        }();
        timespec t0;
        clock_gettime(CLOCK_MONOTONIC, &t0);
        for (;;) {
            const cudaError_t q = cudaStreamQuery(s);
            if (q == cudaSuccess) return TCA_OK;
            if (q != cudaErrorNotReady) return cuda_fail(q, "stream (sharded solve)");
            int ae = ncclSuccess;
            if (nccl().CommGetAsyncError && nccl().CommGetAsyncError(comm_, &ae) == ncclSuccess &&
                ae != ncclSuccess && ae != ncclInProgress) {
                abort_comm();
                return nccl_fail(ae, "asynchronous NCCL error");
            }
            timespec t1;
            clock_gettime(CLOCK_MONOTONIC, &t1);
            if ((t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec) > limit) {
                abort_comm();
                return fail(TCA_ERR_NCCL, "sharded solve: no completion within TCA_NCCL_TIMEOUT_S (" +
                                              std::to_string(limit) + " s); communicator aborted");
            }
            const timespec nap{0, 50000};
            nanosleep(&nap, nullptr);
        }
    }
    tca_status halo(int which, char *ext, size_t slab_bytes, int64_t nloc, cudaStream_t s) override
    {
        (void)which;
        if (aborted_) return fail(TCA_ERR_NCCL, "NCCL communicator aborted after an earlier error");
        const size_t hb = (size_t)kHG * slab_bytes;   // 3 slabs
        char *own_first = ext + hb, *own_last = ext + (size_t)nloc * slab_bytes;   // [3, 6) and [nloc, nloc+3)
        char *ghost_lo = ext, *ghost_hi = ext + (size_t)(nloc + kHG) * slab_bytes;
        TCA_NCCL_TRY(nccl().GroupStart());
        if (rank_ > 0) {
            TCA_NCCL_TRY(nccl().Send(own_first, hb, 0 /*ncclInt8*/, rank_ - 1, comm_, s));
            TCA_NCCL_TRY(nccl().Recv(ghost_lo, hb, 0, rank_ - 1, comm_, s));
        }
        if (rank_ + 1 < nranks_) {
            TCA_NCCL_TRY(nccl().Send(own_last, hb, 0, rank_ + 1, comm_, s));
            TCA_NCCL_TRY(nccl().Recv(ghost_hi, hb, 0, rank_ + 1, comm_, s));
        }
        TCA_NCCL_TRY(nccl().GroupEnd());
        return TCA_OK;
    }

  private:
    void abort_comm()
    {
        if (!aborted_ && nccl().CommAbort) nccl().CommAbort(comm_);
        aborted_ = true;
    }
    void *comm_;
    int rank_, nranks_;
    bool aborted_ = false;
};

}  // namespace

// ---------------------------------------------------------------- local group
struct LocalGroup {
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    int64_t generation = 0;
    std::vector<double> vals;
    std::vector<char *> ext[2];   // per rank: [0] p buffer, [1] apply-input buffer (ghosted)
    std::vector<int64_t> nloc;
    std::vector<size_t> slab;

    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const int64_t g = generation;
        if (++arrived == n) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != g; });
        }
    }
};

namespace {

class LocalTransport final : public Transport {
  public:
    LocalTransport(LocalGroup *g, int rank) : g_(g), rank_(rank) {}
    tca_status allreduce(double *dev, int count, cudaStream_t s) override
    {
        std::vector<double> mine((size_t)count), sum((size_t)count, 0.0);
        TCA_CUDA_TRY(cudaMemcpyAsync(mine.data(), dev, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
        TCA_CUDA_TRY(cudaStreamSynchronize(s));
        {
            std::lock_guard<std::mutex> lk(g_->mu);
            if ((int)g_->vals.size() < g_->n * count) g_->vals.assign((size_t)g_->n * count, 0.0);
            for (int i = 0; i < count; ++i) g_->vals[(size_t)rank_ * count + i] = mine[i];
        }
        g_->barrier();
        for (int r = 0; r < g_->n; ++r)   // fixed rank order: identical bits on every shard
            for (int i = 0; i < count; ++i) sum[i] += g_->vals[(size_t)r * count + i];
        g_->barrier();
        TCA_CUDA_TRY(cudaMemcpyAsync(dev, sum.data(), sizeof(double) * count, cudaMemcpyHostToDevice, s));
        TCA_CUDA_TRY(cudaStreamSynchronize(s));
        return TCA_OK;
    }
    tca_status halo(int which, char *ext, size_t slab_bytes, int64_t nloc, cudaStream_t s) override
    {
        {
            std::lock_guard<std::mutex> lk(g_->mu);
            g_->ext[which][rank_] = ext;
            g_->nloc[rank_] = nloc;
            g_->slab[rank_] = slab_bytes;
        }
        TCA_CUDA_TRY(cudaStreamSynchronize(s));   // my own slabs are final
        g_->barrier();
        const size_t hb = (size_t)kHG * slab_bytes;
        if (rank_ > 0) {
            const char *nb = g_->ext[which][rank_ - 1];
            const int64_t nl = g_->nloc[rank_ - 1];
            TCA_CUDA_TRY(cudaMemcpy(ext, nb + (size_t)nl * slab_bytes, hb, cudaMemcpyDefault));
        }
        if (rank_ + 1 < g_->n) {
            const char *nb = g_->ext[which][rank_ + 1];
            TCA_CUDA_TRY(cudaMemcpy(ext + (size_t)(nloc + kHG) * slab_bytes, nb + hb, hb, cudaMemcpyDefault));
        }
        g_->barrier();   // neighbours finished reading my slabs
        return TCA_OK;
    }

  private:
    LocalGroup *g_;
    int rank_;
};

}  // namespace

Transport *make_transport(const tca_dist *d)
{
    if (!d || (!d->nccl_comm && !d->local_group)) return nullptr;
    if (d->local_group) {
        auto *g = reinterpret_cast<LocalGroup *>(d->local_group);
        return new LocalTransport(g, d->rank);
    }
    return new NcclTransport(d->nccl_comm, d->rank, d->nranks);
}

}  // namespace tca

using namespace tca;

extern "C" {

tca_status tca_shard_layout(int64_t n1, int64_t m1, const double *A1, int rank, int nranks, int64_t *out4)
{
    if (!A1 || !out4) return fail(TCA_ERR_INVALID_ARG, "A1 and out4 must be non-NULL");
    if (n1 < 1 || m1 < 1) return fail(TCA_ERR_SHAPE, "n1 and m1 must be >= 1");
    return shard_layout(n1, A1, m1, rank, nranks, out4);
}

tca_status tca_nccl_get_unique_id(void *uid128)
{
    if (!uid128) return fail(TCA_ERR_INVALID_ARG, "uid128 is NULL");
    if (!nccl().ok) return fail(TCA_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId_t id;
    TCA_NCCL_TRY(nccl().GetUniqueId(&id));
    memcpy(uid128, &id, sizeof(id));
    return TCA_OK;
}

tca_status tca_nccl_comm_create(void **comm, int nranks, const void *uid128, int rank)
{
    if (!comm || !uid128) return fail(TCA_ERR_INVALID_ARG, "comm and uid128 must be non-NULL");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TCA_ERR_INVALID_ARG, "bad rank / nranks");
    if (!nccl().ok) return fail(TCA_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId_t id;
    memcpy(&id, uid128, sizeof(id));
    ncclComm_t c = nullptr;
    TCA_NCCL_TRY(nccl().CommInitRank(&c, nranks, id, rank));
    *comm = c;
    return TCA_OK;
}

void tca_nccl_comm_destroy(void *comm)
{
    if (comm && nccl().ok) nccl().CommDestroy(comm);
}

tca_status tca_local_group_create(void **group, int nranks)
{
    if (!group) return fail(TCA_ERR_INVALID_ARG, "group is NULL");
    if (nranks < 1) return fail(TCA_ERR_INVALID_ARG, "nranks must be >= 1");
    auto *g = new LocalGroup();
    g->n = nranks;
    for (auto &e : g->ext) e.assign(nranks, nullptr);
    g->nloc.assign(nranks, 0);
    g->slab.assign(nranks, 0);
    *group = g;
    return TCA_OK;
}

void tca_local_group_destroy(void *group) { delete reinterpret_cast<LocalGroup *>(group); }

}  // extern "C"
