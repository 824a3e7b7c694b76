// comm.cu -- NCCL and loopback transports of the exchange layer (comm.cuh).
#include "comm.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>

void cd_loopback::barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t gen = generation;
    if (++arrived == nranks) {
        arrived = 0;
        ++generation;
        cv.notify_all();
    } else {
        cv.wait(lk, [&] { return generation != gen; });
    }
}

namespace cdk {

// ---------------------------------------------------------------------------
// NCCL (dlopen'ed)
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};

NcclApi &nccl() {
    static NcclApi api;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (api.loaded)
        return api;
    // the soname torch already loaded (if any) is reused by the dynamic loader
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h)
        h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h)
        fail(CD_ENCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char *name) {
        void *p = dlsym(h, name);
        if (!p)
            fail(CD_ENCCL, std::string("libnccl lacks ") + name);
        return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.loaded = true;
    return api;
}

#define CD_NCCL(x)                                                                                   \
    do {                                                                                             \
        ncclResult_t r_ = (x);                                                                       \
        if (r_ != ncclSuccess)                                                                       \
            ::cdk::fail(CD_ENCCL, std::string(#x) + ": " + nccl().GetErrorString(r_));               \
    } while (0)

class NcclComm final : public Comm {
  public:
    NcclComm(int nranks, int r, const uint8_t id[128]) {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        CD_NCCL(nccl().CommInitRank(&comm_, nranks, uid, r));
        rank = r;
        size = nranks;
    }
    ~NcclComm() override {
        if (comm_)
            nccl().CommDestroy(comm_);
    }
    const char *kind() const override { return "nccl"; }
    void allgather(cd_ctx *ctx, const void *send, void *recv, size_t bytes) override {
        CD_NCCL(nccl().AllGather(send, recv, bytes, ncclInt8, comm_, ctx->stream));
    }
    void allreduce_sum_i64(cd_ctx *ctx, int64_t *buf, size_t count) override {
        CD_NCCL(nccl().AllReduce(buf, buf, count, ncclInt64, ncclSum, comm_, ctx->stream));
    }
    void allreduce_sum_f64(cd_ctx *ctx, double *buf, size_t count) override {
        CD_NCCL(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm_, ctx->stream));
    }
    void broadcast(cd_ctx *ctx, void *buf, size_t bytes, int root) override {
        CD_NCCL(nccl().Broadcast(buf, buf, bytes, ncclInt8, root, comm_, ctx->stream));
    }
    void alltoallv(cd_ctx *ctx, const void *send, const size_t *sdispl, const size_t *scount, void *recv,
                   const size_t *rdispl, const size_t *rcount) override {
        CD_NCCL(nccl().GroupStart());
        for (int p = 0; p < size; ++p) {
            if (scount[p])
                CD_NCCL(nccl().Send(static_cast<const unsigned char *>(send) + sdispl[p], scount[p], ncclInt8, p,
                                    comm_, ctx->stream));
            if (rcount[p])
                CD_NCCL(nccl().Recv(static_cast<unsigned char *>(recv) + rdispl[p], rcount[p], ncclInt8, p, comm_,
                                    ctx->stream));
        }
        CD_NCCL(nccl().GroupEnd());
    }

  private:
    ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------------------
// loopback (host threads, one device)
// ---------------------------------------------------------------------------
class LoopbackComm final : public Comm {
  public:
    LoopbackComm(cd_loopback *g, int r) : g_(g) {
        rank = r;
        size = g->nranks;
    }
    const char *kind() const override { return "loopback"; }
    void allgather(cd_ctx *ctx, const void *send, void *recv, size_t bytes) override {
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        publish(send);
        for (int r = 0; r < size; ++r)
            if (bytes && static_cast<unsigned char *>(recv) + r * bytes != g_->slot[r])  // in-place block
                CD_CUDA(cudaMemcpyAsync(static_cast<unsigned char *>(recv) + r * bytes, g_->slot[r], bytes,
                                        cudaMemcpyDeviceToDevice, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        g_->barrier();  // peers may reuse their send buffers after this
    }
    template <class T>
    void allreduce(cd_ctx *ctx, T *buf, size_t count) {
        const size_t bytes = count * sizeof(T);
        std::vector<unsigned char> &mine = g_->host[rank];
        mine.resize(bytes);
        CD_CUDA(cudaMemcpyAsync(mine.data(), buf, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        publish(nullptr);
        // every rank sums in rank order: identical results on all ranks
        std::vector<T> acc(count, T(0));
        for (int r = 0; r < size; ++r) {
            const T *p = reinterpret_cast<const T *>(g_->host[r].data());
            for (size_t i = 0; i < count; ++i)
                acc[i] += p[i];
        }
        g_->barrier();
        CD_CUDA(cudaMemcpyAsync(buf, acc.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    void allreduce_sum_i64(cd_ctx *ctx, int64_t *buf, size_t count) override { allreduce(ctx, buf, count); }
    void allreduce_sum_f64(cd_ctx *ctx, double *buf, size_t count) override { allreduce(ctx, buf, count); }
    void broadcast(cd_ctx *ctx, void *buf, size_t bytes, int root) override {
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        publish(buf);
        if (rank != root && bytes)
            CD_CUDA(cudaMemcpyAsync(buf, g_->slot[root], bytes, cudaMemcpyDeviceToDevice, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        g_->barrier();
    }
    void alltoallv(cd_ctx *ctx, const void *send, const size_t *sdispl, const size_t *scount, void *recv,
                   const size_t *rdispl, const size_t *rcount) override {
        // peers pull their blocks from the published send buffers; the send
        // displacements travel as a host array next to the device pointer
        struct Pub {
            const void *send;
            const size_t *sdispl;
        } mine{send, sdispl};
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        publish(&mine);
        for (int p = 0; p < size; ++p) {
            const Pub *pp = static_cast<const Pub *>(g_->slot[p]);
            if (rcount[p])
                CD_CUDA(cudaMemcpyAsync(static_cast<unsigned char *>(recv) + rdispl[p],
                                        static_cast<const unsigned char *>(pp->send) + pp->sdispl[rank], rcount[p],
                                        cudaMemcpyDeviceToDevice, ctx->stream));
        }
        (void)scount;
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        g_->barrier();  // peers may reuse their send buffers (and `mine` goes out of scope) after this
    }

  private:
    void publish(const void *p) {
        {
            std::lock_guard<std::mutex> lk(g_->m);
            g_->slot[rank] = p;
        }
        g_->barrier();
    }
    cd_loopback *g_;
};

__global__ void k_shard_bounds(int64_t n, const int64_t *off, int nranks, int64_t *bounds) {
    const int r = threadIdx.x;
    if (r > nranks)
        return;
    const int64_t D = off[n];
    if (r == 0 || r == nranks) {
        bounds[r] = r == 0 ? 0 : n;
        return;
    }
    // first u with off[u] >= D * r / G  (lower_bound over off[0..n])
    const int64_t target = static_cast<int64_t>((static_cast<__int128>(D) * r) / nranks);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (off[mid] < target)
            lo = mid + 1;
        else
            hi = mid;
    }
    bounds[r] = lo;
}

}  // namespace

Comm *comm_nccl_create(int nranks, int rank, const uint8_t id[128]) { return new NcclComm(nranks, rank, id); }

Comm *comm_loopback_create(cd_loopback *group, int rank) { return new LoopbackComm(group, rank); }

void nccl_unique_id(uint8_t out[128]) {
    ncclUniqueId uid;
    CD_NCCL(nccl().GetUniqueId(&uid));
    std::memcpy(out, &uid, sizeof(uid));
}

void shard_bounds_host(int64_t n, const int64_t *off, int nranks, int64_t *bounds) {
    const int64_t D = off[n];
    bounds[0] = 0;
    bounds[nranks] = n;
    for (int r = 1; r < nranks; ++r) {
        const int64_t target = static_cast<int64_t>((static_cast<__int128>(D) * r) / nranks);
        bounds[r] = std::lower_bound(off, off + n, target) - off;
    }
}

void shard_bounds_dev(cd_ctx *ctx, int64_t n, const int64_t *off_dev, int nranks, int64_t *bounds) {
    DBuf<int64_t> b(ctx, nranks + 1);
    CD_LAUNCH(ctx, "shard", k_shard_bounds, 1, 32 * ((nranks + 32) / 32), 0, n, off_dev, nranks, b.p);
    CD_CUDA(cudaMemcpyAsync(bounds, b.p, (nranks + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace cdk
