// comm.cuh -- the exchange layer of the sharded drivers.
//
// The sharded PLP / PLM drivers need four collectives, all on device buffers
// and ordered on the context stream:
//   allgather   every rank's fixed-size block, concatenated in rank order
//               (per-bucket move lists, coarse-graph partials, EPP bases)
//   allreduce   sum of int64 / fp64 vectors (move counts, modularity terms)
//   broadcast   from a root rank
// Two transports implement them:
//   * NCCL (one process per GPU; libnccl is dlopen'ed when a communicator is
//     attached, so the library itself has no link-time NCCL dependency and
//     shares the process's already-loaded libnccl.so.2 with torch);
//   * loopback: ranks are host threads of one process, each with its own
//     cd_ctx on the same device; a host barrier orders them and peers' device
//     buffers are copied with stream-ordered D2D copies.  No kernel ever waits
//     on another rank -- it is the one-GPU emulation of the multi-rank path
//     (B200_PROFILING.md: never run mutually waiting kernels on one GPU).
#pragma once

#include <condition_variable>
#include <mutex>

#include "common.cuh"

struct cd_loopback {
    int nranks = 1;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<const void *> slot;
    std::vector<std::vector<unsigned char>> host;  // allreduce staging per rank
    void barrier();
};

namespace cdk {

class Comm {
  public:
    virtual ~Comm() = default;
    int rank = 0, size = 1;
    virtual const char *kind() const = 0;
    // recv[r * bytes, (r+1) * bytes) = rank r's send block
    virtual void allgather(cd_ctx *ctx, const void *send, void *recv, size_t bytes) = 0;
    virtual void allreduce_sum_i64(cd_ctx *ctx, int64_t *buf, size_t count) = 0;
    virtual void allreduce_sum_f64(cd_ctx *ctx, double *buf, size_t count) = 0;
    virtual void broadcast(cd_ctx *ctx, void *buf, size_t bytes, int root) = 0;
    // personalised exchange: bytes [sdispl[p], +scount[p]) of send go to rank
    // p, which receives them at [rdispl[me], +rcount[me]) of its recv (host
    // arrays of G byte counts / offsets; every pair's counts must agree)
    virtual void alltoallv(cd_ctx *ctx, const void *send, const size_t *sdispl, const size_t *scount, void *recv,
                           const size_t *rdispl, const size_t *rcount) = 0;
};

Comm *comm_nccl_create(int nranks, int rank, const uint8_t id[128]);
Comm *comm_loopback_create(cd_loopback *group, int rank);
void nccl_unique_id(uint8_t out[128]);

// world of a context (1 when no communicator is attached)
inline int world_size(const cd_ctx *ctx) { return ctx->comm ? ctx->comm->size : 1; }
inline int world_rank(const cd_ctx *ctx) { return ctx->comm ? ctx->comm->rank : 0; }

// Degree-balanced 1D ownership: rank r owns nodes [b[r], b[r+1]), chosen so
// each range holds about D*r/G CSR entries (binary search on off[]).
void shard_bounds_host(int64_t n, const int64_t *off_host, int nranks, int64_t *bounds);
void shard_bounds_dev(cd_ctx *ctx, int64_t n, const int64_t *off_dev, int nranks, int64_t *bounds);
cd_graph *graph_from_rows_dev(cd_ctx *ctx, int64_t n, const int64_t *off, int64_t lo, int64_t hi,
                              const int32_t *col, const float *w);

}  // namespace cdk
