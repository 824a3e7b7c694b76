// generators.cu -- seeded synthetic graphs on the device.
//   planted partition: bit-exact generate_planted (H/generator.hpp:52-104)
//   R-MAT, LFR-shaped: new (the reference has none, R/SPEC.md:8); their exact
//   definition is ported in oracle/commdet_oracle.c (cdo_generate_rmat /
//   cdo_generate_lfr) so the CPU oracle sees identical bytes.
#include <cmath>
#include <cstring>

#include "comm.cuh"
#include "rows.cuh"

namespace cdk {

#define RMAT_SALT 0x524d41542d4b4559ULL
#define WEIGHT_SALT 0x5745494748542d4bULL
#define LFR_DEG_SALT 0x4c46522d44454731ULL
#define LFR_COM_SALT 0x4c46522d434f4d31ULL
#define LFR_ASG_SALT 0x4c46522d41534731ULL
#define LFR_INT_SALT 0x4c46522d494e5431ULL
#define LFR_EXT_SALT 0x4c46522d45585431ULL

// ---------------------------------------------------------------------------
// planted partition
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t planted_block(int64_t u, int64_t n, int64_t k) {
    // (u * k) / n with a 128-bit product (H/generator.hpp:48-50)
    const unsigned long long a = static_cast<unsigned long long>(u), b = static_cast<unsigned long long>(k);
    const unsigned long long lo = a * b, hi = __umul64hi(a, b);
    if (hi == 0)
        return static_cast<int64_t>(lo / static_cast<unsigned long long>(n));
    // rare: long division of (hi:lo) by n
    unsigned __int128 p = (static_cast<unsigned __int128>(hi) << 64) | lo;
    return static_cast<int64_t>(p / static_cast<unsigned long long>(n));
}

__device__ __forceinline__ bool planted_pair(uint64_t key, int64_t v, double p) {
    // row_uniform(key, v) < p  (H/generator.hpp:35-37, :85)
    const double r = static_cast<double>(splitmix64(key ^ splitmix64(static_cast<uint64_t>(v))) >> 11) * 0x1.0p-53;
    return p > 0.0 && r < p;
}

// warp per row u, lanes stride over v > u; pass 0 counts, pass 1 writes
__global__ void __launch_bounds__(256) k_planted(int64_t n, int64_t k, double p_in, double p_out, uint64_t seed,
                                                 int pass, int64_t *cnt, const int64_t *pre, int32_t *eu,
                                                 int32_t *ev) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t u = gw; u < n; u += nw) {
        const int64_t bu = planted_block(u, n, k);
        int64_t v_end = n;
        if (p_out == 0.0) {
            // first v with block(v) > bu: ceil((bu+1) n / k)  (:75-80)
            const unsigned __int128 num = static_cast<unsigned __int128>(bu + 1) * static_cast<unsigned __int128>(n);
            v_end = static_cast<int64_t>((num + static_cast<unsigned __int128>(k - 1)) / static_cast<unsigned __int128>(k));
            if (v_end > n)
                v_end = n;
        }
        const uint64_t key = splitmix64(seed ^ splitmix64(static_cast<uint64_t>(u)));
        int64_t c = 0;
        int64_t base = pass ? pre[u] : 0;
        for (int64_t v0 = u + 1; v0 < v_end; v0 += 32) {
            const int64_t v = v0 + lane;
            bool e = false;
            if (v < v_end) {
                const double p = planted_block(v, n, k) == bu ? p_in : p_out;
                e = planted_pair(key, v, p);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, e);
            if (pass && e) {
                const int64_t pos = base + c + __popc(m & lanemask_lt());
                eu[pos] = static_cast<int32_t>(u);
                ev[pos] = static_cast<int32_t>(v);
            }
            c += __popc(m);
        }
        if (!pass && lane == 0)
            cnt[u] = c;
    }
}

struct I64Gen {
    const int64_t *a;
    __device__ int64_t operator()(int64_t i) const { return a[i]; }
};

cd_graph *generate_planted_dev(cd_ctx *ctx, int64_t n, int64_t k, double p_in, double p_out, uint64_t seed,
                               int32_t *truth_dev) {
    if (k < 1 || (n > 0 && k > n))
        fail(CD_EINVAL, "planted partition: need 1 <= k <= n");
    if (p_out < 0.0 || p_in > 1.0 || p_out > p_in)
        fail(CD_EINVAL, "planted partition: need 0 <= p_out <= p_in <= 1");
    DBuf<int64_t> cnt(ctx, std::max<int64_t>(n, 1)), pre(ctx, n + 1);
    const int grid = grid_for(n, 8, ctx->num_sms * 16);
    if (n > 0)
        CD_LAUNCH(ctx, "generate", k_planted, grid, 256, 0, n, k, p_in, p_out, seed, 0, cnt.p,
                  static_cast<const int64_t *>(nullptr), static_cast<int32_t *>(nullptr),
                  static_cast<int32_t *>(nullptr));
    exclusive_scan<int64_t>(ctx, n, I64Gen{cnt.p}, pre.p, pre.p + n);
    int64_t m = 0;
    CD_CUDA(cudaMemcpyAsync(&m, pre.p + n, sizeof(m), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    DBuf<int32_t> eu(ctx, std::max<int64_t>(m, 1)), ev(ctx, std::max<int64_t>(m, 1));
    if (n > 0)
        CD_LAUNCH(ctx, "generate", k_planted, grid, 256, 0, n, k, p_in, p_out, seed, 1, cnt.p,
                  static_cast<const int64_t *>(pre.p), eu.p, ev.p);
    if (truth_dev && n > 0) {
        std::vector<int32_t> t(n);
        for (int64_t u = 0; u < n; ++u)
            t[u] = static_cast<int32_t>((static_cast<unsigned __int128>(u) * static_cast<uint64_t>(k)) /
                                        static_cast<uint64_t>(n));
        CD_CUDA(cudaMemcpyAsync(truth_dev, t.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return graph_from_pairs(ctx, n, m, eu.p, ev.p, nullptr, DUP_ERROR);
}

// ---------------------------------------------------------------------------
// R-MAT
// ---------------------------------------------------------------------------
// Draw e of the R-MAT stream: `scale` quadrant choices from the 32-bit
// halves of splitmix64 words (the oracle's cdo_generate_rmat).  Canonical
// (u < v); false for a self-loop.
struct RmatSpec {
    int scale;
    uint64_t key, ta, tab, tabc;
};

__device__ __forceinline__ bool rmat_draw(const RmatSpec &R, int64_t e, uint32_t &u, uint32_t &v) {
    uint32_t a = 0, b = 0;
    for (int lvl = 0; lvl < R.scale; lvl += 2) {
        const uint64_t r = splitmix64(R.key ^ (static_cast<uint64_t>(e) * 16u + static_cast<uint64_t>(lvl >> 1)));
        for (int h = 0; h < 2 && lvl + h < R.scale; ++h) {
            const uint64_t r32 = h ? (r >> 32) : (r & 0xffffffffu);
            const uint32_t bu = r32 >= R.tab, bv = (r32 >= R.ta && r32 < R.tab) || r32 >= R.tabc;
            a = (a << 1) | bu;
            b = (b << 1) | bv;
        }
    }
    u = a < b ? a : b;
    v = a < b ? b : a;
    return a != b;
}

// pass 1: raw adjacency length of every node (both directions, duplicates
// included) -- an upper bound of its degree and the chunking / ownership key
__global__ void k_rmat_degree(int64_t M, RmatSpec R, int32_t *deg) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < M;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t u, v;
        if (rmat_draw(R, e, u, v)) {
            atomicAdd(&deg[u], 1);
            atomicAdd(&deg[v], 1);
        }
    }
}

// pass 2 (per row chunk [lo, hi)): regenerate the stream and scatter the raw
// adjacency of the chunk's rows
__global__ void k_rmat_scatter(int64_t M, RmatSpec R, int64_t lo, int64_t hi, unsigned long long *cursor,
                               int32_t *rk) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < M;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t u, v;
        if (!rmat_draw(R, e, u, v))
            continue;
        if (u >= lo && u < hi)
            rk[atomicAdd(&cursor[u - lo], 1ULL)] = static_cast<int32_t>(v);
        if (v >= lo && v < hi)
            rk[atomicAdd(&cursor[v - lo], 1ULL)] = static_cast<int32_t>(u);
    }
}

// global statistics of a row shard from the replicated node volumes
__global__ void k_vol_stats(int64_t n, const double *vol, unsigned long long *acc) {
    unsigned long long iso = 0, mx = 0;
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double x = vol[u];
        iso += x == 0.0;
        mx = max(mx, static_cast<unsigned long long>(__double_as_longlong(x)));  // x >= 0: bits are monotone
    }
    iso = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(iso));
    for (int o = 16; o > 0; o >>= 1)
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane_id() == 0) {
        atomicAdd(&acc[0], iso);
        atomicMax(&acc[1], mx);
    }
}
__global__ void k_pair_weights(int64_t n, const int64_t *off, const int32_t *col, uint64_t wkey, float *w) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t u = gw; u < n; u += nw)
        for (int64_t i = off[u] + lane; i < off[u + 1]; i += 32) {
            const uint64_t a = static_cast<uint64_t>(u), b = static_cast<uint64_t>(col[i]);
            const uint64_t pair = a < b ? ((a << 32) | b) : ((b << 32) | a);
            // (k+1) * 2^-24, k = top 24 bits: uniform in (0, 1], exact in fp32
            w[i] = static_cast<float>(static_cast<double>((splitmix64(wkey ^ pair) >> 40) + 1) * 0x1.0p-24);
        }
}

// Raw entries per build chunk: the row engine needs ~20 B of scratch per raw
// entry (raw list, hash keys and values, chunk columns), so a chunk of 2^30
// entries stays near 24 GB whatever the scale (C5: 8.6e9 entries, 9 chunks).
constexpr int64_t RMAT_CHUNK_ENTRIES = int64_t(1) << 30;

// The R-MAT graph, built in row chunks: pass 1 counts every node's raw
// adjacency; each chunk of rows regenerates the stream, scatters its rows'
// raw adjacency and reduces it (duplicates merged) with the row engine into
// its slice of the CSR.  With `shard`, rank r of the context's communicator
// builds only the rows it owns -- ranges splitting the raw adjacency evenly
// (comm.cuh) -- with empty rows elsewhere and the global per-node state.
cd_graph *generate_rmat_dev(cd_ctx *ctx, int scale, int edge_factor, double a, double b, double c, int weighted,
                            uint64_t seed, bool shard) {
    if (scale < 1 || scale > 30 || edge_factor < 1)
        fail(CD_EINVAL, "rmat: need 1 <= scale <= 30 and edge_factor >= 1");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0)
        fail(CD_EINVAL, "rmat: probabilities must be >= 0 with a + b + c <= 1");
    const int64_t n = int64_t(1) << scale;
    const int64_t M = static_cast<int64_t>(edge_factor) << scale;
    RmatSpec R;
    R.scale = scale;
    R.ta = static_cast<uint64_t>(a * 4294967296.0);
    R.tab = static_cast<uint64_t>((a + b) * 4294967296.0);
    R.tabc = static_cast<uint64_t>((a + b + c) * 4294967296.0);
    R.key = splitmix64(seed ^ RMAT_SALT);
    const int G = shard ? world_size(ctx) : 1, rank = shard ? world_rank(ctx) : 0;
    const int gen_grid = ctx->num_sms * 16;

    DBuf<int64_t> pre(ctx, n + 1);
    {
        DBuf<int32_t> deg(ctx, n);
        deg.zero();
        CD_LAUNCH(ctx, "generate", k_rmat_degree, gen_grid, 256, 0, M, R, deg.p);
        exclusive_scan<int64_t>(ctx, n, ArrayGen<int32_t>{deg.p}, pre.p, pre.p + n);
    }
    int64_t lo = 0, hi = n;
    if (G > 1) {
        std::vector<int64_t> bnd(G + 1);
        shard_bounds_dev(ctx, n, pre.p, G, bnd.data());
        lo = bnd[rank];
        hi = bnd[rank + 1];
    }
    int64_t praw[2];
    CD_CUDA(cudaMemcpyAsync(&praw[0], pre.p + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaMemcpyAsync(&praw[1], pre.p + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t F = praw[1] - praw[0];
    const std::vector<int64_t> cut =
        split_rows(ctx, pre.p, lo, hi, env_i64("CD_BUILD_CHUNK_ENTRIES", RMAT_CHUNK_ENTRIES));
    const int nchunks = static_cast<int>(cut.size()) - 1;

    auto *g = new cd_graph();
    try {
        g->ctx = ctx;
        g->n = n;
        g->off.alloc(ctx, n + 1);
        g->col.alloc(ctx, std::max<int64_t>(F, 1));  // raw bound; the merged rows fill a prefix
        if (lo > 0)
            CD_LAUNCH(ctx, "build.prep", k_fill_i64, grid_for(lo, 256, ctx->num_sms * 8), 256, 0, lo, int64_t(0), g->off.p);
        int64_t D = 0;
        for (int k = 0; k < nchunks; ++k) {
            const int64_t a0 = cut[k], a1 = cut[k + 1], rows = a1 - a0;
            if (rows == 0)
                continue;
            int64_t pr[2];
            CD_CUDA(cudaMemcpyAsync(&pr[0], pre.p + a0, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
            CD_CUDA(cudaMemcpyAsync(&pr[1], pre.p + a1, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
            CD_CUDA(cudaStreamSynchronize(ctx->stream));
            const int64_t Fc = pr[1] - pr[0];
            DBuf<int64_t> fpre(ctx, rows + 1);
            CD_LAUNCH(ctx, "build.prep", k_rebase, grid_for(rows + 1, 256, ctx->num_sms * 8), 256, 0, rows + 1,
                      static_cast<const int64_t *>(pre.p + a0), pr[0], int64_t(0), fpre.p);
            DBuf<int32_t> rk(ctx, std::max<int64_t>(Fc, 1));
            {
                DBuf<int64_t> cursor(ctx, rows);
                CD_CUDA(cudaMemcpyAsync(cursor.p, fpre.p, rows * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                                        ctx->stream));
                CD_LAUNCH(ctx, "generate", k_rmat_scatter, gen_grid, 256, 0, M, R, a0, a1,
                          reinterpret_cast<unsigned long long *>(cursor.p), rk.p);
            }
            DBuf<int64_t> off2;
            DBuf<int32_t> col2;
            DBuf<float> w2;
            bool want_w = false;
            const int64_t Dc = run_row_engine(ctx, SrcFlat{fpre.p, rk.p, nullptr}, rows, fpre.p, Fc, n, DUP_ONE,
                                              want_w, off2, col2, w2, nullptr, "build");
            CD_LAUNCH(ctx, "build.prep", k_rebase, grid_for(rows, 256, ctx->num_sms * 8), 256, 0, rows,
                      static_cast<const int64_t *>(off2.p), int64_t(0), D, g->off.p + a0);
            if (Dc)
                CD_CUDA(cudaMemcpyAsync(g->col.p + D, col2.p, Dc * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                        ctx->stream));
            D += Dc;
        }
        CD_LAUNCH(ctx, "build.prep", k_fill_i64, grid_for(n + 1 - hi, 256, ctx->num_sms * 8), 256, 0, n + 1 - hi, D,
                  g->off.p + hi);
        pre.release();
        g->D = D;
        if (weighted) {
            g->w.alloc(ctx, std::max<int64_t>(D, 1));
            const uint64_t wkey = splitmix64(seed ^ WEIGHT_SALT);
            CD_LAUNCH(ctx, "generate", k_pair_weights, grid_for(n, 8, ctx->num_sms * 16), 256, 0, n,
                      static_cast<const int64_t *>(g->off.p), static_cast<const int32_t *>(g->col.p), wkey, g->w.p);
            g->weighted = true;
        }
        graph_finalize(ctx, g);
        if (G > 1)
            shard_globalize(ctx, g, lo, hi);
    } catch (...) {
        delete g;
        throw;
    }
    return g;
}

// Turn a graph holding only rows [lo, hi) (finalized locally) into a row
// shard: node volumes and loops summed over the ranks (each node's row lives
// on one rank), m / total summed (each undirected entry is counted by the
// rank owning its smaller endpoint), the maxima and isolated count taken from
// the global volumes.
void shard_globalize(cd_ctx *ctx, cd_graph *g, int64_t lo, int64_t hi) {
    Comm *cm = ctx->comm;
    const int G = world_size(ctx);
    const int64_t n = g->n;
    struct Local {
        int64_t D, m, max_degree, nonint;
        double total;
    } mine{g->D, g->m, g->max_degree, g->int_weights ? 0 : 1, g->total};
    DBuf<Local> all(ctx, G), one(ctx, 1);
    CD_CUDA(cudaMemcpyAsync(one.p, &mine, sizeof(Local), cudaMemcpyHostToDevice, ctx->stream));
    cm->allgather(ctx, one.p, all.p, sizeof(Local));
    std::vector<Local> h(G);
    CD_CUDA(cudaMemcpyAsync(h.data(), all.p, G * sizeof(Local), cudaMemcpyDeviceToHost, ctx->stream));
    if (n) {
        cm->allreduce_sum_f64(ctx, g->vol.p, n);
        cm->allreduce_sum_f64(ctx, g->loop.p, n);
    }
    DBuf<unsigned long long> acc(ctx, 2);
    acc.zero();
    if (n)
        CD_LAUNCH(ctx, "finalize", k_vol_stats, grid_for(n, 256, ctx->num_sms * 8), 256, 0, n,
                  static_cast<const double *>(g->vol.p), acc.p);
    unsigned long long ha[2];
    CD_CUDA(cudaMemcpyAsync(ha, acc.p, sizeof(ha), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    int64_t Dg = 0, m = 0, maxd = 0;
    bool nonint = false;
    double total = 0.0;
    for (const Local &l : h) {
        Dg += l.D;
        m += l.m;
        maxd = std::max(maxd, l.max_degree);
        total += l.total;
    }
    // integral weights: every rank's rows integral and the global max volume
    // below 2^31 (a local overflow implies the global one)
    for (const Local &l : h)
        nonint |= l.nonint != 0;
    double max_vol;
    std::memcpy(&max_vol, &ha[1], sizeof(double));
    g->isolated = static_cast<int64_t>(ha[0]);
    g->max_vol = max_vol;
    g->m = m;
    g->total = total;
    g->max_degree = maxd;
    g->int_weights = !nonint && max_vol < 2147483648.0;
    g->rows_local = true;
    g->shard_rank = world_rank(ctx);
    g->shard_size = G;
    g->own_lo = lo;
    g->own_hi = hi;
    g->D_global = Dg;
}

// ---------------------------------------------------------------------------
// LFR-shaped: host setup (degrees, community sizes, assignment) restated
// exactly like cdo_generate_lfr; device Chung-Lu style edge sampling.
// ---------------------------------------------------------------------------
static double unit53(uint64_t r) { return static_cast<double>(r >> 11) * 0x1.0p-53; }

static int64_t cdf_pick(const std::vector<double> &cdf, double u) {
    int64_t lo = 0, hi = static_cast<int64_t>(cdf.size()) - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (u < cdf[mid])
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ int64_t prefix_find(const int64_t *prefix, int64_t len, int64_t s) {
    int64_t lo = 0, hi = len - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= s)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

__global__ void k_lfr_internal(int64_t m_int, int64_t C, uint64_t ki, const int64_t *eoff, const int64_t *coff,
                               const int64_t *vin, const int64_t *kin_prefix, const int32_t *members, int32_t *eu,
                               int32_t *ev, int32_t *count) {
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < m_int;
         base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e = base + threadIdx.x;
        bool ok = e < m_int;
        int32_t a = 0, b = 0;
        if (ok) {
            const int64_t j = prefix_find(eoff, C + 1, e);
            const int64_t len = coff[j + 1] - coff[j];
            const uint64_t r1 = splitmix64(ki ^ (2u * static_cast<uint64_t>(e)));
            const uint64_t r2 = splitmix64(ki ^ (2u * static_cast<uint64_t>(e) + 1u));
            const int64_t s1 = static_cast<int64_t>(__umul64hi(r1, static_cast<uint64_t>(vin[j])));
            const int64_t s2 = static_cast<int64_t>(__umul64hi(r2, static_cast<uint64_t>(vin[j])));
            a = members[coff[j] + prefix_find(kin_prefix + coff[j], len, s1)];
            b = members[coff[j] + prefix_find(kin_prefix + coff[j], len, s2)];
            ok = a != b;
        }
        const int32_t pos = warp_append(count, ok);
        if (ok) {
            eu[pos] = a < b ? a : b;
            ev[pos] = a < b ? b : a;
        }
    }
}

__global__ void k_lfr_external(int64_t m_ext, int64_t n, uint64_t ke, int64_t kout_total, const int64_t *kout_prefix,
                               const int32_t *comm, int32_t *eu, int32_t *ev, int32_t *count) {
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < m_ext;
         base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e = base + threadIdx.x;
        bool ok = false;
        int32_t a = 0, b = 0;
        if (e < m_ext) {
            for (uint64_t att = 0; att < 8; ++att) {
                const uint64_t r1 = splitmix64(ke ^ (static_cast<uint64_t>(e) * 16u + 2u * att));
                const uint64_t r2 = splitmix64(ke ^ (static_cast<uint64_t>(e) * 16u + 2u * att + 1u));
                const int64_t s1 = static_cast<int64_t>(__umul64hi(r1, static_cast<uint64_t>(kout_total)));
                const int64_t s2 = static_cast<int64_t>(__umul64hi(r2, static_cast<uint64_t>(kout_total)));
                a = static_cast<int32_t>(prefix_find(kout_prefix, n, s1));
                b = static_cast<int32_t>(prefix_find(kout_prefix, n, s2));
                if (comm[a] != comm[b]) {
                    ok = true;
                    break;
                }
            }
        }
        const int32_t pos = warp_append(count, ok);
        if (ok) {
            eu[pos] = a < b ? a : b;
            ev[pos] = a < b ? b : a;
        }
    }
}

template <class T>
static T *upload(cd_ctx *ctx, DBuf<T> &buf, const std::vector<T> &v) {
    buf.alloc(ctx, std::max<size_t>(v.size(), 1));
    if (!v.empty())
        CD_CUDA(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    return buf.p;
}

cd_graph *generate_lfr_dev(cd_ctx *ctx, const cd_lfr_spec &sp, uint64_t seed, int32_t *truth_dev) {
    const int64_t n = sp.n;
    if (n < 2 || sp.max_degree < 1 || sp.min_community < 1 || sp.max_community < sp.min_community || sp.mu < 0.0 ||
        sp.mu > 1.0)
        fail(CD_EINVAL, "lfr: invalid specification");
    const int32_t kmax = sp.max_degree;
    int32_t kmin = 1;
    double best_err = 1e300;
    for (int32_t k0 = 1; k0 <= kmax; ++k0) {
        double s0 = 0.0, s1 = 0.0;
        for (int32_t k = k0; k <= kmax; ++k) {
            const double p = std::pow(static_cast<double>(k), -sp.tau1);
            s0 += p;
            s1 += p * static_cast<double>(k);
        }
        const double err = std::fabs(s1 / s0 - sp.avg_degree);
        if (err < best_err) {
            best_err = err;
            kmin = k0;
        }
    }
    const int64_t nk = kmax - kmin + 1, ns = sp.max_community - sp.min_community + 1;
    std::vector<double> cdf_k(nk), cdf_s(ns);
    {
        double tot = 0.0, acc = 0.0;
        for (int64_t i = 0; i < nk; ++i)
            tot += std::pow(static_cast<double>(kmin + i), -sp.tau1);
        for (int64_t i = 0; i < nk; ++i) {
            acc += std::pow(static_cast<double>(kmin + i), -sp.tau1);
            cdf_k[i] = acc / tot;
        }
        cdf_k[nk - 1] = 2.0;
        tot = 0.0;
        acc = 0.0;
        for (int64_t i = 0; i < ns; ++i)
            tot += std::pow(static_cast<double>(sp.min_community + i), -sp.tau2);
        for (int64_t i = 0; i < ns; ++i) {
            acc += std::pow(static_cast<double>(sp.min_community + i), -sp.tau2);
            cdf_s[i] = acc / tot;
        }
        cdf_s[ns - 1] = 2.0;
    }
    std::vector<int32_t> deg(n), kin(n);
    const uint64_t kd = splitmix64(seed ^ LFR_DEG_SALT);
    for (int64_t i = 0; i < n; ++i)
        deg[i] = kmin + static_cast<int32_t>(cdf_pick(cdf_k, unit53(splitmix64(kd ^ static_cast<uint64_t>(i)))));
    const uint64_t ks = splitmix64(seed ^ LFR_COM_SALT);
    std::vector<int64_t> csz;
    int64_t sum = 0;
    while (sum < n) {
        int64_t s = sp.min_community + cdf_pick(cdf_s, unit53(splitmix64(ks ^ static_cast<uint64_t>(csz.size()))));
        if (sum + s > n)
            s = n - sum;
        csz.push_back(s);
        sum += s;
    }
    if (csz.size() > 1 && csz.back() < sp.min_community) {
        csz[csz.size() - 2] += csz.back();
        csz.pop_back();
    }
    const int64_t C = static_cast<int64_t>(csz.size());
    for (int64_t i = 0; i < n; ++i)
        kin[i] = static_cast<int32_t>(std::floor((1.0 - sp.mu) * static_cast<double>(deg[i]) + 0.5));
    // node order: kin desc, id asc (counting sort)
    std::vector<int32_t> node_order(n);
    {
        std::vector<int64_t> cnt(kmax + 2, 0);
        for (int64_t i = 0; i < n; ++i)
            cnt[kmax - kin[i] + 1]++;
        for (int32_t d = 0; d <= kmax; ++d)
            cnt[d + 1] += cnt[d];
        for (int64_t i = 0; i < n; ++i)
            node_order[cnt[kmax - kin[i]]++] = static_cast<int32_t>(i);
    }
    std::vector<int64_t> com_order(C);
    {
        int64_t top = std::min<int64_t>(sp.max_community, n);
        for (int64_t j = 0; j < C; ++j)
            top = std::max(top, csz[j]);
        std::vector<int64_t> cnt(top + 2, 0);
        for (int64_t j = 0; j < C; ++j)
            cnt[top - csz[j] + 1]++;
        for (int64_t d = 0; d <= top; ++d)
            cnt[d + 1] += cnt[d];
        for (int64_t j = 0; j < C; ++j)
            com_order[cnt[top - csz[j]]++] = j;
    }
    std::vector<int32_t> comm(n);
    std::vector<int64_t> capleft(csz), avail;
    avail.reserve(C);
    int64_t elig = 0;
    const uint64_t ka = splitmix64(seed ^ LFR_ASG_SALT);
    for (int64_t t = 0; t < n; ++t) {
        const int32_t i = node_order[t];
        while (elig < C && csz[com_order[elig]] > kin[i]) {
            const int64_t j = com_order[elig++];
            if (capleft[j] > 0)
                avail.push_back(j);
        }
        int64_t c;
        if (!avail.empty()) {
            const int64_t idx = static_cast<int64_t>(splitmix64(ka ^ static_cast<uint64_t>(i)) % avail.size());
            c = avail[idx];
            if (--capleft[c] == 0) {
                avail[idx] = avail.back();
                avail.pop_back();
            }
        } else {
            int64_t j = 0;
            while (capleft[com_order[j]] == 0)
                ++j;
            c = com_order[j];
            --capleft[c];
            if (kin[i] > csz[c] - 1)
                kin[i] = static_cast<int32_t>(csz[c] - 1);
            if (capleft[c] == 0)
                for (size_t q = 0; q < avail.size(); ++q)
                    if (avail[q] == c) {
                        avail[q] = avail.back();
                        avail.pop_back();
                        break;
                    }
        }
        comm[i] = static_cast<int32_t>(c);
    }
    std::vector<int64_t> coff(C + 1, 0);
    for (int64_t i = 0; i < n; ++i)
        coff[comm[i] + 1]++;
    for (int64_t j = 0; j < C; ++j)
        coff[j + 1] += coff[j];
    std::vector<int32_t> members(n);
    {
        std::vector<int64_t> fill(coff.begin(), coff.end() - 1);
        for (int64_t i = 0; i < n; ++i)
            members[fill[comm[i]]++] = static_cast<int32_t>(i);
    }
    std::vector<int64_t> kin_prefix(n), vin(C), eoff(C + 1, 0), kout_prefix(n);
    for (int64_t j = 0; j < C; ++j) {
        int64_t acc = 0;
        for (int64_t p = coff[j]; p < coff[j + 1]; ++p) {
            kin_prefix[p] = acc;
            acc += kin[members[p]];
        }
        vin[j] = acc;
        eoff[j + 1] = eoff[j] + acc / 2;
    }
    int64_t kout_total = 0;
    for (int64_t i = 0; i < n; ++i) {
        kout_prefix[i] = kout_total;
        kout_total += deg[i] - kin[i];
    }
    const int64_t m_int = eoff[C], m_ext = kout_total / 2;
    DBuf<int64_t> d_eoff, d_coff, d_vin, d_kinp, d_koutp;
    DBuf<int32_t> d_mem, d_comm;
    upload(ctx, d_eoff, eoff);
    upload(ctx, d_coff, coff);
    upload(ctx, d_vin, vin);
    upload(ctx, d_kinp, kin_prefix);
    upload(ctx, d_koutp, kout_prefix);
    upload(ctx, d_mem, members);
    upload(ctx, d_comm, comm);
    DBuf<int32_t> eu(ctx, std::max<int64_t>(m_int + m_ext, 1)), ev(ctx, std::max<int64_t>(m_int + m_ext, 1));
    DBuf<int32_t> cnt(ctx, 1);
    cnt.zero();
    if (m_int > 0)
        CD_LAUNCH(ctx, "generate", k_lfr_internal, grid_for(m_int, 256, ctx->num_sms * 16), 256, 0, m_int, C,
                  splitmix64(seed ^ LFR_INT_SALT), static_cast<const int64_t *>(d_eoff.p),
                  static_cast<const int64_t *>(d_coff.p), static_cast<const int64_t *>(d_vin.p),
                  static_cast<const int64_t *>(d_kinp.p), static_cast<const int32_t *>(d_mem.p), eu.p, ev.p, cnt.p);
    if (m_ext > 0)
        CD_LAUNCH(ctx, "generate", k_lfr_external, grid_for(m_ext, 256, ctx->num_sms * 16), 256, 0, m_ext, n,
                  splitmix64(seed ^ LFR_EXT_SALT), kout_total, static_cast<const int64_t *>(d_koutp.p),
                  static_cast<const int32_t *>(d_comm.p), eu.p, ev.p, cnt.p);
    int32_t m = 0;
    CD_CUDA(cudaMemcpyAsync(&m, cnt.p, sizeof(m), cudaMemcpyDeviceToHost, ctx->stream));
    if (truth_dev)
        CD_CUDA(cudaMemcpyAsync(truth_dev, comm.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return graph_from_pairs(ctx, n, m, eu.p, ev.p, nullptr, DUP_ONE);
}

}  // namespace cdk
