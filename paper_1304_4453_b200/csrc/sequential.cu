// sequential.cu -- the reference's one-worker move phase (H/louvain.hpp:65-141
// with workers == 1) and its MoveObserver (:60, :127-128).
//
// The device's own move phase evaluates a bucket of nodes against frozen
// labels, so the moves of one sub-sweep happen together and
// an observer could not see a partition after every single move.  This path
// keeps the reference's order instead: nodes u = 0..n-1, each move applied to
// (z, vols) before the next node is evaluated.  It is a test / debugging
// hook (the reference says the observer's ordering is meaningful only with
// one worker), so it is one warp walking the nodes in order:
//   * the row is read 32 entries at a time; lanes holding the same community
//     are grouped by match_any and their leader adds the weights into the
//     dense fp64 tally aff[d] in row order -- the reference's summation
//     order, so the tallies are bit-identical for any weights;
//   * candidates are scored with the reference's expression (no FMA) and
//     reduced with its tie rule (largest gain, then smallest id);
//   * lane 0 applies the move and appends (u, c, d, gain) to the pass log,
//     which the host replays to the observer after the pass.
#include "comm.cuh"
#include "detect.cuh"
#include "graph.cuh"

namespace cdk {

struct SeqMove {
    int32_t u, c, d, pad;
    double gain;
};

__global__ void __launch_bounds__(32) k_move_sequential(int64_t n, const int64_t *off, const int32_t *col,
                                                        const float *w, const double *vol, double gamma,
                                                        double inv_total, double inv_sq2, int32_t *z, double *vols,
                                                        double *aff, int32_t *touched, SeqMove *log,
                                                        int64_t *nlog) {
    __shared__ float s_w[32];
    __shared__ int32_t s_nt;
    const int lane = threadIdx.x;
    int64_t moves = 0;
    for (int64_t u = 0; u < n; ++u) {
        const int64_t b = off[u], e = off[u + 1];
        if (b == e)  // g.degree(u) == 0 (H/louvain.hpp:91-92)
            continue;
        const int32_t c = z[u];
        if (lane == 0)
            s_nt = 0;
        __syncwarp();
        for (int64_t i0 = b; i0 < e; i0 += 32) {
            const int64_t i = i0 + lane;
            int32_t d = -1;
            float wi = 0.0f;
            if (i < e) {
                const int32_t v = col[i];
                if (v != u) {
                    d = z[v];
                    wi = w ? w[i] : 1.0f;
                }
            }
            s_w[lane] = wi;
            __syncwarp();
            const unsigned grp = __match_any_sync(0xffffffffu, d);
            if (d >= 0 && __ffs(grp) - 1 == lane) {
                double a = aff[d];
                if (a == 0.0)
                    touched[atomicAdd(&s_nt, 1)] = d;
                for (unsigned m = grp; m; m &= m - 1)
                    a = __dadd_rn(a, static_cast<double>(s_w[__ffs(m) - 1]));
                aff[d] = a;
            }
            __syncwarp();
        }
        const int32_t nt = s_nt;
        const double vol_u = vol[u];
        const double w_c = aff[c];
        const double vol_c = __dsub_rn(vols[c], vol_u);
        double best_delta = 0.0;
        int32_t best = c;
        for (int32_t j = lane; j < nt; j += 32) {
            const int32_t d = touched[j];
            if (d == c)
                continue;
            // (aff[d] - w_c) * inv_total + gamma * (vol_c - vols[d]) * vol_u * inv_sq2
            const double delta =
                __dadd_rn(__dmul_rn(__dsub_rn(aff[d], w_c), inv_total),
                          __dmul_rn(__dmul_rn(__dmul_rn(gamma, __dsub_rn(vol_c, vols[d])), vol_u), inv_sq2));
            if (delta > best_delta || (delta == best_delta && best != c && d < best)) {
                best_delta = delta;
                best = d;
            }
        }
        // the reference's rule is order-free: the largest positive gain, ties to the smallest id
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, best_delta, o);
            const int32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
            if (od > best_delta || (od == best_delta && od > 0.0 && ob < best)) {
                best_delta = od;
                best = ob;
            }
        }
        for (int32_t j = lane; j < nt; j += 32)
            aff[touched[j]] = 0.0;
        if (best != c && best_delta > 0.0) {
            if (lane == 0) {
                vols[c] = __dsub_rn(vols[c], vol_u);
                vols[best] = __dadd_rn(vols[best], vol_u);
                z[u] = best;
                log[moves] = SeqMove{static_cast<int32_t>(u), c, best, 0, best_delta};
            }
            ++moves;
        }
        __syncwarp();
    }
    if (lane == 0)
        *nlog = moves;
}

bool move_phase_sequential_dev(cd_ctx *ctx, cd_graph *g, int32_t *z, int64_t ub, double gamma, int64_t max_passes,
                               cd_move_observer observer, void *user) {
    const int64_t n = g->n;
    if (n == 0 || g->total == 0.0)
        return false;
    DBuf<double> vols(ctx, ub), aff(ctx, ub);
    DBuf<int32_t> touched(ctx, std::max<int64_t>(g->max_degree, 1));
    DBuf<SeqMove> log(ctx, n);
    DBuf<int64_t> nlog(ctx, 1);
    community_volumes_dev(ctx, g, z, vols.p, ub);  // H/louvain.hpp:75
    CD_CUDA(cudaMemsetAsync(aff.p, 0, ub * sizeof(double), ctx->stream));
    const double inv_total = 1.0 / g->total;
    const double inv_sq2 = 1.0 / (2.0 * g->total * g->total);
    std::vector<SeqMove> host;
    bool changed = false;
    for (int64_t pass = 0; pass < max_passes; ++pass) {
        CD_LAUNCH(ctx, "move_seq", k_move_sequential, 1, 32, 0, n, g->off.p, g->col.p, g->weighted ? g->w.p : nullptr, g->vol.p, gamma,
                  inv_total, inv_sq2, z, vols.p, aff.p, touched.p, log.p, nlog.p);
        int64_t k = 0;
        CD_CUDA(cudaMemcpyAsync(&k, nlog.p, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        ctx_sync(ctx);
        if (k == 0)
            break;
        changed = true;
        if (observer) {
            host.resize(k);
            CD_CUDA(cudaMemcpyAsync(host.data(), log.p, k * sizeof(SeqMove), cudaMemcpyDeviceToHost, ctx->stream));
            ctx_sync(ctx);
            for (const SeqMove &mv : host)
                observer(user, mv.u, mv.c, mv.d, mv.gain);
        }
    }
    return changed;
}

}  // namespace cdk
