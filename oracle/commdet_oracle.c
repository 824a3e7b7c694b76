/*
 * commdet_oracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see the header).
 *
 * Restates the reference (/root/reference/proj/include/commdet, "H/" below)
 * in plain C, single-threaded, plus ports of this repo's device update order
 * and generators.  Build: oracle/Makefile (gcc -O2 -ffp-contract=off).
 */
#include "commdet_oracle.h"

/* per-move gains summed in fixed point (units of 2^-44): order-free, like the device */
#define CDO_GAIN_FX_SCALE 17592186044416.0

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* small utilities                                                          */
/* ------------------------------------------------------------------------ */

void cdo_graph_free(cdo_graph *g) {
    if (!g)
        return;
    free(g->off);
    free(g->col);
    free(g->w);
    free(g->vol);
    free(g->loop);
    memset(g, 0, sizeof(*g));
}

/* LSD radix sort of uint64 keys with an optional uint64 payload (stable). */
static int radix_sort_u64(uint64_t *key, uint64_t *val, int64_t len, int key_bits) {
    if (len <= 1)
        return 0;
    uint64_t *tk = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)len);
    uint64_t *tv = val ? (uint64_t *)malloc(sizeof(uint64_t) * (size_t)len) : NULL;
    if (!tk || (val && !tv)) {
        free(tk);
        free(tv);
        return CDO_ENOMEM;
    }
    int64_t cnt[65537];
    for (int shift = 0; shift < key_bits; shift += 16) {
        memset(cnt, 0, sizeof(cnt));
        for (int64_t i = 0; i < len; ++i)
            cnt[((key[i] >> shift) & 0xffff) + 1]++;
        for (int d = 0; d < 65536; ++d)
            cnt[d + 1] += cnt[d];
        for (int64_t i = 0; i < len; ++i) {
            int64_t p = cnt[(key[i] >> shift) & 0xffff]++;
            tk[p] = key[i];
            if (val)
                tv[p] = val[i];
        }
        memcpy(key, tk, sizeof(uint64_t) * (size_t)len);
        if (val)
            memcpy(val, tv, sizeof(uint64_t) * (size_t)len);
    }
    free(tk);
    free(tv);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* graph construction                                                       */
/* ------------------------------------------------------------------------ */

/* H/graph.hpp:229-255 */
void cdo_finalize(cdo_graph *g) {
    const int64_t n = g->n;
    double total = 0.0;
    int64_t m = 0;
    for (int64_t u = 0; u < n; ++u) {
        double vol = 0.0;
        g->loop[u] = 0.0;
        for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
            const int64_t v = g->col[i];
            const double w = g->w[i];
            vol += w;
            if (v == u) {
                g->loop[u] = w;
                vol += w;
                total += w;
                ++m;
            } else if (v > u) {
                total += w;
                ++m;
            }
        }
        g->vol[u] = vol;
    }
    g->total = total;
    g->m = m;
}

static int alloc_graph(cdo_graph *g, int64_t n, int64_t D) {
    memset(g, 0, sizeof(*g));
    g->n = n;
    g->D = D;
    g->off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    g->col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(D > 0 ? D : 1));
    g->w = (double *)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
    g->vol = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    g->loop = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    if (!g->off || !g->col || !g->w || !g->vol || !g->loop) {
        cdo_graph_free(g);
        return CDO_ENOMEM;
    }
    return 0;
}

typedef struct {
    int32_t v;
    double w;
} nbr_t;

/* std::sort on pair<node, edgeweight> (H/graph.hpp:177): by v, then by w. */
static int cmp_nbr(const void *a, const void *b) {
    const nbr_t *x = (const nbr_t *)a, *y = (const nbr_t *)b;
    if (x->v != y->v)
        return x->v < y->v ? -1 : 1;
    if (x->w != y->w)
        return x->w < y->w ? -1 : 1;
    return 0;
}

/* H/graph.hpp:48-81 + sort_and_merge :169-204 + compact_storage :207-227 */
int cdo_graph_from_edges(int64_t n, int64_t m, const int32_t *eu, const int32_t *ev, const double *ew,
                         int merge_duplicates, cdo_graph *out) {
    for (int64_t i = 0; i < m; ++i) {
        if (eu[i] < 0 || ev[i] < 0 || eu[i] >= n || ev[i] >= n)
            return CDO_EINPUT;
        const double w = ew ? ew[i] : 1.0;
        if (!(w > 0.0))
            return CDO_EINPUT;
    }
    int64_t *deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!deg)
        return CDO_ENOMEM;
    for (int64_t i = 0; i < m; ++i) {
        deg[eu[i]]++;
        if (eu[i] != ev[i])
            deg[ev[i]]++;
    }
    int64_t D = 0;
    for (int64_t u = 0; u < n; ++u)
        D += deg[u];
    nbr_t *tmp = (nbr_t *)malloc(sizeof(nbr_t) * (size_t)(D > 0 ? D : 1));
    int64_t *start = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *fill = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!tmp || !start || !fill) {
        free(deg);
        free(tmp);
        free(start);
        free(fill);
        return CDO_ENOMEM;
    }
    for (int64_t u = 0; u < n; ++u)
        start[u + 1] = start[u] + deg[u];
    memcpy(fill, start, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < m; ++i) {
        const double w = ew ? ew[i] : 1.0;
        nbr_t a = {ev[i], w};
        tmp[fill[eu[i]]++] = a;
        if (eu[i] != ev[i]) {
            nbr_t b = {eu[i], w};
            tmp[fill[ev[i]]++] = b;
        }
    }
    /* per-row sort; duplicates are an error unless merged (:178-194) */
    int64_t kept = 0;
    for (int64_t u = 0; u < n; ++u) {
        nbr_t *row = tmp + start[u];
        const int64_t len = start[u + 1] - start[u];
        qsort(row, (size_t)len, sizeof(nbr_t), cmp_nbr);
        for (int64_t i = 0; i + 1 < len; ++i)
            if (row[i].v == row[i + 1].v && !merge_duplicates) {
                free(deg);
                free(tmp);
                free(start);
                free(fill);
                return CDO_EINPUT;
            }
        int64_t o = 0;
        for (int64_t i = 0; i < len; ++i) {
            if (o > 0 && row[o - 1].v == row[i].v)
                row[o - 1].w += row[i].w;
            else
                row[o++] = row[i];
        }
        deg[u] = o;
        kept += o;
    }
    int rc = alloc_graph(out, n, kept);
    if (rc) {
        free(deg);
        free(tmp);
        free(start);
        free(fill);
        return rc;
    }
    for (int64_t u = 0; u < n; ++u) {
        out->off[u + 1] = out->off[u] + deg[u];
        for (int64_t i = 0; i < deg[u]; ++i) {
            out->col[out->off[u] + i] = tmp[start[u] + i].v;
            out->w[out->off[u] + i] = tmp[start[u] + i].w;
        }
    }
    free(deg);
    free(tmp);
    free(start);
    free(fill);
    cdo_finalize(out);
    return 0;
}

int cdo_graph_from_csr(int64_t n, const int64_t *off, const int32_t *col, const double *w, cdo_graph *out) {
    const int64_t D = off[n];
    int rc = alloc_graph(out, n, D);
    if (rc)
        return rc;
    memcpy(out->off, off, sizeof(int64_t) * (size_t)(n + 1));
    if (D > 0)
        memcpy(out->col, col, sizeof(int32_t) * (size_t)D);
    for (int64_t i = 0; i < D; ++i)
        out->w[i] = w ? w[i] : 1.0;
    cdo_finalize(out);
    return 0;
}

/* Build from unique canonical undirected pairs (u < v) already sorted by
 * (u, v); used by the generators (every row comes out ascending). */
static int graph_from_sorted_pairs(int64_t n, int64_t m, const uint64_t *keys, const double *w, cdo_graph *out) {
    int rc = alloc_graph(out, n, 2 * m);
    if (rc)
        return rc;
    int64_t *deg = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!deg) {
        cdo_graph_free(out);
        return CDO_ENOMEM;
    }
    for (int64_t i = 0; i < m; ++i) {
        deg[keys[i] >> 32]++;
        deg[keys[i] & 0xffffffffu]++;
    }
    for (int64_t u = 0; u < n; ++u)
        out->off[u + 1] = out->off[u] + deg[u];
    int64_t *fill = deg;
    memcpy(fill, out->off, sizeof(int64_t) * (size_t)n);
    /* Row u lists its smaller neighbours first (they come from rows v < u,
     * visited in ascending v), then its larger ones (ascending v): walking
     * pairs in (u, v) order keeps every row sorted. */
    for (int64_t i = 0; i < m; ++i) {
        const int32_t u = (int32_t)(keys[i] >> 32), v = (int32_t)(keys[i] & 0xffffffffu);
        const double ww = w ? w[i] : 1.0;
        out->col[fill[v]] = u;
        out->w[fill[v]++] = ww;
    }
    for (int64_t i = 0; i < m; ++i) {
        const int32_t u = (int32_t)(keys[i] >> 32), v = (int32_t)(keys[i] & 0xffffffffu);
        const double ww = w ? w[i] : 1.0;
        out->col[fill[u]] = v;
        out->w[fill[u]++] = ww;
    }
    free(deg);
    cdo_finalize(out);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* generators                                                               */
/* ------------------------------------------------------------------------ */

/* H/generator.hpp:24-29 */
uint64_t cdo_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* H/generator.hpp:31-37 */
static uint64_t row_key(uint64_t seed, uint64_t u) { return cdo_splitmix64(seed ^ cdo_splitmix64(u)); }
double cdo_row_uniform(uint64_t key, uint64_t v) {
    return (double)(cdo_splitmix64(key ^ cdo_splitmix64(v)) >> 11) * 0x1.0p-53;
}

/* H/generator.hpp:48-50 */
static int64_t planted_block(int64_t u, int64_t n, int64_t k) {
    return (int64_t)(((unsigned __int128)(uint64_t)u * (uint64_t)k) / (uint64_t)n);
}

/* H/generator.hpp:52-104: pair (u<v) is an edge iff row_uniform(row_key(seed,u), v) < p. */
int cdo_generate_planted(int64_t n, int64_t k, double p_in, double p_out, uint64_t seed, cdo_graph *out,
                         int32_t *truth) {
    if (k < 1 || (n > 0 && k > n))
        return CDO_EINVAL;
    if (p_out < 0.0 || p_in > 1.0 || p_out > p_in)
        return CDO_EINVAL;
    int64_t cap = 1024, m = 0;
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)cap);
    if (!keys)
        return CDO_ENOMEM;
    for (int64_t u = 0; u < n; ++u) {
        const int64_t bu = planted_block(u, n, k);
        if (truth)
            truth[u] = (int32_t)bu;
        int64_t v_end = n;
        if (p_out == 0.0) { /* :75-80 */
            v_end = u + 1;
            while (v_end < n && planted_block(v_end, n, k) == bu)
                ++v_end;
        }
        const uint64_t key = row_key(seed, (uint64_t)u);
        for (int64_t v = u + 1; v < v_end; ++v) {
            const double p = planted_block(v, n, k) == bu ? p_in : p_out;
            if (p > 0.0 && cdo_row_uniform(key, (uint64_t)v) < p) {
                if (m == cap) {
                    cap *= 2;
                    uint64_t *nk = (uint64_t *)realloc(keys, sizeof(uint64_t) * (size_t)cap);
                    if (!nk) {
                        free(keys);
                        return CDO_ENOMEM;
                    }
                    keys = nk;
                }
                keys[m++] = ((uint64_t)u << 32) | (uint64_t)v;
            }
        }
    }
    int rc = graph_from_sorted_pairs(n, m, keys, NULL, out);
    free(keys);
    return rc;
}

/* ---- R-MAT (device generator port) ------------- */

#define RMAT_SALT 0x524d41542d4b4559ULL   /* "RMAT-KEY" */
#define WEIGHT_SALT 0x5745494748542d4bULL /* "WEIGHT-K" */

static void sort_unique(uint64_t *keys, int64_t *m) {
    int64_t o = 0;
    for (int64_t i = 0; i < *m; ++i)
        if (o == 0 || keys[o - 1] != keys[i])
            keys[o++] = keys[i];
    *m = o;
}

static double dyadic_weight(uint64_t wkey, uint64_t pair) {
    return (double)((cdo_splitmix64(wkey ^ pair) >> 40) + 1) * 0x1.0p-24;
}

int cdo_generate_rmat(int scale, int edge_factor, double a, double b, double c, int weighted, uint64_t seed,
                      cdo_graph *out) {
    if (scale < 1 || scale > 30 || edge_factor < 1)
        return CDO_EINVAL;
    const int64_t n = (int64_t)1 << scale;
    const int64_t M = (int64_t)edge_factor << scale;
    const uint64_t ta = (uint64_t)(a * 4294967296.0);
    const uint64_t tab = (uint64_t)((a + b) * 4294967296.0);
    const uint64_t tabc = (uint64_t)((a + b + c) * 4294967296.0);
    const uint64_t key = cdo_splitmix64(seed ^ RMAT_SALT);
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)M);
    if (!keys)
        return CDO_ENOMEM;
    int64_t m = 0;
    for (int64_t e = 0; e < M; ++e) {
        uint64_t u = 0, v = 0;
        for (int lvl = 0; lvl < scale; lvl += 2) {
            const uint64_t r = cdo_splitmix64(key ^ ((uint64_t)e * 16u + (uint64_t)(lvl >> 1)));
            for (int h = 0; h < 2 && lvl + h < scale; ++h) {
                const uint64_t r32 = h ? (r >> 32) : (r & 0xffffffffu);
                uint64_t bu, bv;
                if (r32 < ta) {
                    bu = 0;
                    bv = 0;
                } else if (r32 < tab) {
                    bu = 0;
                    bv = 1;
                } else if (r32 < tabc) {
                    bu = 1;
                    bv = 0;
                } else {
                    bu = 1;
                    bv = 1;
                }
                u = (u << 1) | bu;
                v = (v << 1) | bv;
            }
        }
        if (u == v)
            continue;
        const uint64_t lo = u < v ? u : v, hi = u < v ? v : u;
        keys[m++] = (lo << 32) | hi;
    }
    int rc = radix_sort_u64(keys, NULL, m, 2 * scale <= 32 ? 64 : 64);
    if (rc) {
        free(keys);
        return rc;
    }
    sort_unique(keys, &m);
    double *w = NULL;
    if (weighted) {
        const uint64_t wkey = cdo_splitmix64(seed ^ WEIGHT_SALT);
        w = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
        if (!w) {
            free(keys);
            return CDO_ENOMEM;
        }
        for (int64_t i = 0; i < m; ++i)
            w[i] = dyadic_weight(wkey, keys[i]);
    }
    rc = graph_from_sorted_pairs(n, m, keys, w, out);
    free(keys);
    free(w);
    return rc;
}

/* ---- LFR-shaped (device generator port) -------- */

#define LFR_DEG_SALT 0x4c46522d44454731ULL
#define LFR_COM_SALT 0x4c46522d434f4d31ULL
#define LFR_ASG_SALT 0x4c46522d41534731ULL
#define LFR_INT_SALT 0x4c46522d494e5431ULL
#define LFR_EXT_SALT 0x4c46522d45585431ULL

static double unit53(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

static uint64_t mulhi64(uint64_t a, uint64_t b) { return (uint64_t)(((unsigned __int128)a * b) >> 64); }

/* smallest index i with u < cdf[i]; cdf ascending, cdf[len-1] = 2.0 */
static int64_t cdf_pick(const double *cdf, int64_t len, double u) {
    int64_t lo = 0, hi = len - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (u < cdf[mid])
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

/* largest index i in [0, len) with prefix[i] <= s (prefix ascending, prefix[0]=0) */
static int64_t prefix_find(const int64_t *prefix, int64_t len, int64_t s) {
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

int cdo_generate_lfr(const cdo_lfr_spec *sp, uint64_t seed, cdo_graph *out, int32_t *truth) {
    const int64_t n = sp->n;
    if (n < 2 || sp->max_degree < 1 || sp->min_community < 1 || sp->max_community < sp->min_community ||
        sp->mu < 0.0 || sp->mu > 1.0)
        return CDO_EINVAL;
    const int32_t kmax = sp->max_degree;
    /* 1. degree table: integer power law on [kmin, kmax], kmin chosen so the
     *    mean is closest to avg_degree */
    int32_t kmin = 1;
    double best_err = 1e300;
    for (int32_t k0 = 1; k0 <= kmax; ++k0) {
        double s0 = 0.0, s1 = 0.0;
        for (int32_t k = k0; k <= kmax; ++k) {
            const double p = pow((double)k, -sp->tau1);
            s0 += p;
            s1 += p * (double)k;
        }
        const double err = fabs(s1 / s0 - sp->avg_degree);
        if (err < best_err) {
            best_err = err;
            kmin = k0;
        }
    }
    const int64_t nk = kmax - kmin + 1;
    double *cdf_k = (double *)malloc(sizeof(double) * (size_t)nk);
    const int64_t ns = sp->max_community - sp->min_community + 1;
    double *cdf_s = (double *)malloc(sizeof(double) * (size_t)ns);
    {
        double tot = 0.0;
        for (int64_t i = 0; i < nk; ++i)
            tot += pow((double)(kmin + i), -sp->tau1);
        double acc = 0.0;
        for (int64_t i = 0; i < nk; ++i) {
            acc += pow((double)(kmin + i), -sp->tau1);
            cdf_k[i] = acc / tot;
        }
        cdf_k[nk - 1] = 2.0;
        tot = 0.0;
        for (int64_t i = 0; i < ns; ++i)
            tot += pow((double)(sp->min_community + i), -sp->tau2);
        acc = 0.0;
        for (int64_t i = 0; i < ns; ++i) {
            acc += pow((double)(sp->min_community + i), -sp->tau2);
            cdf_s[i] = acc / tot;
        }
        cdf_s[ns - 1] = 2.0;
    }
    /* 2. degrees */
    int32_t *deg = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    const uint64_t kd = cdo_splitmix64(seed ^ LFR_DEG_SALT);
    for (int64_t i = 0; i < n; ++i)
        deg[i] = kmin + (int32_t)cdf_pick(cdf_k, nk, unit53(cdo_splitmix64(kd ^ (uint64_t)i)));
    /* 3. community sizes */
    const uint64_t ks = cdo_splitmix64(seed ^ LFR_COM_SALT);
    int64_t csz_cap = 1024, C = 0, sum = 0;
    int64_t *csz = (int64_t *)malloc(sizeof(int64_t) * (size_t)csz_cap);
    while (sum < n) {
        int64_t s = sp->min_community + cdf_pick(cdf_s, ns, unit53(cdo_splitmix64(ks ^ (uint64_t)C)));
        if (sum + s > n)
            s = n - sum;
        if (C == csz_cap) {
            csz_cap *= 2;
            csz = (int64_t *)realloc(csz, sizeof(int64_t) * (size_t)csz_cap);
        }
        csz[C++] = s;
        sum += s;
    }
    if (C > 1 && csz[C - 1] < sp->min_community) {
        csz[C - 2] += csz[C - 1];
        --C;
    }
    /* 4. internal / external degrees */
    int32_t *kin = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i)
        kin[i] = (int32_t)floor((1.0 - sp->mu) * (double)deg[i] + 0.5);
    /* 5. assignment: nodes by kin desc (stable by id), communities by size
     *    desc (stable by index); uniform pick among eligible non-full ones */
    int32_t *node_order = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    {
        int64_t *cnt = (int64_t *)calloc((size_t)kmax + 2, sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i)
            cnt[kmax - kin[i] + 1]++;
        for (int32_t d = 0; d <= kmax; ++d)
            cnt[d + 1] += cnt[d];
        for (int64_t i = 0; i < n; ++i)
            node_order[cnt[kmax - kin[i]]++] = (int32_t)i;
        free(cnt);
    }
    int64_t *com_order = (int64_t *)malloc(sizeof(int64_t) * (size_t)C);
    {
        const int64_t smax = sp->max_community > n ? n : sp->max_community;
        int64_t top = smax;
        for (int64_t j = 0; j < C; ++j)
            if (csz[j] > top)
                top = csz[j];
        int64_t *cnt = (int64_t *)calloc((size_t)top + 2, sizeof(int64_t));
        for (int64_t j = 0; j < C; ++j)
            cnt[top - csz[j] + 1]++;
        for (int64_t d = 0; d <= top; ++d)
            cnt[d + 1] += cnt[d];
        for (int64_t j = 0; j < C; ++j)
            com_order[cnt[top - csz[j]]++] = j;
        free(cnt);
    }
    int32_t *comm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int64_t *capleft = (int64_t *)malloc(sizeof(int64_t) * (size_t)C);
    int64_t *avail = (int64_t *)malloc(sizeof(int64_t) * (size_t)C);
    for (int64_t j = 0; j < C; ++j)
        capleft[j] = csz[j];
    int64_t navail = 0, elig = 0;
    const uint64_t ka = cdo_splitmix64(seed ^ LFR_ASG_SALT);
    for (int64_t t = 0; t < n; ++t) {
        const int32_t i = node_order[t];
        while (elig < C && csz[com_order[elig]] > kin[i]) {
            const int64_t j = com_order[elig++];
            if (capleft[j] > 0)
                avail[navail++] = j;
        }
        int64_t c;
        if (navail > 0) {
            const int64_t idx = (int64_t)(cdo_splitmix64(ka ^ (uint64_t)i) % (uint64_t)navail);
            c = avail[idx];
            if (--capleft[c] == 0)
                avail[idx] = avail[--navail];
        } else {
            /* no big-enough community has room: largest with room, clamp kin */
            int64_t j = 0;
            while (capleft[com_order[j]] == 0)
                ++j;
            c = com_order[j];
            --capleft[c];
            if (kin[i] > csz[c] - 1)
                kin[i] = (int32_t)(csz[c] - 1);
            /* a community that is eligible later must not be re-added full */
            if (capleft[c] == 0)
                for (int64_t q = 0; q < navail; ++q)
                    if (avail[q] == c) {
                        avail[q] = avail[--navail];
                        break;
                    }
        }
        comm[i] = (int32_t)c;
    }
    if (truth)
        memcpy(truth, comm, sizeof(int32_t) * (size_t)n);
    /* 6. members per community (ascending id), per-community kin prefix,
     *    global kout prefix, edge counts */
    int64_t *coff = (int64_t *)calloc((size_t)C + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        coff[comm[i] + 1]++;
    for (int64_t j = 0; j < C; ++j)
        coff[j + 1] += coff[j];
    int32_t *members = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)C);
        memcpy(fill, coff, sizeof(int64_t) * (size_t)C);
        for (int64_t i = 0; i < n; ++i)
            members[fill[comm[i]]++] = (int32_t)i;
        free(fill);
    }
    /* kin_prefix[p] over the member array (global positions), per-community
     * start at 0: stored as exclusive prefix within each community segment */
    int64_t *kin_prefix = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *vin = (int64_t *)malloc(sizeof(int64_t) * (size_t)C);
    int64_t *eoff = (int64_t *)calloc((size_t)C + 1, sizeof(int64_t));
    for (int64_t j = 0; j < C; ++j) {
        int64_t acc = 0;
        for (int64_t p = coff[j]; p < coff[j + 1]; ++p) {
            kin_prefix[p] = acc;
            acc += kin[members[p]];
        }
        vin[j] = acc;
        eoff[j + 1] = eoff[j] + acc / 2;
    }
    int64_t *kout_prefix = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t kout_total = 0;
    for (int64_t i = 0; i < n; ++i) {
        kout_prefix[i] = kout_total;
        kout_total += deg[i] - kin[i];
    }
    const int64_t m_int = eoff[C];
    const int64_t m_ext = kout_total / 2;
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(m_int + m_ext + 1));
    int64_t m = 0;
    /* 7. internal edges */
    const uint64_t ki = cdo_splitmix64(seed ^ LFR_INT_SALT);
    for (int64_t e = 0; e < m_int; ++e) {
        /* community of edge e: largest j with eoff[j] <= e */
        const int64_t j = prefix_find(eoff, C + 1, e);
        const int64_t len = coff[j + 1] - coff[j];
        const uint64_t r1 = cdo_splitmix64(ki ^ (2u * (uint64_t)e));
        const uint64_t r2 = cdo_splitmix64(ki ^ (2u * (uint64_t)e + 1u));
        const int64_t s1 = (int64_t)mulhi64(r1, (uint64_t)vin[j]);
        const int64_t s2 = (int64_t)mulhi64(r2, (uint64_t)vin[j]);
        const int32_t a = members[coff[j] + prefix_find(kin_prefix + coff[j], len, s1)];
        const int32_t b = members[coff[j] + prefix_find(kin_prefix + coff[j], len, s2)];
        if (a == b)
            continue;
        const uint64_t lo = (uint64_t)(a < b ? a : b), hi = (uint64_t)(a < b ? b : a);
        keys[m++] = (lo << 32) | hi;
    }
    /* 8. external edges: endpoints proportional to kout, 8 attempts to find
     *    a cross-community pair */
    const uint64_t ke = cdo_splitmix64(seed ^ LFR_EXT_SALT);
    for (int64_t e = 0; e < m_ext; ++e) {
        for (uint64_t att = 0; att < 8; ++att) {
            const uint64_t r1 = cdo_splitmix64(ke ^ ((uint64_t)e * 16u + 2u * att));
            const uint64_t r2 = cdo_splitmix64(ke ^ ((uint64_t)e * 16u + 2u * att + 1u));
            const int64_t s1 = (int64_t)mulhi64(r1, (uint64_t)kout_total);
            const int64_t s2 = (int64_t)mulhi64(r2, (uint64_t)kout_total);
            const int32_t a = (int32_t)prefix_find(kout_prefix, n, s1);
            const int32_t b = (int32_t)prefix_find(kout_prefix, n, s2);
            if (comm[a] == comm[b])
                continue;
            const uint64_t lo = (uint64_t)(a < b ? a : b), hi = (uint64_t)(a < b ? b : a);
            keys[m++] = (lo << 32) | hi;
            break;
        }
    }
    int rc = radix_sort_u64(keys, NULL, m, 64);
    if (!rc) {
        sort_unique(keys, &m);
        rc = graph_from_sorted_pairs(n, m, keys, NULL, out);
    }
    free(keys);
    free(cdf_k);
    free(cdf_s);
    free(deg);
    free(csz);
    free(kin);
    free(node_order);
    free(com_order);
    free(comm);
    free(capleft);
    free(avail);
    free(coff);
    free(members);
    free(kin_prefix);
    free(vin);
    free(eoff);
    free(kout_prefix);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* quality                                                                  */
/* ------------------------------------------------------------------------ */

/* H/quality.hpp:35-51: for_edges (u <= v) intra, per-community volumes. */
int cdo_modularity(const cdo_graph *g, const int32_t *z, int64_t ub, double gamma, double *q) {
    const double total = g->total;
    if (total == 0.0)
        return CDO_EDOMAIN;
    double *intra = (double *)calloc((size_t)ub, sizeof(double));
    double *vol = (double *)calloc((size_t)ub, sizeof(double));
    if (!intra || !vol) {
        free(intra);
        free(vol);
        return CDO_ENOMEM;
    }
    for (int64_t u = 0; u < g->n; ++u) {
        if (z[u] < 0 || z[u] >= ub) {
            free(intra);
            free(vol);
            return CDO_ERANGE;
        }
    }
    for (int64_t u = 0; u < g->n; ++u)
        for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i)
            if (g->col[i] >= u && z[u] == z[g->col[i]])
                intra[z[u]] += g->w[i];
    for (int64_t u = 0; u < g->n; ++u)
        vol[z[u]] += g->vol[u];
    double mod = 0.0;
    for (int64_t c = 0; c < ub; ++c)
        mod += intra[c] / total - gamma * vol[c] * vol[c] / (4.0 * total * total);
    *q = mod;
    free(intra);
    free(vol);
    return 0;
}

/* H/quality.hpp:21-31 */
double cdo_coverage(const cdo_graph *g, const int32_t *z) {
    if (g->total == 0.0)
        return 0.0;
    double intra = 0.0;
    for (int64_t u = 0; u < g->n; ++u)
        for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i)
            if (g->col[i] >= u && z[u] == z[g->col[i]])
                intra += g->w[i];
    return intra / g->total;
}

/* H/louvain.hpp:27-31 */
void cdo_community_volumes(const cdo_graph *g, const int32_t *z, int64_t ub, double *vols) {
    memset(vols, 0, sizeof(double) * (size_t)ub);
    for (int64_t u = 0; u < g->n; ++u)
        vols[z[u]] += g->vol[u];
}

/* ------------------------------------------------------------------------ */
/* partition                                                                */
/* ------------------------------------------------------------------------ */

static int64_t max_label_plus_one(int64_t n, const int32_t *z) {
    int64_t ub = 1;
    for (int64_t u = 0; u < n; ++u)
        if ((int64_t)z[u] + 1 > ub)
            ub = (int64_t)z[u] + 1;
    return ub;
}

/* H/partition.hpp:39-53: first-appearance order */
int64_t cdo_compact(int64_t n, const int32_t *z, int32_t *out) {
    const int64_t ub = max_label_plus_one(n, z);
    int32_t *map = (int32_t *)malloc(sizeof(int32_t) * (size_t)ub);
    for (int64_t c = 0; c < ub; ++c)
        map[c] = -1;
    int32_t next = 0;
    for (int64_t u = 0; u < n; ++u) {
        if (map[z[u]] < 0)
            map[z[u]] = next++;
        out[u] = map[z[u]];
    }
    free(map);
    return next;
}

/* H/partition.hpp:55-60 */
int64_t cdo_community_count(int64_t n, const int32_t *z) {
    const int64_t ub = max_label_plus_one(n, z);
    uint8_t *seen = (uint8_t *)calloc((size_t)ub, 1);
    int64_t k = 0;
    for (int64_t u = 0; u < n; ++u)
        if (!seen[z[u]]) {
            seen[z[u]] = 1;
            ++k;
        }
    free(seen);
    return k;
}

/* ------------------------------------------------------------------------ */
/* PLP                                                                      */
/* ------------------------------------------------------------------------ */

/* H/plp.hpp:32-53 (linear tally, in neighbour order) */
int cdo_dominant_label(const cdo_graph *g, const int32_t *z, int32_t u, int32_t *out) {
    const int64_t lo = g->off[u], hi = g->off[u + 1];
    if (hi == lo)
        return CDO_EINVAL;
    int32_t *lab = (int32_t *)calloc((size_t)(hi - lo), sizeof(int32_t));
    double *wt = (double *)calloc((size_t)(hi - lo), sizeof(double));
    int64_t k = 0;
    for (int64_t i = lo; i < hi; ++i) {
        const int32_t l = z[g->col[i]];
        int64_t j = 0;
        for (; j < k; ++j)
            if (lab[j] == l) {
                wt[j] += g->w[i];
                break;
            }
        if (j == k) {
            lab[k] = l;
            wt[k++] = g->w[i];
        }
    }
    int32_t best = lab[0];
    double bw = wt[0];
    for (int64_t j = 0; j < k; ++j)
        if (wt[j] > bw || (wt[j] == bw && lab[j] < best)) {
            best = lab[j];
            bw = wt[j];
        }
    *out = best;
    free(lab);
    free(wt);
    return 0;
}

typedef struct {
    double *aff;
    int32_t *touched;
    int64_t cap;
} scratch_t;

static int scratch_init(scratch_t *s, int64_t ub, int64_t maxdeg) {
    s->aff = (double *)calloc((size_t)(ub > 0 ? ub : 1), sizeof(double));
    s->touched = (int32_t *)malloc(sizeof(int32_t) * (size_t)(maxdeg > 0 ? maxdeg : 1));
    s->cap = ub;
    return (s->aff && s->touched) ? 0 : CDO_ENOMEM;
}

static void scratch_free(scratch_t *s) {
    free(s->aff);
    free(s->touched);
}

static int64_t max_degree(const cdo_graph *g) {
    int64_t d = 0;
    for (int64_t u = 0; u < g->n; ++u)
        if (g->off[u + 1] - g->off[u] > d)
            d = g->off[u + 1] - g->off[u];
    return d;
}

/* dense-scratch tally of H/plp.hpp:111-126 against frozen z */
static int32_t plp_best(const cdo_graph *g, const int32_t *z, int32_t u, scratch_t *s) {
    int64_t nt = 0;
    for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
        const int32_t l = z[g->col[i]];
        if (s->aff[l] == 0.0)
            s->touched[nt++] = l;
        s->aff[l] += g->w[i];
    }
    int32_t best = s->touched[0];
    double bw = s->aff[best];
    for (int64_t j = 0; j < nt; ++j) {
        const int32_t l = s->touched[j];
        if (s->aff[l] > bw || (s->aff[l] == bw && l < best)) {
            best = l;
            bw = s->aff[l];
        }
    }
    for (int64_t j = 0; j < nt; ++j)
        s->aff[s->touched[j]] = 0.0;
    return best;
}

int64_t cdo_plp_sweep_sync(const cdo_graph *g, const int32_t *z_in, int32_t *z_out) {
    const int64_t ub = max_label_plus_one(g->n, z_in);
    scratch_t s;
    if (scratch_init(&s, ub, max_degree(g))) {
        scratch_free(&s);
        return CDO_ENOMEM;
    }
    int64_t updated = 0;
    for (int64_t u = 0; u < g->n; ++u) {
        if (g->off[u + 1] == g->off[u]) {
            z_out[u] = z_in[u];
            continue;
        }
        z_out[u] = plp_best(g, z_in, (int32_t)u, &s);
        if (z_out[u] != z_in[u])
            ++updated;
    }
    scratch_free(&s);
    return updated;
}

/* H/plp.hpp:57-62 */
int cdo_is_stable(const cdo_graph *g, const int32_t *z) {
    for (int64_t u = 0; u < g->n; ++u) {
        if (g->off[u + 1] == g->off[u])
            continue;
        int32_t d;
        cdo_dominant_label(g, z, (int32_t)u, &d);
        if (d != z[u])
            return 0;
    }
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Louvain                                                                  */
/* ------------------------------------------------------------------------ */

/* H/louvain.hpp:37-56 */
double cdo_delta_mod(const cdo_graph *g, const int32_t *z, const double *vols, int32_t u, int32_t target,
                     double gamma) {
    const int32_t c = z[u];
    if (target == c)
        return 0.0;
    double w_c = 0.0, w_d = 0.0;
    for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
        const int32_t v = g->col[i];
        if (v == u)
            continue;
        if (z[v] == c)
            w_c += g->w[i];
        else if (z[v] == target)
            w_d += g->w[i];
    }
    const double total = g->total;
    const double vol_u = g->vol[u];
    const double vol_c = vols[c] - vol_u;
    const double vol_d = vols[target];
    return (w_d - w_c) / total + gamma * (vol_c - vol_d) * vol_u / (2.0 * total * total);
}

/* Decision rule of H/louvain.hpp:91-120 against frozen (z, vols). */
static int32_t move_best(const cdo_graph *g, const int32_t *z, const double *vols, double gamma, double inv_total,
                         double inv_sq2, int32_t u, scratch_t *s, double *gain) {
    const int32_t c = z[u];
    int64_t nt = 0;
    for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
        const int32_t v = g->col[i];
        if (v == u)
            continue;
        const int32_t d = z[v];
        if (s->aff[d] == 0.0)
            s->touched[nt++] = d;
        s->aff[d] += g->w[i];
    }
    const double vol_u = g->vol[u];
    const double w_c = s->aff[c];
    const double vol_c = vols[c] - vol_u;
    double best_delta = 0.0;
    int32_t best = c;
    for (int64_t j = 0; j < nt; ++j) {
        const int32_t d = s->touched[j];
        if (d == c)
            continue;
        const double delta = (s->aff[d] - w_c) * inv_total + gamma * (vol_c - vols[d]) * vol_u * inv_sq2;
        if (delta > best_delta || (delta == best_delta && best != c && d < best)) {
            best_delta = delta;
            best = d;
        }
    }
    for (int64_t j = 0; j < nt; ++j)
        s->aff[s->touched[j]] = 0.0;
    *gain = best_delta;
    return best;
}

void cdo_move_eval(const cdo_graph *g, const int32_t *z, const double *vols, int64_t ub, double gamma,
                   int32_t *best, double *gain) {
    scratch_t s;
    scratch_init(&s, ub, max_degree(g));
    const double total = g->total;
    const double inv_total = 1.0 / total;
    const double inv_sq2 = 1.0 / (2.0 * total * total);
    for (int64_t u = 0; u < g->n; ++u) {
        double gval = 0.0;
        int32_t b = z[u];
        if (g->off[u + 1] > g->off[u] && total > 0.0) {
            b = move_best(g, z, vols, gamma, inv_total, inv_sq2, (int32_t)u, &s, &gval);
            if (!(b != z[u] && gval > 0.0)) {
                b = z[u];
                gval = 0.0;
            }
        }
        best[u] = b;
        gain[u] = gval;
    }
    scratch_free(&s);
}

/* move_phase (H/louvain.hpp:65-141) with one worker: passes over u = 0..n-1,
 * each move applied in place (z, vols) before the next node is evaluated;
 * stops after a pass without moves or max_passes.  Every applied move is
 * appended to the log (H/louvain.hpp:127-128's observer arguments). */
int cdo_move_phase_sequential(const cdo_graph *g, int32_t *z, int64_t ub, double gamma, int64_t max_passes,
                              cdo_move_log *log, int32_t *changed_out) {
    *changed_out = 0;
    if (log)
        log->count = 0;
    if (g->n == 0 || g->total == 0.0)
        return 0;
    for (int64_t u = 0; u < g->n; ++u)
        if (z[u] < 0 || z[u] >= ub)
            return CDO_ERANGE;
    scratch_t s;
    if (scratch_init(&s, ub, max_degree(g)))
        return CDO_ENOMEM;
    double *vols = (double *)calloc((size_t)ub, sizeof(double));
    if (!vols) {
        scratch_free(&s);
        return CDO_ENOMEM;
    }
    cdo_community_volumes(g, z, ub, vols);
    const double inv_total = 1.0 / g->total;
    const double inv_sq2 = 1.0 / (2.0 * g->total * g->total);
    for (int64_t pass = 0; pass < max_passes; ++pass) {
        int moved = 0;
        for (int64_t u = 0; u < g->n; ++u) {
            if (g->off[u + 1] == g->off[u])
                continue;
            const int32_t c = z[u];
            double gain = 0.0;
            const int32_t best = move_best(g, z, vols, gamma, inv_total, inv_sq2, (int32_t)u, &s, &gain);
            if (best != c && gain > 0.0) {
                vols[c] -= g->vol[u];
                vols[best] += g->vol[u];
                z[u] = best;
                moved = 1;
                if (log && log->count < log->capacity) {
                    log->node[log->count] = (int32_t)u;
                    log->source[log->count] = c;
                    log->target[log->count] = best;
                    log->gain[log->count] = gain;
                }
                if (log)
                    log->count++;
            }
        }
        if (!moved)
            break;
        *changed_out = 1;
    }
    free(vols);
    scratch_free(&s);
    return 0;
}

/* H/louvain.hpp:154-220.  Single worker: rows accumulate in (fine u asc,
 * row position asc) order; coarse rows sorted ascending; pi = z. */
int cdo_coarsen(const cdo_graph *g, const int32_t *z, cdo_graph *coarse) {
    const int64_t n = g->n;
    int64_t nc = 0;
    for (int64_t u = 0; u < n; ++u)
        if ((int64_t)z[u] + 1 > nc)
            nc = (int64_t)z[u] + 1;
    /* is_compact (H/partition.hpp:73-84) */
    uint8_t *used = (uint8_t *)calloc((size_t)(nc > 0 ? nc : 1), 1);
    for (int64_t u = 0; u < n; ++u) {
        if (z[u] < 0) {
            free(used);
            return CDO_EINVAL;
        }
        used[z[u]] = 1;
    }
    for (int64_t c = 0; c < nc; ++c)
        if (!used[c]) {
            free(used);
            return CDO_EINVAL;
        }
    free(used);
    /* members of each coarse node in ascending fine order */
    int64_t *moff = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    int32_t *mem = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t u = 0; u < n; ++u)
        moff[z[u] + 1]++;
    for (int64_t c = 0; c < nc; ++c)
        moff[c + 1] += moff[c];
    {
        int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
        memcpy(fill, moff, sizeof(int64_t) * (size_t)nc);
        for (int64_t u = 0; u < n; ++u)
            mem[fill[z[u]]++] = (int32_t)u;
        free(fill);
    }
    double *acc = (double *)calloc((size_t)(nc > 0 ? nc : 1), sizeof(double));
    uint8_t *hit = (uint8_t *)calloc((size_t)(nc > 0 ? nc : 1), 1);
    int32_t *touched = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nc > 0 ? nc : 1));
    int64_t cap = g->D + 1, D2 = 0;
    int32_t *col = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    double *wt = (double *)malloc(sizeof(double) * (size_t)cap);
    int64_t *off = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    for (int64_t c = 0; c < nc; ++c) {
        int64_t nt = 0;
        for (int64_t p = moff[c]; p < moff[c + 1]; ++p) {
            const int32_t u = mem[p];
            for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
                const int32_t v = g->col[i];
                const int32_t cv = z[v];
                if (cv == c && v < u)
                    continue; /* intra: each non-loop edge once (v >= u) */
                if (!hit[cv]) {
                    hit[cv] = 1;
                    touched[nt++] = cv;
                }
                acc[cv] += g->w[i];
            }
        }
        /* sort touched ascending (insertion into counting order) */
        for (int64_t a = 1; a < nt; ++a) {
            int32_t x = touched[a];
            int64_t b = a - 1;
            while (b >= 0 && touched[b] > x) {
                touched[b + 1] = touched[b];
                --b;
            }
            touched[b + 1] = x;
        }
        for (int64_t j = 0; j < nt; ++j) {
            col[D2] = touched[j];
            wt[D2++] = acc[touched[j]];
            acc[touched[j]] = 0.0;
            hit[touched[j]] = 0;
        }
        off[c + 1] = D2;
    }
    int rc = cdo_graph_from_csr(nc, off, col, wt, coarse);
    free(moff);
    free(mem);
    free(acc);
    free(hit);
    free(touched);
    free(col);
    free(wt);
    free(off);
    return rc;
}

/* H/louvain.hpp:223-233 */
int cdo_prolong(int64_t nc, const int32_t *zc, int64_t n, const int32_t *pi, int32_t *out) {
    for (int64_t v = 0; v < n; ++v) {
        if (pi[v] < 0 || pi[v] >= nc)
            return CDO_ERANGE;
        out[v] = zc[pi[v]];
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* ensemble                                                                 */
/* ------------------------------------------------------------------------ */

/* H/ensemble.hpp:75-80 */
uint64_t cdo_djb2(const uint8_t *data, uint64_t len) {
    uint64_t h = 5381;
    for (uint64_t i = 0; i < len; ++i)
        h = h * 33 + data[i];
    return h;
}

/* H/ensemble.hpp:86-107: djb2 over 8 LE bytes of each (zero-extended) id,
 * then first-appearance compaction of the 64-bit hashes. */
int64_t cdo_combine_hashed(int64_t b, int64_t n, const int32_t *const *solutions, int32_t *out) {
    if (b < 1)
        return CDO_EINVAL;
    uint64_t *h = (uint64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint64_t));
    uint64_t *idx = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t v = 0; v < n; ++v) {
        uint64_t x = 5381;
        for (int64_t i = 0; i < b; ++i) {
            uint64_t id = (uint64_t)(uint32_t)solutions[i][v];
            for (int byte = 0; byte < 8; ++byte) {
                x = x * 33 + (uint8_t)(id & 0xff);
                id >>= 8;
            }
        }
        h[v] = x;
        idx[v] = (uint64_t)v;
    }
    /* group equal hashes: sort (hash, node) pairs, first member = min node */
    uint64_t *hk = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
    memcpy(hk, h, sizeof(uint64_t) * (size_t)n);
    radix_sort_u64(hk, idx, n, 64);
    int64_t *first = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n;) {
        int64_t j = i;
        while (j < n && hk[j] == hk[i])
            ++j;
        for (int64_t t = i; t < j; ++t)
            first[idx[t]] = (int64_t)idx[i]; /* stable sort: idx[i] is the min node */
        i = j;
    }
    int32_t *rank = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t next = 0;
    for (int64_t v = 0; v < n; ++v)
        if (first[v] == v)
            rank[v] = next++;
    for (int64_t v = 0; v < n; ++v)
        out[v] = rank[first[v]];
    free(h);
    free(idx);
    free(hk);
    free(first);
    free(rank);
    return next;
}

/* ------------------------------------------------------------------------ */
/* ports of the device drivers                                              */
/* ------------------------------------------------------------------------ */

uint64_t cdo_bucket_key(uint64_t seed, uint64_t salt) {
    return cdo_splitmix64(seed ^ cdo_splitmix64(salt ^ 0xb5ad4eceda1ce2a9ULL));
}

int32_t cdo_bucket_of(uint64_t key, int32_t u, int32_t buckets) {
    return (int32_t)((uint32_t)(cdo_splitmix64(key ^ (uint64_t)(uint32_t)u) >> 32) % (uint32_t)buckets);
}

/* PLP salt = iteration index; see paper_1304_4453_b200/csrc/plp.cu. */
int cdo_plp_bucketed(const cdo_graph *g, const cdo_plp_config *cfg, const int32_t *initial, int32_t *labels,
                     int64_t *iterations, int64_t *updated_trace, int64_t trace_cap) {
    const int64_t n = g->n;
    const int64_t theta = cfg->theta >= 0 ? cfg->theta : (n / 100000 > 1 ? n / 100000 : 1);
    const int32_t K = cfg->buckets > 0 ? cfg->buckets : 1;
    for (int64_t u = 0; u < n; ++u)
        labels[u] = initial ? initial[u] : (int32_t)u;
    const int64_t ub = max_label_plus_one(n, labels);
    scratch_t s;
    if (scratch_init(&s, ub, max_degree(g))) {
        scratch_free(&s);
        return CDO_ENOMEM;
    }
    uint8_t *active = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    memset(active, 1, (size_t)(n > 0 ? n : 1));
    int32_t *mv_u = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *mv_l = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int64_t updated = n, iter = 0;
    while (updated > theta && iter < cfg->max_iterations) {
        updated = 0;
        const uint64_t key = cdo_bucket_key(cfg->seed, (uint64_t)iter);
        for (int32_t b = 0; b < K; ++b) {
            int64_t nm = 0;
            for (int64_t u = 0; u < n; ++u) {
                if (!active[u] || g->off[u + 1] == g->off[u])
                    continue;
                if (K > 1 && cdo_bucket_of(key, (int32_t)u, K) != b)
                    continue;
                const int32_t best = plp_best(g, labels, (int32_t)u, &s);
                if (best != labels[u]) {
                    mv_u[nm] = (int32_t)u;
                    mv_l[nm++] = best;
                } else {
                    active[u] = 0;
                }
            }
            for (int64_t j = 0; j < nm; ++j) {
                const int32_t u = mv_u[j];
                labels[u] = mv_l[j];
                for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i)
                    active[g->col[i]] = 1;
            }
            updated += nm;
        }
        if (updated_trace && iter < trace_cap)
            updated_trace[iter] = updated;
        ++iter;
    }
    *iterations = iter;
    scratch_free(&s);
    free(active);
    free(mv_u);
    free(mv_l);
    return 0;
}

/* One PLP sub-sweep restricted to the nodes [lo, hi) one rank owns (the
 * sharded protocol of the device drivers): evaluates the
 * bucket's active nodes against the frozen labels, deactivates non-movers
 * and returns the moves without applying them.  The caller concatenates the
 * ranks' moves in rank order and applies them as cdo_plp_bucketed does. */
int64_t cdo_plp_subsweep(const cdo_graph *g, const int32_t *labels, uint8_t *active, uint64_t key, int32_t bucket,
                         int32_t buckets, int64_t lo, int64_t hi, int32_t *mv_u, int32_t *mv_l) {
    scratch_t s;
    if (scratch_init(&s, max_label_plus_one(g->n, labels), max_degree(g))) {
        scratch_free(&s);
        return CDO_ENOMEM;
    }
    int64_t nm = 0;
    for (int64_t u = lo; u < hi; ++u) {
        if (!active[u] || g->off[u + 1] == g->off[u])
            continue;
        if (buckets > 1 && cdo_bucket_of(key, (int32_t)u, buckets) != bucket)
            continue;
        const int32_t best = plp_best(g, labels, (int32_t)u, &s);
        if (best != labels[u]) {
            mv_u[nm] = (int32_t)u;
            mv_l[nm++] = best;
        } else {
            active[u] = 0;
        }
    }
    scratch_free(&s);
    return nm;
}

void cdo_activate(const cdo_graph *g, int64_t nm, const int32_t *mv_u, uint8_t *active) {
    if (nm > g->n / 16) { /* dense activation (device k_apply_*) */
        memset(active, 1, (size_t)g->n);
        return;
    }
    for (int64_t j = 0; j < nm; ++j) {
        const int32_t u = mv_u[j];
        for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i)
            active[g->col[i]] = 1;
    }
}

/* One move-phase sub-sweep over [lo, hi) against frozen (z, vols, csize);
 * the decision rule of cdo_move_phase_bucketed; moves are returned.  With
 * cfg->prune, only active nodes are evaluated and non-movers deactivated. */
int64_t cdo_move_subsweep(const cdo_graph *g, const int32_t *z, const double *vols, const int32_t *csize,
                          uint8_t *active, const cdo_louvain_config *cfg, uint64_t key, int32_t bucket, int64_t lo,
                          int64_t hi, int32_t *mv_u, int32_t *mv_l, long long *gain_fx) {
    if (gain_fx)
        *gain_fx = 0;
    const int32_t K = cfg->buckets > 0 ? cfg->buckets : 1;
    const double inv_total = 1.0 / g->total;
    const double inv_sq2 = 1.0 / (2.0 * g->total * g->total);
    scratch_t s;
    if (scratch_init(&s, g->n, max_degree(g))) {
        scratch_free(&s);
        return CDO_ENOMEM;
    }
    const int prune = cfg->prune && active;
    int64_t nm = 0;
    for (int64_t u = lo; u < hi; ++u) {
        if (g->off[u + 1] == g->off[u])
            continue;
        if (K > 1 && cdo_bucket_of(key, (int32_t)u, K) != bucket)
            continue;
        if (prune && !active[u])
            continue;
        double gain;
        const int32_t c = z[u];
        const int32_t best = move_best(g, z, vols, cfg->gamma, inv_total, inv_sq2, (int32_t)u, &s, &gain);
        int moved = best != c && gain > 0.0;
        if (moved && cfg->singleton_guard && csize[c] == 1 && csize[best] == 1 && best > c)
            moved = 0;
        if (!moved) {
            if (prune)
                active[u] = 0;
            continue;
        }
        mv_u[nm] = (int32_t)u;
        mv_l[nm++] = best;
        if (gain_fx)
            *gain_fx += llrint(gain * CDO_GAIN_FX_SCALE);
    }
    scratch_free(&s);
    return nm;
}

/* The device's default schedule (paper_1304_4453_b200/csrc/detect.cu
 * resolve_louvain_schedule): buckets <= 0 and move_qtol < 0 mean "by graph":
 * a skewed graph (max degree > 4096: R-MAT-like hubs) takes 8 buckets and
 * a gain tolerance of 5e-3, anything else 4 and 2e-3.  Resolved once on the
 * graph a run starts from; every level of the run uses the same values. */
static cdo_louvain_config resolve_schedule(const cdo_louvain_config *cfg, const cdo_graph *g) {
    cdo_louvain_config c = *cfg;
    const int skewed = max_degree(g) > 4096;
    if (c.buckets <= 0)
        c.buckets = skewed ? 8 : 4;
    if (c.move_qtol < 0.0)
        c.move_qtol = skewed ? 5e-3 : 2e-3;
    return c;
}

static int move_phase_impl(const cdo_graph *g, int32_t *z, const cdo_louvain_config *cfg, uint64_t salt,
                           int32_t *changed_out);

/* Bucketed move phase: the order of paper_1304_4453_b200/csrc/detect.cu move_phase_dev. */
int cdo_move_phase_bucketed(const cdo_graph *g, int32_t *z, const cdo_louvain_config *cfg, uint64_t salt,
                            int32_t *changed_out) {
    const cdo_louvain_config c = resolve_schedule(cfg, g);
    return move_phase_impl(g, z, &c, salt, changed_out);
}

static int move_phase_impl(const cdo_graph *g, int32_t *z, const cdo_louvain_config *cfg, uint64_t salt,
                           int32_t *changed_out) {
    const int64_t n = g->n;
    *changed_out = 0;
    if (n == 0 || g->total == 0.0)
        return 0;
    const int32_t K = cfg->buckets > 0 ? cfg->buckets : 1;
    const int64_t ub = n; /* device labels are always < n */
    for (int64_t u = 0; u < n; ++u)
        if (z[u] < 0 || z[u] >= ub)
            return CDO_ERANGE;
    const double total = g->total;
    const double inv_total = 1.0 / total;
    const double inv_sq2 = 1.0 / (2.0 * total * total);
    int64_t theta = cfg->move_theta >= 0 ? cfg->move_theta : n / 100000;
    if ((int64_t)(cfg->move_tol * (double)n) > theta)
        theta = (int64_t)(cfg->move_tol * (double)n);
    double *vols = (double *)malloc(sizeof(double) * (size_t)ub);
    int32_t *csize = (int32_t *)calloc((size_t)ub, sizeof(int32_t));
    cdo_community_volumes(g, z, ub, vols);
    for (int64_t u = 0; u < n; ++u)
        csize[z[u]]++;
    scratch_t s;
    scratch_init(&s, ub, max_degree(g));
    int32_t *mv_u = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *mv_l = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    uint8_t *active = NULL;
    if (cfg->prune) {
        active = (uint8_t *)malloc((size_t)n);
        memset(active, 1, (size_t)n);
    }
    int changed = 0;
    int64_t hist0 = -1, hist1 = -1; /* moves two passes / one pass earlier */
    long long cum_fx = 0;           /* the phase's summed gain, fixed point 2^-44 */
    for (int64_t pass = 0; pass < cfg->max_move_iterations; ++pass) {
        int64_t moved = 0;
        long long pass_fx = 0;
        const uint64_t key = cdo_bucket_key(cfg->seed, salt + (uint64_t)pass);
        for (int32_t b = 0; b < K; ++b) {
            int64_t nm = 0;
            for (int64_t u = 0; u < n; ++u) {
                if (g->off[u + 1] == g->off[u])
                    continue;
                if (K > 1 && cdo_bucket_of(key, (int32_t)u, K) != b)
                    continue;
                if (active && !active[u])
                    continue;
                double gain;
                const int32_t c = z[u];
                const int32_t best = move_best(g, z, vols, cfg->gamma, inv_total, inv_sq2, (int32_t)u, &s, &gain);
                int mv = best != c && gain > 0.0;
                if (mv && cfg->singleton_guard && csize[c] == 1 && csize[best] == 1 && best > c)
                    mv = 0;
                if (!mv) {
                    if (active)
                        active[u] = 0; /* pruned until a neighbour moves */
                    continue;
                }
                mv_u[nm] = (int32_t)u;
                mv_l[nm++] = best;
                pass_fx += llrint(gain * CDO_GAIN_FX_SCALE);
            }
            for (int64_t j = 0; j < nm; ++j) {
                const int32_t u = mv_u[j], d = mv_l[j], c = z[u];
                vols[c] -= g->vol[u];
                vols[d] += g->vol[u];
                csize[c]--;
                csize[d]++;
                z[u] = d;
            }
            if (active)
                cdo_activate(g, nm, mv_u, active);
            moved += nm;
        }
        if (moved == 0)
            break;
        changed = 1;
        if (moved <= theta)
            break;
        if (cfg->move_stall > 0.0 && pass >= 8 && (double)moved > cfg->move_stall * (double)hist0)
            break;
        cum_fx += pass_fx;
        if (cfg->move_qtol > 0.0 && (double)pass_fx <= cfg->move_qtol * (double)cum_fx)
            break;
        hist0 = hist1;
        hist1 = moved;
    }
    *changed_out = changed;
    free(active);
    free(vols);
    free(csize);
    scratch_free(&s);
    free(mv_u);
    free(mv_l);
    return 0;
}

/* coarse weights are stored as fp32 on the device */
static void round_weights_to_float(cdo_graph *g) {
    for (int64_t i = 0; i < g->D; ++i)
        g->w[i] = (double)(float)g->w[i];
    cdo_finalize(g);
}

static uint64_t louvain_salt(int64_t level, int phase) {
    return (1ULL << 62) | ((uint64_t)level << 40) | ((uint64_t)phase << 32);
}

/* H/louvain.hpp:237-267 with the bucketed move phase */
static int louvain_recurse(const cdo_graph *g, const cdo_louvain_config *cfg, int64_t level, int32_t *z,
                           int64_t *levels) {
    const int64_t n = g->n;
    if (level + 1 > *levels)
        *levels = level + 1;
    for (int64_t u = 0; u < n; ++u)
        z[u] = (int32_t)u;
    int32_t changed = 0;
    /* pruning: 1 = the input graph's move phases only, 2 = every level */
    cdo_louvain_config lc = *cfg;
    if (level > 0 && lc.prune < 2)
        lc.prune = 0;
    cfg = &lc;
    int rc = move_phase_impl(g, z, cfg, louvain_salt(level, 0), &changed);
    if (rc)
        return rc;
    if (changed && level + 1 < cfg->max_levels) {
        int32_t *zc = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        const int64_t k = cdo_compact(n, z, zc);
        if (k < n) {
            cdo_graph coarse;
            rc = cdo_coarsen(g, zc, &coarse);
            if (rc) {
                free(zc);
                return rc;
            }
            round_weights_to_float(&coarse);
            int32_t *zcoarse = (int32_t *)malloc(sizeof(int32_t) * (size_t)(k > 0 ? k : 1));
            rc = louvain_recurse(&coarse, cfg, level + 1, zcoarse, levels);
            if (!rc)
                rc = cdo_prolong(k, zcoarse, n, zc, z);
            free(zcoarse);
            cdo_graph_free(&coarse);
            if (!rc && cfg->refine) {
                int32_t ch2;
                rc = move_phase_impl(g, z, cfg, louvain_salt(level, 1), &ch2);
            }
        }
        free(zc);
    }
    return rc;
}

int cdo_louvain_bucketed(const cdo_graph *g, const cdo_louvain_config *cfg, int32_t *z, int64_t *k,
                         int64_t *levels) {
    if (g->total == 0.0)
        return CDO_EDOMAIN;
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
    *levels = 0;
    const cdo_louvain_config c = resolve_schedule(cfg, g);
    int rc = louvain_recurse(g, &c, 0, tmp, levels);
    if (!rc)
        *k = cdo_compact(g->n, tmp, z);
    free(tmp);
    return rc;
}

/* H/ensemble.hpp:111-199 with bucketed bases and final PLMR */
int cdo_epp_bucketed(const cdo_graph *g, int64_t b, uint64_t seed, const cdo_plp_config *base,
                     const cdo_louvain_config *final_cfg, int32_t *z, int64_t *k) {
    if (b < 1)
        return CDO_EINVAL;
    if (g->total == 0.0)
        return CDO_EDOMAIN;
    const int64_t n = g->n;
    int32_t **bases = (int32_t **)malloc(sizeof(int32_t *) * (size_t)b);
    int rc = 0;
    for (int64_t i = 0; i < b; ++i) {
        bases[i] = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        cdo_plp_config pc = *base;
        pc.seed = seed + (uint64_t)i;
        int64_t iters;
        rc = cdo_plp_bucketed(g, &pc, NULL, bases[i], &iters, NULL, 0);
        if (rc)
            break;
    }
    int32_t *core = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!rc)
        cdo_combine_hashed(b, n, (const int32_t *const *)bases, core);
    cdo_graph coarse;
    memset(&coarse, 0, sizeof(coarse));
    if (!rc)
        rc = cdo_coarsen(g, core, &coarse);
    if (!rc) {
        round_weights_to_float(&coarse);
        cdo_louvain_config fc = *final_cfg;
        fc.seed = seed;
        fc.refine = 1;
        int32_t *zc = (int32_t *)malloc(sizeof(int32_t) * (size_t)(coarse.n > 0 ? coarse.n : 1));
        int64_t kc, lv;
        if (coarse.total == 0.0) {
            for (int64_t c = 0; c < coarse.n; ++c)
                zc[c] = (int32_t)c;
        } else {
            rc = cdo_louvain_bucketed(&coarse, &fc, zc, &kc, &lv);
        }
        int32_t *fine = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
        if (!rc)
            rc = cdo_prolong(coarse.n, zc, n, core, fine);
        if (!rc)
            *k = cdo_compact(n, fine, z);
        free(zc);
        free(fine);
    }
    cdo_graph_free(&coarse);
    for (int64_t i = 0; i < b; ++i)
        free(bases[i]);
    free(bases);
    free(core);
    return rc;
}
