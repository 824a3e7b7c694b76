// text.cu -- device ingest of the reference's text formats (SURVEY.md §8(f)
// rank 1): read_metis (H/io.hpp:83-165) and read_edge_list (H/io.hpp:190-237).
//
// The whole file sits in device memory; lines and tokens are found with
// scans over byte flags, every token is parsed by its own thread (strict
// std::from_chars rules: unsigned decimal integers; decimal floating point
// with optional fraction / exponent, inf / nan), and the result goes through
// the same CSR builder as cd_graph_from_edges.  Validation follows the
// reference rule by rule and reports the reference's first error (the
// earliest line / token in its order of checks):
//   METIS: header "n m [fmt]" (fmt 1 = edge weights, other codes rejected);
//   '%' lines skipped; n adjacency lines (1-based ids, weights > 0, an even
//   token count when weighted); only the first non-comment line after them is
//   checked for trailing content; every (u, v, w) with v > u needs v's
//   smallest weight towards u to equal w; duplicates rejected; the edge
//   count must equal the header's m.
//   Edge list: '#' starts a comment; lines of 0, 2 or 3 tokens; ids are
//   densified in ascending numeric order (kept for cd_graph_original_ids);
//   duplicates rejected unless merged.
// Weights are parsed as fp64 (exactly for literals with <= 19 significant
// digits and |exponent| <= 22, the common case; otherwise to within one ulp
// before the fp32 storage rounding) and stored as fp32 like every device
// graph.
#include <cstdio>
#include <string>

#include "graph.cuh"
#include "scan.cuh"
#include "sort.cuh"

namespace cdk {

namespace {

// Weights are stored as fp32 (rounded to nearest).  A positive finite fp64
// weight below the smallest fp32 subnormal would round to 0 (breaking the
// w > 0 invariant, H/graph.hpp:52-53) and one beyond FLT_MAX to inf; both
// are rejected like a nonpositive weight.  A literal inf is accepted, as the
// reference's `w > 0` accepts it.
__device__ __host__ __forceinline__ bool fp32_weight_ok(double w) {
    const float f = static_cast<float>(w);
    return f > 0.0f && (f <= 3.402823466e38f || isinf(w));
}

__device__ __host__ __forceinline__ bool is_ws(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// std::from_chars(uint64): decimal digits only, whole token, no overflow
__device__ __host__ inline bool parse_u64(const char *p, int len, uint64_t &out) {
    if (len <= 0)
        return false;
    uint64_t v = 0;
    for (int i = 0; i < len; ++i) {
        const unsigned d = static_cast<unsigned char>(p[i]) - '0';
        if (d > 9)
            return false;
        if (v > (UINT64_MAX - d) / 10)
            return false;
        v = v * 10 + d;
    }
    out = v;
    return true;
}

__device__ __forceinline__ char lower(char c) { return (c >= 'A' && c <= 'Z') ? static_cast<char>(c + 32) : c; }

__device__ bool match_word(const char *p, int len, int &i, const char *w) {
    int k = 0;
    while (w[k]) {
        if (i + k >= len || lower(p[i + k]) != w[k])
            return false;
        ++k;
    }
    i += k;
    return true;
}

// std::from_chars(double, chars_format::general): [-] (digits [. digits] | . digits)
// [e|E [+|-] digits] | [-] inf | infinity | nan [ (chars) ]
__device__ bool parse_f64(const char *p, int len, double &out) {
    int i = 0;
    bool neg = false;
    if (i < len && p[i] == '-') {
        neg = true;
        ++i;
    }
    if (i < len && (lower(p[i]) == 'i' || lower(p[i]) == 'n')) {
        int j = i;
        if (match_word(p, len, j, "infinity") || (j = i, match_word(p, len, j, "inf"))) {
            if (j != len)
                return false;
            out = neg ? -INFINITY : INFINITY;
            return true;
        }
        j = i;
        if (match_word(p, len, j, "nan")) {
            if (j < len && p[j] == '(') {
                while (j < len && p[j] != ')')
                    ++j;
                if (j >= len)
                    return false;
                ++j;
            }
            if (j != len)
                return false;
            out = NAN;
            return true;
        }
        return false;
    }
    uint64_t mant = 0;
    int digits = 0, exp10 = 0;
    bool any = false, inexact = false;
    while (i < len && p[i] >= '0' && p[i] <= '9') {
        any = true;
        if (mant == 0 && p[i] == '0') {
            ++i;
            continue;
        }
        if (digits < 19) {
            mant = mant * 10 + (p[i] - '0');
            ++digits;
        } else {
            ++exp10;
            inexact |= p[i] != '0';
        }
        ++i;
    }
    if (i < len && p[i] == '.') {
        ++i;
        while (i < len && p[i] >= '0' && p[i] <= '9') {
            any = true;
            if (mant == 0 && p[i] == '0') {
                --exp10;
            } else if (digits < 19) {
                mant = mant * 10 + (p[i] - '0');
                ++digits;
                --exp10;
            } else {
                inexact |= p[i] != '0';
            }
            ++i;
        }
    }
    if (!any)
        return false;
    if (i < len && lower(p[i]) == 'e') {
        int j = i + 1;
        bool eneg = false;
        if (j < len && (p[j] == '+' || p[j] == '-')) {
            eneg = p[j] == '-';
            ++j;
        }
        if (j < len && p[j] >= '0' && p[j] <= '9') {
            int e = 0;
            while (j < len && p[j] >= '0' && p[j] <= '9') {
                if (e < 100000)
                    e = e * 10 + (p[j] - '0');
                ++j;
            }
            exp10 += eneg ? -e : e;
            i = j;
        }  // a bare 'e' is not part of the number (then the token is not fully consumed)
    }
    if (i != len)
        return false;
    double v;
    if (mant == 0) {
        v = 0.0;
    } else if (!inexact && mant <= (uint64_t(1) << 53) && exp10 >= -22 && exp10 <= 22) {
        // exact: both operands are exact doubles, one correctly rounded op
        const double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
        v = exp10 >= 0 ? static_cast<double>(mant) * p10[exp10] : static_cast<double>(mant) / p10[-exp10];
    } else {
        v = static_cast<double>(mant) * pow(10.0, static_cast<double>(exp10));
    }
    out = neg ? -v : v;
    return true;
}

// ---- text indexing -----------------------------------------------------------
struct LineStartFlag {
    const char *t;
    __device__ int64_t operator()(int64_t i) const { return (i == 0 || t[i - 1] == '\n') ? 1 : 0; }
};
struct TokStartFlag {
    const char *t;
    __device__ int64_t operator()(int64_t i) const { return (!is_ws(t[i]) && (i == 0 || is_ws(t[i - 1]))) ? 1 : 0; }
};

template <class F>
__global__ void k_scatter_flags(int64_t n, F f, const int64_t *rank, int64_t *pos) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (f(i))
            pos[rank[i]] = i;
}

__device__ __forceinline__ int64_t upper_bound_i64(const int64_t *a, int64_t n, int64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// token lengths and lines
__global__ void k_tok_info(int64_t ntok, const char *t, int64_t len, const int64_t *tok_start,
                           const int64_t *line_start, int64_t nlines, int32_t *tok_len, int64_t *tok_line) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < ntok;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = tok_start[k];
        int64_t e = s;
        while (e < len && !is_ws(t[e]))
            ++e;
        tok_len[k] = static_cast<int32_t>(e - s < INT32_MAX ? e - s : INT32_MAX);
        tok_line[k] = upper_bound_i64(line_start, nlines, s) - 1;
    }
}

// first token of every line (tokens are in line order): line_tok[l] = lower_bound(tok_line, l)
__global__ void k_line_tok(int64_t nlines, const int64_t *tok_line, int64_t ntok, int64_t *line_tok) {
    for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l <= nlines;
         l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t lo = 0, hi = ntok;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (tok_line[mid] < l)
                lo = mid + 1;
            else
                hi = mid;
        }
        line_tok[l] = lo;
    }
}

// edge lists: everything from the first '#' of a line to its end is blank
__global__ void k_blank_comments(int64_t nlines, const int64_t *line_start, int64_t len, char *t) {
    for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nlines;
         l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t e = l + 1 < nlines ? line_start[l + 1] - 1 : len;
        bool in = false;
        for (int64_t i = line_start[l]; i < e; ++i) {
            if (t[i] == '#')
                in = true;
            if (in)
                t[i] = ' ';
        }
    }
}

struct Text {
    int64_t len = 0, nlines = 0, ntok = 0;
    DBuf<char> buf;
    DBuf<int64_t> line_start;  // [nlines]
    DBuf<int64_t> tok_start, tok_line;
    DBuf<int32_t> tok_len;
    DBuf<int64_t> line_tok;  // [nlines + 1]
};

void index_lines(cd_ctx *ctx, Text &T) {
    const int64_t len = T.len;
    DBuf<int64_t> rank(ctx, len + 1);
    exclusive_scan<int64_t>(ctx, len, LineStartFlag{T.buf.p}, rank.p, rank.p + len);
    CD_CUDA(cudaMemcpyAsync(&T.nlines, rank.p + len, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    T.line_start.alloc(ctx, std::max<int64_t>(T.nlines, 1));
    if (len)
        CD_LAUNCH(ctx, "ingest", k_scatter_flags<LineStartFlag>, grid_for(len, 256, ctx->num_sms * 16), 256, 0, len,
                  LineStartFlag{T.buf.p}, static_cast<const int64_t *>(rank.p), T.line_start.p);
}

void index_tokens(cd_ctx *ctx, Text &T) {
    const int64_t len = T.len;
    DBuf<int64_t> rank(ctx, len + 1);
    exclusive_scan<int64_t>(ctx, len, TokStartFlag{T.buf.p}, rank.p, rank.p + len);
    CD_CUDA(cudaMemcpyAsync(&T.ntok, rank.p + len, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    T.tok_start.alloc(ctx, std::max<int64_t>(T.ntok, 1));
    T.tok_line.alloc(ctx, std::max<int64_t>(T.ntok, 1));
    T.tok_len.alloc(ctx, std::max<int64_t>(T.ntok, 1));
    T.line_tok.alloc(ctx, T.nlines + 1);
    if (len)
        CD_LAUNCH(ctx, "ingest", k_scatter_flags<TokStartFlag>, grid_for(len, 256, ctx->num_sms * 16), 256, 0, len,
                  TokStartFlag{T.buf.p}, static_cast<const int64_t *>(rank.p), T.tok_start.p);
    if (T.ntok)
        CD_LAUNCH(ctx, "ingest", k_tok_info, grid_for(T.ntok, 256, ctx->num_sms * 16), 256, 0, T.ntok,
                  static_cast<const char *>(T.buf.p), len, static_cast<const int64_t *>(T.tok_start.p),
                  static_cast<const int64_t *>(T.line_start.p), T.nlines, T.tok_len.p, T.tok_line.p);
    CD_LAUNCH(ctx, "ingest", k_line_tok, grid_for(T.nlines + 1, 256, ctx->num_sms * 16), 256, 0, T.nlines,
              static_cast<const int64_t *>(T.tok_line.p), T.ntok, T.line_tok.p);
}

void load_text(cd_ctx *ctx, Text &T, const char *text, int64_t len) {
    T.len = len;
    T.buf.alloc(ctx, std::max<int64_t>(len, 1));
    if (len)
        CD_CUDA(cudaMemcpyAsync(T.buf.p, text, len, cudaMemcpyDefault, ctx->stream));
}

template <class T>
T read1(cd_ctx *ctx, const T *p) {
    T h;
    CD_CUDA(cudaMemcpyAsync(&h, p, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    return h;
}

// first error (smallest key) of a parallel validation pass
struct ErrSlot {
    DBuf<unsigned long long> v;
    explicit ErrSlot(cd_ctx *ctx) : v(ctx, 1) { v.fill_bytes(0xff); }
    unsigned long long get(cd_ctx *ctx) { return read1(ctx, v.p); }
};
constexpr unsigned long long NO_ERR = ~0ULL;

// ---- METIS -----------------------------------------------------------------------
struct NonCommentFlag {
    const char *t;
    const int64_t *line_start;
    int64_t nlines, len;
    __device__ int64_t operator()(int64_t l) const {
        const int64_t s = line_start[l];
        const int64_t e = l + 1 < nlines ? line_start[l + 1] - 1 : len;
        return (e > s && t[s] == '%') ? 0 : 1;
    }
};

__global__ void k_ordinal_lines(int64_t nlines, NonCommentFlag f, const int64_t *rank, int64_t *line_of) {
    for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nlines;
         l += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (f(l))
            line_of[rank[l]] = l;
}

struct MetisLines {
    const int64_t *line_of;  // ordinal -> line (ordinal 0 = header)
    const int64_t *line_tok;
};

// entries per adjacency line u; dangling weight token -> error (line, 0, code 5)
__global__ void k_metis_count(int64_t n, MetisLines M, int stride, int64_t *cnt, unsigned long long *err) {
    for (int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < n;
         u += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t l = M.line_of[u + 1];
        const int64_t c = M.line_tok[l + 1] - M.line_tok[l];
        cnt[u] = c / stride;
        if (c % stride)
            atomicMin(err, (static_cast<unsigned long long>(l) << 24) | 5ULL);
    }
}

struct CountGen64 {
    const int64_t *c;
    __device__ int64_t operator()(int64_t i) const { return c[i]; }
};

// codes: 1 malformed id, 2 id out of range, 3 malformed weight, 4 weight <= 0
__global__ void k_metis_entries(int64_t nadj, int64_t n, MetisLines M, const char *t, const int64_t *tok_start,
                                const int32_t *tok_len, int weighted, const int64_t *eoff, int32_t *eu, int32_t *ev,
                                double *ew, unsigned long long *err) {
    const int lane = lane_id();
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int stride = weighted ? 2 : 1;
    for (int64_t u = gw; u < nadj; u += nw) {
        const int64_t l = M.line_of[u + 1];
        const int64_t t0 = M.line_tok[l];
        const int64_t ne = eoff[u + 1] - eoff[u];
        for (int64_t j = lane; j < ne; j += 32) {
            const int64_t k = t0 + j * stride;
            const int64_t e = eoff[u] + j;
            uint64_t v1 = 0;
            int code = 0;
            int which = 0;
            if (!parse_u64(t + tok_start[k], tok_len[k], v1)) {
                code = 1;
            } else if (v1 < 1 || v1 > static_cast<uint64_t>(n)) {
                code = 2;
            }
            double w = 1.0;
            if (!code && weighted) {
                which = 1;
                if (!parse_f64(t + tok_start[k + 1], tok_len[k + 1], w))
                    code = 3;
                else if (!(w > 0.0))
                    code = 4;
                else if (!fp32_weight_ok(w))
                    code = 6;
            }
            if (code) {
                const unsigned long long tok = static_cast<unsigned long long>(j * stride + which + 1);
                atomicMin(err, (static_cast<unsigned long long>(l) << 24) | ((tok < (1u << 19) ? tok : (1u << 19) - 1)
                                                                            << 4) | code);
                v1 = 1;
            }
            eu[e] = static_cast<int32_t>(u);
            ev[e] = static_cast<int32_t>(v1 - 1);
            ew[e] = w;
        }
    }
}

// lower entries (v < u) keyed by (v, u); upper entries (v >= u) kept for the build
__global__ void k_metis_split(int64_t D, const int32_t *eu, const int32_t *ev, uint64_t *lkey, uint32_t *lidx,
                              int32_t *uu, int32_t *uv, const double *ew, float *uw, int64_t *counters) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < D;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t u = eu[e], v = ev[e];
        if (v < u) {
            const int64_t p = atomicAdd(reinterpret_cast<unsigned long long *>(&counters[0]), 1ULL);
            lkey[p] = (static_cast<uint64_t>(v) << 32) | static_cast<uint32_t>(u);
            lidx[p] = static_cast<uint32_t>(e);
        } else {
            const int64_t p = atomicAdd(reinterpret_cast<unsigned long long *>(&counters[1]), 1ULL);
            uu[p] = u;
            uv[p] = v;
            if (uw)
                uw[p] = static_cast<float>(ew[e]);
        }
    }
}

// after sorting the lower keys: min weight of every key run, at the run head
__global__ void k_run_min(int64_t L, const uint64_t *lkey, const uint32_t *lidx, const double *ew, double *minw) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < L;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i > 0 && lkey[i - 1] == lkey[i]) {
            minw[i] = 0.0;
            continue;
        }
        double m = ew[lidx[i]];
        for (int64_t j = i + 1; j < L && lkey[j] == lkey[i]; ++j)
            m = fmin(m, ew[lidx[j]]);
        minw[i] = m;
    }
}

// every upper entry (u, v > u, w): the reverse's smallest weight must be w
__global__ void k_metis_symmetry(int64_t D, const int32_t *eu, const int32_t *ev, const double *ew, int64_t L,
                                 const uint64_t *lkey, const double *minw, unsigned long long *err) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < D;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t u = eu[e], v = ev[e];
        if (v <= u)
            continue;
        const uint64_t key = (static_cast<uint64_t>(u) << 32) | static_cast<uint32_t>(v);
        int64_t lo = 0, hi = L;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (lkey[mid] < key)
                lo = mid + 1;
            else
                hi = mid;
        }
        if (lo >= L || lkey[lo] != key || minw[lo] != ew[e])
            atomicMin(err, key);
    }
}

std::vector<std::string> split_ws_host(const std::string &s) {
    std::vector<std::string> out;
    size_t i = 0;
    while (i < s.size()) {
        while (i < s.size() && is_ws(s[i]))
            ++i;
        size_t j = i;
        while (j < s.size() && !is_ws(s[j]))
            ++j;
        if (j > i)
            out.push_back(s.substr(i, j - i));
        i = j;
    }
    return out;
}

std::string line_text(cd_ctx *ctx, const Text &T, int64_t l, int64_t max_bytes) {
    int64_t se[2];
    CD_CUDA(cudaMemcpyAsync(&se[0], T.line_start.p + l, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    se[1] = T.len;
    if (l + 1 < T.nlines)
        CD_CUDA(cudaMemcpyAsync(&se[1], T.line_start.p + l + 1, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    int64_t e = se[1];
    if (l + 1 < T.nlines)
        --e;  // drop '\n'
    const int64_t nbytes = std::min<int64_t>(e - se[0], max_bytes);
    std::string s(static_cast<size_t>(std::max<int64_t>(nbytes, 0)), ' ');
    if (nbytes > 0) {
        CD_CUDA(cudaMemcpyAsync(&s[0], T.buf.p + se[0], nbytes, cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return s;
}

uint64_t parse_uint_host(const std::string &tok, const std::string &where) {
    uint64_t v = 0;
    if (!parse_u64(tok.data(), static_cast<int>(tok.size()), v))
        fail(CD_EINPUT, "malformed integer '" + tok + "' in " + where);
    return v;
}

}  // namespace

// H/io.hpp:83-165
cd_graph *read_metis_dev(cd_ctx *ctx, const char *text, int64_t len, const std::string &name) {
    Text T;
    load_text(ctx, T, text, len);
    index_lines(ctx, T);
    // non-comment lines in order: ordinal 0 = header, 1..n = adjacency lines
    const int64_t nlines = T.nlines;
    DBuf<int64_t> rank(ctx, nlines + 1);
    NonCommentFlag ncf{T.buf.p, T.line_start.p, nlines, T.len};
    exclusive_scan<int64_t>(ctx, nlines, ncf, rank.p, rank.p + nlines);
    const int64_t nc = read1(ctx, rank.p + nlines);
    if (nc == 0)
        fail(CD_EINPUT, name + ": unexpected end of file");
    DBuf<int64_t> line_of(ctx, nc);
    CD_LAUNCH(ctx, "ingest", k_ordinal_lines, grid_for(nlines, 256, ctx->num_sms * 16), 256, 0, nlines, ncf,
              static_cast<const int64_t *>(rank.p), line_of.p);
    // header (host: a few bytes)
    const int64_t hl = read1(ctx, line_of.p);
    const auto header = split_ws_host(line_text(ctx, T, hl, 4096));
    if (header.size() < 2 || header.size() > 3)
        fail(CD_EINPUT, name + ": malformed header");
    const uint64_t n = parse_uint_host(header[0], name + " header");
    const uint64_t m = parse_uint_host(header[1], name + " header");
    bool weighted = false;
    if (header.size() == 3) {
        const uint64_t fmt = parse_uint_host(header[2], name + " header");
        if (fmt == 1)
            weighted = true;
        else if (fmt != 0)
            fail(CD_EINPUT, name + ": unsupported fmt code " + std::to_string(fmt) +
                                " (node weights are not supported)");
    }
    if (n >= static_cast<uint64_t>(INT32_MAX))
        fail(CD_EINVAL, name + ": device node ids are int32 (n < 2^31 - 1)");
    index_tokens(ctx, T);
    const int64_t nn = static_cast<int64_t>(n);
    const int64_t nadj = std::min<int64_t>(nn, nc - 1);  // adjacency lines present
    MetisLines ML{line_of.p, T.line_tok.p};
    const int stride = weighted ? 2 : 1;
    ErrSlot err(ctx);
    DBuf<int64_t> cnt(ctx, std::max<int64_t>(nadj, 1)), eoff(ctx, nadj + 1);
    if (nadj)
        CD_LAUNCH(ctx, "ingest", k_metis_count, grid_for(nadj, 256, ctx->num_sms * 16), 256, 0, nadj, ML, stride,
                  cnt.p, err.v.p);
    exclusive_scan<int64_t>(ctx, nadj, CountGen64{cnt.p}, eoff.p, eoff.p + nadj);
    const int64_t D = read1(ctx, eoff.p + nadj);
    DBuf<int32_t> eu(ctx, std::max<int64_t>(D, 1)), ev(ctx, std::max<int64_t>(D, 1));
    DBuf<double> ew(ctx, std::max<int64_t>(D, 1));
    if (nadj)
        CD_LAUNCH(ctx, "ingest", k_metis_entries, grid_for(nadj, 8, ctx->num_sms * 16), 256, 0, nadj, nn, ML,
                  static_cast<const char *>(T.buf.p), static_cast<const int64_t *>(T.tok_start.p),
                  static_cast<const int32_t *>(T.tok_len.p), int(weighted), static_cast<const int64_t *>(eoff.p),
                  eu.p, ev.p, ew.p, err.v.p);
    const unsigned long long e1 = err.get(ctx);
    if (e1 != NO_ERR) {
        const int64_t l = static_cast<int64_t>(e1 >> 24);
        const int code = static_cast<int>(e1 & 15);
        const std::string where = name + ":" + std::to_string(l + 1);
        if (code == 5)
            fail(CD_EINPUT, where + ": dangling weight token");
        // re-derive the message from the offending token on the host
        const auto toks = split_ws_host(line_text(ctx, T, l, INT64_MAX));
        const size_t ti = static_cast<size_t>(((e1 >> 4) & ((1u << 20) - 1)) - 1);
        const std::string tok = ti < toks.size() ? toks[ti] : std::string();
        if (code == 1)
            fail(CD_EINPUT, "malformed integer '" + tok + "' in " + where);
        if (code == 2)
            fail(CD_EINPUT, where + ": neighbor id " + tok + " out of range");
        if (code == 3)
            fail(CD_EINPUT, "malformed weight '" + tok + "' in " + where);
        if (code == 6)
            fail(CD_EINPUT, "weight '" + tok + "' in " + where + " is not a positive finite fp32 value");
        fail(CD_EINPUT, where + ": nonpositive edge weight");
    }
    if (nc - 1 < nn)
        fail(CD_EINPUT, name + ": expected " + std::to_string(n) + " adjacency lines, got " + std::to_string(nc - 1));
    if (nc > nn + 1) {  // only the first line after the adjacency lines is checked
        const int64_t lt = read1(ctx, line_of.p + nn + 1);
        int64_t tk[2];
        CD_CUDA(cudaMemcpyAsync(tk, T.line_tok.p + lt, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CD_CUDA(cudaStreamSynchronize(ctx->stream));
        if (tk[1] != tk[0])
            fail(CD_EINPUT, name + ": trailing content after " + std::to_string(n) + " adjacency lines");
    }
    T.buf.release();
    // symmetry (reference: sorted rows, lower_bound(u, 0.0) = v's smallest weight towards u)
    DBuf<uint64_t> lkey(ctx, std::max<int64_t>(D, 1));
    DBuf<uint32_t> lidx(ctx, std::max<int64_t>(D, 1));
    DBuf<int32_t> uu(ctx, std::max<int64_t>(D, 1)), uv(ctx, std::max<int64_t>(D, 1));
    DBuf<float> uw(ctx, weighted ? std::max<int64_t>(D, 1) : 0);
    DBuf<int64_t> counters(ctx, 2);
    counters.zero();
    if (D > INT32_MAX)
        fail(CD_EINVAL, name + ": more than 2^31 adjacency entries");
    if (D)
        CD_LAUNCH(ctx, "ingest", k_metis_split, grid_for(D, 256, ctx->num_sms * 16), 256, 0, D,
                  static_cast<const int32_t *>(eu.p), static_cast<const int32_t *>(ev.p), lkey.p, lidx.p, uu.p, uv.p,
                  static_cast<const double *>(ew.p), weighted ? uw.p : nullptr, counters.p);
    int64_t hc[2];
    CD_CUDA(cudaMemcpyAsync(hc, counters.p, sizeof(hc), cudaMemcpyDeviceToHost, ctx->stream));
    CD_CUDA(cudaStreamSynchronize(ctx->stream));
    const int64_t L = hc[0], U = hc[1];
    int bits = 1;
    while ((int64_t(1) << bits) < nn && bits < 31)
        ++bits;
    radix_sort_pairs(ctx, lkey.p, lidx.p, L, 32 + bits);  // (v << 32 | u): v needs `bits` bits
    DBuf<double> minw(ctx, std::max<int64_t>(L, 1));
    if (L)
        CD_LAUNCH(ctx, "ingest", k_run_min, grid_for(L, 256, ctx->num_sms * 16), 256, 0, L,
                  static_cast<const uint64_t *>(lkey.p), static_cast<const uint32_t *>(lidx.p),
                  static_cast<const double *>(ew.p), minw.p);
    ErrSlot serr(ctx);
    if (D)
        CD_LAUNCH(ctx, "ingest", k_metis_symmetry, grid_for(D, 256, ctx->num_sms * 16), 256, 0, D,
                  static_cast<const int32_t *>(eu.p), static_cast<const int32_t *>(ev.p),
                  static_cast<const double *>(ew.p), L, static_cast<const uint64_t *>(lkey.p),
                  static_cast<const double *>(minw.p), serr.v.p);
    const unsigned long long e2 = serr.get(ctx);
    if (e2 != NO_ERR)
        fail(CD_EINPUT, name + ": asymmetric adjacency between nodes " + std::to_string((e2 >> 32) + 1) + " and " +
                            std::to_string((e2 & 0xffffffffULL) + 1));
    lkey.release();
    lidx.release();
    minw.release();
    eu.release();
    ev.release();
    ew.release();
    cd_graph *g = graph_from_pairs(ctx, nn, U, uu.p, uv.p, weighted ? uw.p : nullptr, DUP_ERROR);
    if (static_cast<uint64_t>(g->m) != m) {
        const int64_t gm = g->m;
        delete g;
        fail(CD_EINPUT, name + ": header promises " + std::to_string(m) + " edges, file contains " +
                            std::to_string(gm));
    }
    return g;
}

// ---- edge list (H/io.hpp:190-237) -------------------------------------------------
namespace {

__global__ void k_el_lines(int64_t nlines, const int64_t *line_tok, int64_t *cnt, unsigned long long *err) {
    for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nlines;
         l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = line_tok[l + 1] - line_tok[l];
        cnt[l] = c ? 1 : 0;
        if (c && c != 2 && c != 3)
            atomicMin(err, (static_cast<unsigned long long>(l) << 24) | 5ULL);
    }
}

__global__ void k_el_parse(int64_t nlines, const int64_t *line_tok, const int64_t *eidx, const char *t,
                           const int64_t *tok_start, const int32_t *tok_len, uint64_t *ids, double *w,
                           int *any_w, unsigned long long *err) {
    for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nlines;
         l += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = line_tok[l], c = line_tok[l + 1] - k;
        if (c != 2 && c != 3)
            continue;
        const int64_t e = eidx[l];
        uint64_t u = 0, v = 0;
        double wt = 1.0;
        int code = 0, tok = 0;
        if (!parse_u64(t + tok_start[k], tok_len[k], u)) {
            code = 1;
            tok = 1;
        } else if (!parse_u64(t + tok_start[k + 1], tok_len[k + 1], v)) {
            code = 1;
            tok = 2;
        } else if (c == 3 && !parse_f64(t + tok_start[k + 2], tok_len[k + 2], wt)) {
            code = 3;
            tok = 3;
        } else if (!(wt > 0.0)) {
            code = 4;
        } else if (!fp32_weight_ok(wt)) {
            code = 6;  // parsed and positive, but the stored fp32 weight would be 0 or inf
            tok = 3;
        }
        if (code)
            atomicMin(err, (static_cast<unsigned long long>(l) << 24) | (static_cast<unsigned long long>(tok) << 4) |
                               code);
        if (c == 3)
            *any_w = 1;
        ids[2 * e] = u;
        ids[2 * e + 1] = v;
        w[e] = wt;
    }
}

struct UniqFlag {
    const uint64_t *k;
    __device__ int64_t operator()(int64_t i) const { return (i == 0 || k[i - 1] != k[i]) ? 1 : 0; }
};

__global__ void k_uniq_scatter(int64_t N, const uint64_t *k, const int64_t *rank, uint64_t *out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < N;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (i == 0 || k[i - 1] != k[i])
            out[rank[i]] = k[i];
}

__global__ void k_remap(int64_t m, const uint64_t *ids, int64_t n, const uint64_t *uniq, int32_t *eu, int32_t *ev,
                        const double *w, float *wf) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        for (int s = 0; s < 2; ++s) {
            const uint64_t x = ids[2 * e + s];
            int64_t lo = 0, hi = n;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (uniq[mid] < x)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            (s ? ev : eu)[e] = static_cast<int32_t>(lo);
        }
        if (wf)
            wf[e] = static_cast<float>(w[e]);
    }
}

}  // namespace

cd_graph *read_edge_list_dev(cd_ctx *ctx, const char *text, int64_t len, bool merge, const std::string &name) {
    Text T;
    load_text(ctx, T, text, len);
    index_lines(ctx, T);
    if (T.nlines)
        CD_LAUNCH(ctx, "ingest", k_blank_comments, grid_for(T.nlines, 256, ctx->num_sms * 16), 256, 0, T.nlines,
                  static_cast<const int64_t *>(T.line_start.p), len, T.buf.p);
    index_tokens(ctx, T);
    const int64_t nl = T.nlines;
    ErrSlot err(ctx);
    DBuf<int64_t> has(ctx, std::max<int64_t>(nl, 1)), eidx(ctx, nl + 1);
    if (nl)
        CD_LAUNCH(ctx, "ingest", k_el_lines, grid_for(nl, 256, ctx->num_sms * 16), 256, 0, nl,
                  static_cast<const int64_t *>(T.line_tok.p), has.p, err.v.p);
    exclusive_scan<int64_t>(ctx, nl, CountGen64{has.p}, eidx.p, eidx.p + nl);
    const int64_t m = read1(ctx, eidx.p + nl);
    DBuf<uint64_t> ids(ctx, std::max<int64_t>(2 * m, 1));
    DBuf<double> w(ctx, std::max<int64_t>(m, 1));
    DBuf<int> any_w(ctx, 1);
    any_w.zero();
    if (nl)
        CD_LAUNCH(ctx, "ingest", k_el_parse, grid_for(nl, 256, ctx->num_sms * 16), 256, 0, nl,
                  static_cast<const int64_t *>(T.line_tok.p), static_cast<const int64_t *>(eidx.p),
                  static_cast<const char *>(T.buf.p), static_cast<const int64_t *>(T.tok_start.p),
                  static_cast<const int32_t *>(T.tok_len.p), ids.p, w.p, any_w.p, err.v.p);
    const unsigned long long e1 = err.get(ctx);
    if (e1 != NO_ERR) {
        const int64_t l = static_cast<int64_t>(e1 >> 24);
        const int code = static_cast<int>(e1 & 15);
        const std::string where = name + ":" + std::to_string(l + 1);
        if (code == 5)
            fail(CD_EINPUT, where + ": expected 'u v [w]'");
        const auto toks = split_ws_host(line_text(ctx, T, l, INT64_MAX));
        const size_t ti = static_cast<size_t>(((e1 >> 4) & ((1u << 20) - 1)) - 1);
        const std::string tok = ti < toks.size() ? toks[ti] : std::string();
        if (code == 1)
            fail(CD_EINPUT, "malformed integer '" + tok + "' in " + where);
        if (code == 3)
            fail(CD_EINPUT, "malformed weight '" + tok + "' in " + where);
        if (code == 6)
            fail(CD_EINPUT, "weight '" + tok + "' in " + where + " is not a positive finite fp32 value");
        fail(CD_EINPUT, where + ": nonpositive edge weight");
    }
    const bool weighted = read1(ctx, any_w.p) != 0;
    T = Text();
    // densify ids in ascending numeric order (H/io.hpp:220-229)
    DBuf<uint64_t> sorted(ctx, std::max<int64_t>(2 * m, 1));
    if (m)
        CD_CUDA(cudaMemcpyAsync(sorted.p, ids.p, 2 * m * sizeof(uint64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    radix_sort_pairs(ctx, sorted.p, nullptr, 2 * m, 64);
    DBuf<int64_t> urank(ctx, 2 * m + 1);
    exclusive_scan<int64_t>(ctx, 2 * m, UniqFlag{sorted.p}, urank.p, urank.p + 2 * m);
    const int64_t n = read1(ctx, urank.p + 2 * m);
    if (n >= INT32_MAX)
        fail(CD_EINVAL, name + ": device node ids are int32 (n < 2^31 - 1)");
    DBuf<uint64_t> uniq(ctx, std::max<int64_t>(n, 1));
    if (m)
        CD_LAUNCH(ctx, "ingest", k_uniq_scatter, grid_for(2 * m, 256, ctx->num_sms * 16), 256, 0, 2 * m,
                  static_cast<const uint64_t *>(sorted.p), static_cast<const int64_t *>(urank.p), uniq.p);
    sorted.release();
    urank.release();
    DBuf<int32_t> eu(ctx, std::max<int64_t>(m, 1)), ev(ctx, std::max<int64_t>(m, 1));
    DBuf<float> wf(ctx, weighted ? std::max<int64_t>(m, 1) : 0);
    if (m)
        CD_LAUNCH(ctx, "ingest", k_remap, grid_for(m, 256, ctx->num_sms * 16), 256, 0, m,
                  static_cast<const uint64_t *>(ids.p), n, static_cast<const uint64_t *>(uniq.p), eu.p, ev.p,
                  static_cast<const double *>(w.p), weighted ? wf.p : nullptr);
    ids.release();
    w.release();
    cd_graph *g = graph_from_pairs(ctx, n, m, eu.p, ev.p, weighted ? wf.p : nullptr, merge ? DUP_SUM : DUP_ERROR);
    g->orig_ids = std::move(uniq);
    return g;
}

}  // namespace cdk
