// zs_train.cuh -- dictionary training on the device.
//
// The reference trainer (dictionary.py:169-320) counts every alphabet-only
// substring of length l_min..l_max (one np.unique per length), then picks t
// patterns by repeated argmax of occurrences * (length - greedy cover by the
// already-selected patterns), recomputing every cover after each pick.
//
// Census, B200 shape: one sort instead of one per length.  Every start
// position whose alphabet run reaches l_min is sorted by its first l_max
// bytes (LSD over big-endian 8-byte words, CUB radix passes); in that order
// the windows sharing any L-byte prefix are contiguous, so for each length
// L the distinct patterns are the runs between neighbours whose common
// prefix is shorter than L (lcp, capped by both alphabet runs, decides that
// exactly).  One flags -> scan -> scatter sweep per L then yields the rows in
// the reference's RankTable order (length-major, bytewise ascending), with
// occurrences = run length.
//
//   tr_runs     alphabet run length from each position (capped at l_max)
//   tr_key      big-endian 8-byte key word w of each candidate start
//   tr_lcp      common prefix of sorted neighbours, capped by both runs
//   tr_flags    per L: group boundary (lcp < L) and candidate (run >= L)
//   tr_scatter  per L: group starts and candidate slots
//   tr_rows     per L: rows (first position, length, occurrences)
//
// Selection (dictionary.py:241-307): the working set (top-cap rows by
// initial rank, stable) is a CUB descending sort; each pick is two launches
// with no host round trip -- tr_rank (thread per live candidate: greedy
// cover against the selected-pattern trie, rank, permanent drop at rank <= 0,
// block argmax under the _pick tie rule) and tr_pick (one CTA: final argmax,
// the exclusion check, trie insert).
#pragma once
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <stdint.h>

namespace zs {

// smiles.py ALPHABET: letters, digits and []()=#-+@/\%.:*$~
__host__ __device__ constexpr bool tr_is_alpha(unsigned b) {
    return (b >= 'A' && b <= 'Z') || (b >= 'a' && b <= 'z') || (b >= '0' && b <= '9') || b == '[' || b == ']' ||
           b == '(' || b == ')' || b == '=' || b == '#' || b == '-' || b == '+' || b == '@' || b == '/' ||
           b == '\\' || b == '%' || b == '.' || b == ':' || b == '*' || b == '$' || b == '~';
}

constexpr int TR_NT = 256;
constexpr int TR_SPAN = 32;  // positions per thread in tr_runs

__global__ void __launch_bounds__(TR_NT) tr_runs(const uint8_t *__restrict__ buf, long long n, int lmax,
                                                 uint8_t *__restrict__ run) {
    const long long nc = (n + TR_SPAN - 1) / TR_SPAN;
    for (long long c = blockIdx.x * (long long)TR_NT + threadIdx.x; c < nc; c += (long long)gridDim.x * TR_NT) {
        const long long a = c * TR_SPAN, b = min(n, a + TR_SPAN);
        int r = 0;
        for (long long j = b; j < n && r < lmax && tr_is_alpha(buf[j]); ++j) ++r;  // seed: the run at b
        for (long long i = b - 1; i >= a; --i) {
            r = tr_is_alpha(buf[i]) ? min(lmax, r + 1) : 0;
            run[i] = (uint8_t)r;
        }
    }
}

struct TrAtLeast {
    const uint8_t *run;
    int lmin;
    __device__ __forceinline__ bool operator()(const uint32_t &i) const { return run[i] >= lmin; }
};

// key word w of position p: bytes p + 8w .. p + 8w + nb (big-endian, zero past the buffer)
__global__ void tr_key(const uint8_t *__restrict__ buf, long long n, const uint32_t *__restrict__ pos, long long m,
                       int w, int nb, unsigned long long *__restrict__ key) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const long long p = (long long)pos[i] + 8ll * w;
        unsigned long long k = 0;
        for (int j = 0; j < 8; ++j) k = (k << 8) | (j < nb && p + j < n ? buf[p + j] : 0u);
        key[i] = k;
    }
}

// lcp[i] = common prefix of sorted neighbours i - 1, i, capped by both runs
// (exact for every group test the census makes, see the header); run_s[i] =
// run of the i-th sorted position
__global__ void tr_lcp(const uint8_t *__restrict__ buf, const uint32_t *__restrict__ pos, long long m,
                       const uint8_t *__restrict__ run, uint8_t *__restrict__ lcp, uint8_t *__restrict__ run_s) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const uint32_t p = pos[i];
        const int r = run[p];
        run_s[i] = (uint8_t)r;
        int l = 0;
        if (i > 0) {
            const uint32_t q = pos[i - 1];
            const int c = min(r, (int)run[q]);
            while (l < c && buf[p + l] == buf[q + l]) ++l;
        }
        lcp[i] = (uint8_t)l;
    }
}

// v = (boundary << 32) | candidate
__global__ void tr_flags(const uint8_t *__restrict__ lcp, const uint8_t *__restrict__ run_s, long long m, int L,
                         unsigned long long *__restrict__ v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long f = (i == 0 || lcp[i] < L) ? 1ull : 0ull;
        v[i] = (f << 32) | (f && run_s[i] >= L ? 1ull : 0ull);
    }
}

__global__ void tr_scatter(const unsigned long long *__restrict__ v, const unsigned long long *__restrict__ ex,
                           long long m, uint32_t *__restrict__ bstart, uint32_t *__restrict__ cand) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long x = v[i], e = ex[i];
        if (x >> 32) bstart[e >> 32] = (uint32_t)i;
        if (x & 1ull) cand[e & 0xffffffffull] = (uint32_t)i;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // sentinel: one past the last group
        const unsigned long long x = v[m - 1], e = ex[m - 1];
        bstart[(e >> 32) + (x >> 32)] = (uint32_t)m;
    }
}

__global__ void tr_rows(const uint32_t *__restrict__ cand, long long c, const uint32_t *__restrict__ pos,
                        const unsigned long long *__restrict__ ex, const uint32_t *__restrict__ bstart, int L,
                        uint32_t *__restrict__ row_pos, uint32_t *__restrict__ row_occ, uint8_t *__restrict__ row_len) {
    for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < c; o += (long long)gridDim.x * blockDim.x) {
        const uint32_t i = cand[o];
        const uint32_t g = (uint32_t)(ex[i] >> 32);
        row_pos[o] = pos[i];
        row_occ[o] = bstart[g + 1] - i;
        row_len[o] = (uint8_t)L;
    }
}

__global__ void tr_init_rank(const uint32_t *__restrict__ occ, const uint8_t *__restrict__ len, long long m,
                             unsigned long long *__restrict__ rank, uint32_t *__restrict__ idx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        rank[i] = (unsigned long long)occ[i] * len[i];
        idx[i] = (uint32_t)i;
    }
}

// ---- selection ----
constexpr int TR_TRIE_W = 256;  // trie row width (any byte of an uploaded table)

// greedy longest-match cover (numba_impl.py:149-169) of p[0..n) against a
// byte trie: child(node, b) < 0 = no edge, term(node) != 0 = terminal
template <typename Child, typename Term>
__device__ __forceinline__ int tr_cover(const uint8_t *p, int n, Child child, Term term) {
    int pos = 0, cov = 0;
    while (pos < n) {
        int node = 0, best = 0;
        for (int j = pos; j < n; ++j) {
            node = child(node, p[j]);
            if (node < 0) break;
            if (term(node)) best = j + 1 - pos;
        }
        if (best > 0) {
            cov += best;
            pos += best;
        } else {
            pos += 1;
        }
    }
    return cov;
}

struct TrBest {
    unsigned long long k1;  // rank << 7 | length (higher wins); 0 = none
    uint32_t row, slot;     // equal k1: bytewise smaller pattern wins (dictionary.py:229-238)
};

struct TrRows {
    const uint8_t *buf;
    const uint32_t *pos;
    const uint8_t *len;
    // a beats b under _pick: higher rank, then longer, then bytewise smaller
    __device__ __forceinline__ bool better(const TrBest &a, const TrBest &b) const {
        if (a.k1 != b.k1) return a.k1 > b.k1;
        if (a.k1 == 0 || a.row == b.row) return false;
        const uint8_t *p = buf + pos[a.row], *q = buf + pos[b.row];
        const int L = len[a.row];
        for (int j = 0; j < L; ++j)
            if (p[j] != q[j]) return p[j] < q[j];
        return a.row < b.row;
    }
};

__device__ __forceinline__ TrBest tr_shfl(const TrBest &b, int o) {
    TrBest y;
    y.k1 = __shfl_xor_sync(0xffffffffu, b.k1, o);
    y.row = __shfl_xor_sync(0xffffffffu, b.row, o);
    y.slot = __shfl_xor_sync(0xffffffffu, b.slot, o);
    return y;
}

__device__ __forceinline__ TrBest tr_block_best(TrBest b, const TrRows &R) {
    __shared__ TrBest s[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const TrBest y = tr_shfl(b, o);
        if (R.better(y, b)) b = y;
    }
    if (lane == 0) s[wid] = b;
    __syncthreads();
    if (wid == 0) {
        b = lane < (int)(blockDim.x >> 5) ? s[lane] : TrBest{0ull, 0u, 0u};
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const TrBest y = tr_shfl(b, o);
            if (R.better(y, b)) b = y;
        }
    }
    return b;  // valid in thread 0
}

struct TrCtl {
    int done, fail, nsel, nodes;
};

__global__ void __launch_bounds__(TR_NT) tr_rank(TrRows R, const uint32_t *__restrict__ row_occ,
                                                 const uint32_t *__restrict__ ws, long long nws, uint8_t *__restrict__ dead,
                                                 const int16_t *__restrict__ child, const uint8_t *__restrict__ term,
                                                 const TrCtl *__restrict__ ctl, TrBest *__restrict__ blk) {
    if (ctl->done) return;
    TrBest b{0ull, 0u, 0u};
    auto ch = [&](int node, unsigned c) -> int { return child[node * TR_TRIE_W + c]; };
    auto tm = [&](int node) -> bool { return term[node] != 0; };
    for (long long k = blockIdx.x * (long long)TR_NT + threadIdx.x; k < nws; k += (long long)gridDim.x * TR_NT) {
        if (dead[k]) continue;
        const uint32_t r = ws[k];
        const int L = R.len[r];
        const int cov = tr_cover(R.buf + R.pos[r], L, ch, tm);
        const unsigned long long rank = (unsigned long long)row_occ[r] * (unsigned)(L - cov);
        if (rank == 0) {  // dictionary.py:279-284: dropped from the working set for good
            dead[k] = 1;
            continue;
        }
        const TrBest c{(rank << 7) | (unsigned)L, r, (uint32_t)k};
        if (R.better(c, b)) b = c;
    }
    b = tr_block_best(b, R);
    if (threadIdx.x == 0) blk[blockIdx.x] = b;
}

__global__ void __launch_bounds__(1024) tr_pick(TrRows R, uint8_t *__restrict__ dead, int16_t *__restrict__ child,
                                                uint8_t *__restrict__ term, TrCtl *__restrict__ ctl,
                                                const TrBest *__restrict__ blk, int nblk, long long excluded_max,
                                                uint32_t *__restrict__ sel) {
    if (ctl->done) return;
    TrBest b{0ull, 0u, 0u};
    for (int i = threadIdx.x; i < nblk; i += blockDim.x)
        if (R.better(blk[i], b)) b = blk[i];
    b = tr_block_best(b, R);
    if (threadIdx.x != 0) return;
    if (b.k1 == 0) {  // working set exhausted (dictionary.py:285-286)
        ctl->done = 1;
        return;
    }
    if ((long long)(b.k1 >> 7) <= excluded_max) {  // dictionary.py:288-289: retry with a bigger cap
        ctl->fail = 1;
        ctl->done = 1;
        return;
    }
    sel[ctl->nsel++] = b.row;
    dead[b.slot] = 1;
    // trie insert (trie.py:22-50)
    const uint8_t *p = R.buf + R.pos[b.row];
    int node = 0;
    for (int j = 0; j < R.len[b.row]; ++j) {
        int nx = child[node * TR_TRIE_W + p[j]];
        if (nx < 0) {
            nx = ctl->nodes++;
            child[node * TR_TRIE_W + p[j]] = (int16_t)nx;
        }
        node = nx;
    }
    term[node] = 1;
}

// overlap_batch parity shim (numba_impl.py:142-169), reference trie layout
__global__ void tr_overlap_batch(const int32_t *__restrict__ children, const int16_t *__restrict__ term_len,
                                 const uint8_t *__restrict__ pats, int width, const long long *__restrict__ lens,
                                 long long n, long long *__restrict__ out) {
    auto ch = [&](int node, unsigned c) -> int { return children[(size_t)node * 256 + c]; };
    auto tm = [&](int node) -> bool { return term_len[node] >= 0; };
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
        out[r] = tr_cover(pats + r * (long long)width, (int)lens[r], ch, tm);
}

}  // namespace zs
