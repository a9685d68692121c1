// zs_ll.cuh -- long lines: lines longer than compress_cx's staged window,
// coded with every phase of the per-line codec spread over 256-byte blocks of
// the line across the whole GPU (a 14 MB line is ~55k blocks, one thread
// each), instead of one thread walking the line in HBM.
//
// compress_cx (mode 0) records the long lines it meets; the host sorts them
// and runs, on the lines' bytes in the input:
//
//   ll_setup        first byte of each line (the tiles' last-newline table)
//   ll_tok_map      per block: the tokenizer's transfer function over its 8
//                   states (smiles.py:83-137 as tk_entry), nibble-packed and
//                   applied byte by byte with two PRMTs; '\r' -> fallback
//   ll_scan<Map>    exclusive composition scan: each block's entry state
//   ll_tok_count    ring tokens per block, XOR parity of their ids
//   ll_scan<Add>,
//   ll_scan<Xor>    event offsets; id parity before each block
//   ll_tok_events   events (line position, id, '%nn' flag, open/close by parity)
//   ll_pair         each closing event's opening partner (nearest earlier
//                   event with the same id: ids alternate open / close,
//                   smiles.py:140-160)
//   ll_colour       closing events in order, cut into segments (a thread
//                   each): colour = smallest k whose last close precedes the
//                   ring's opening (smiles.py:163-183); a segment enters with
//                   a guessed lc[] and is re-run until its neighbour's exit
//                   agrees with it where its own rings can see
//   ll_rlen / ll_scan<Add> / ll_rewrite
//                   renumbered bytes per block, offsets, the renumbered lines
//   ll_parse (+ ll_parse_fix until stable)
//                   min-cost parse right to left (numba_impl.py:32-56) with the
//                   product automaton; a block is entered in a guessed state
//                   (warm-up from the line-end state over the next block's
//                   first bytes), checked against its right neighbour's exit
//                   and re-parsed only up to where the two walks meet
//   ll_emit_count (+ ll_emit_fix until stable)
//                   forward decision walk (numba_impl.py:57-69): output bytes
//                   per block from a guessed path entry, repaired the same way
//   ll_scan<Add> / ll_emit_write
//                   output offsets, the coded bytes, per-line totals
//
// then compress_cx again (mode 1: a long line's output size comes from its
// entry, its bytes are left out) and ll_place copies each coded line to the
// offset compress_cx reserved.  A line with a '\r', a tokenize error, an
// unpaired ring or more than 100 overlapping rings keeps the general routine
// (compress_line_global), which carries the error contract.
#pragma once
#include "zs_device.cuh"

namespace zs {

constexpr int LL_B = 256;        // bytes of the original line per block
constexpr int LL_NT = 128;       // threads per CTA of the per-block kernels (small CTAs: a MB line fills the SMs)
constexpr int LL_SNT = 1024;     // the scan CTA
constexpr int LL_CAP = 32768;    // long lines per launch
constexpr long long LL_MAXBYTES = 1ll << 28;  // long-line bytes per launch (beyond: general routine; keeps offsets 32-bit)
constexpr int LL_WARM = 8;       // parse warm-up bytes of a guessed entry

struct LLWork {
    const uint8_t *in;
    long long n;            // input bytes (reads stay inside [in, in + n))
    LLine *ln;
    int n_ll;
    int nb;                 // blocks
    int preprocess;
    // per block (scanned arrays have nb + 1 entries: [nb] = total)
    unsigned *map;          // tokenizer transfer maps -> exclusive composition
    int *cnt;               // ring tokens -> first event index
    uint4 *par;             // id parity -> parity before the block
    int *rlen;              // renumbered bytes -> offset in R
    unsigned *pin, *pout;   // parse: assumed entry state, exit state
    int *g, *x;             // emit: path entry, exit (R positions)
    int *ocnt;              // output bytes per block
    int *ooff;              // (scan) their offsets in O
    int *oesc;              // escapes
    // per event
    int *epos;              // position in the line
    uint16_t *eflag;        // id | 0x80 '%nn' | 0x100 opens a ring | 0x200 the line's first event
    int *epart;             // closing event: the opening event's index; -1 opens
    uint8_t *ecol;          // colour
    uint8_t *R;             // the (renumbered) lines
    uint8_t *D;             // decisions, aligned with R
    uint8_t *O;             // coded lines
    int *changed;           // fix-loop flag
    // product automaton (build_pa): rows of nc u32, state = row byte offset
    const uint32_t *pa;
    const uint8_t *cmap;
    int pa_words;
    const uint8_t *explen;
    const struct LLTok *tok;  // tokenizer tables (ll_tok_build)
    long long ecap, rcap, ocap;  // events, R / D bytes, O bytes allocated (ZS_CHECKS asserts)
};

// Sequential byte reads (either direction) through aligned 16-byte loads: a
// thread walks its block's bytes in registers instead of one L2 request per
// byte.  A 16-byte chunk that is not inside [lo, hi) is read bytewise.
struct LLRd {
    uintptr_t lo, hi, ck = ~(uintptr_t)0;
    uint4 v;
    __device__ LLRd(const void *lo_, const void *hi_)
        : lo(reinterpret_cast<uintptr_t>(lo_)), hi(reinterpret_cast<uintptr_t>(hi_)) {}
    __device__ __forceinline__ unsigned operator()(const uint8_t *p) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p), c = a & ~(uintptr_t)15;
        if (c != ck) {
            if (c < lo || c + 16 > hi) return *p;
            v = __ldg(reinterpret_cast<const uint4 *>(c));
            ck = c;
        }
        const unsigned k = (unsigned)(a & 15);
        const unsigned w = k < 8 ? (k < 4 ? v.x : v.y) : (k < 12 ? v.z : v.w);
        return (w >> (8 * (k & 3))) & 0xffu;
    }
};
// workspace buffers carry slack past their last byte: no upper bound needed
__device__ __forceinline__ LLRd ll_rd(const uint8_t *base) {
    return LLRd(base, reinterpret_cast<const void *>(~(uintptr_t)0 >> 1));
}

// Sequential byte writes (either direction): a whole 4-byte word leaves with
// one store; the partial words at the ends of a thread's range go byte by
// byte (the neighbouring threads own their other bytes).
struct LLWr {
    uintptr_t wd = 0;
    unsigned val = 0, mask = 0;
    __device__ __forceinline__ void flush() {
        if (mask == 0xfu) {
            *reinterpret_cast<unsigned *>(wd) = val;
        } else if (mask) {
            for (int k = 0; k < 4; ++k)
                if ((mask >> k) & 1u) reinterpret_cast<uint8_t *>(wd)[k] = (uint8_t)(val >> (8 * k));
        }
        mask = val = 0;
    }
    __device__ __forceinline__ void put(uint8_t *p, unsigned b) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p), w = a & ~(uintptr_t)3;
        if (w != wd) {
            flush();
            wd = w;
        }
        const unsigned k = (unsigned)(a & 3);
        val |= (b & 0xffu) << (8 * k);
        mask |= 1u << k;
    }
};

__device__ __forceinline__ int ll_line_of(const LLine *ln, int n_ll, int b) {
    int lo = 0, hi = n_ll - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ln[mid].blk0 <= b) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// block b of its line: line index, offset, length (0: a fallback line's block)
struct LLBlk {
    int line, off, len;
    bool head, last;
};
__device__ __forceinline__ LLBlk ll_blk(const LLWork &W, int b) {
    LLBlk k;
    k.line = ll_line_of(W.ln, W.n_ll, b);
    const LLine &L = W.ln[k.line];
    const int r = b - L.blk0;
    const long long len = L.ge - L.gs;
    k.off = r * LL_B;
    k.len = (int)min((long long)LL_B, len - k.off);
    k.head = r == 0;
    k.last = r == L.nblk - 1;
    return k;
}

// ---------------------------------------------------------------- setup
// First byte of each long line: one past the last '\n' of the nearest tile
// before the line's tile that has one (tl[], written by compress_cx); a warp
// per line checks 32 tiles per step.
__global__ void ll_setup(LLine *ln, int n_ll, const long long *tl, long long n_tiles, long long tile) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_ll) return;
    const long long ge = ln[w].ge;
    long long t = min(ge / tile, n_tiles - 1) - 1;  // tiles strictly before the line's tile
    long long gs = 0;
    for (; t >= 0; t -= 32) {
        const long long q = t - lane;
        const long long v = q >= 0 ? tl[q] : -1;
        const unsigned m = __ballot_sync(0xffffffffu, v >= 0);
        if (m) {
            const int j = __ffs(m) - 1;  // lowest lane = latest tile
            gs = __shfl_sync(0xffffffffu, v, j) + 1;
            break;
        }
    }
    if (lane == 0) {
        ln[w].gs = gs;
        ln[w].dst = -1;
        ln[w].cost = ln[w].esc = 0;
        ln[w].status = LL_OK;
    }
}

// ---------------------------------------------------------------- scans
struct LLAdd {
    using T = int;
    __device__ static T id() { return 0; }
    __device__ static T op(T a, T b) { return a + b; }
};
struct LLXor {
    using T = uint4;
    __device__ static T id() { return make_uint4(0, 0, 0, 0); }
    __device__ static T op(T a, T b) { return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w); }
};
// transfer maps: nibble s = image of state s; op(a, b) = b after a
__device__ __forceinline__ unsigned ll_nib_pack(unsigned x) {
    return (x & 7u) | ((x >> 4) & 0x70u) | ((x >> 8) & 0x700u) | ((x >> 12) & 0x7000u);
}
__device__ __forceinline__ unsigned ll_apply(unsigned lo, unsigned hi, unsigned v) {
    // v's nibbles index the byte table (lo: images of states 0-3, hi: 4-7)
    return ll_nib_pack(__byte_perm(lo, hi, v & 0xffffu)) | (ll_nib_pack(__byte_perm(lo, hi, v >> 16)) << 16);
}
__device__ __forceinline__ void ll_unpack(unsigned m, unsigned &lo, unsigned &hi) {
    lo = (m & 7u) | ((m & 0x70u) << 4) | ((m & 0x700u) << 8) | ((m & 0x7000u) << 12);
    m >>= 16;
    hi = (m & 7u) | ((m & 0x70u) << 4) | ((m & 0x700u) << 8) | ((m & 0x7000u) << 12);
}
struct LLMap {
    using T = unsigned;
    __device__ static T id() { return 0x76543210u; }
    __device__ static T op(T a, T b) {
        unsigned lo, hi;
        ll_unpack(b, lo, hi);
        return ll_apply(lo, hi, a);
    }
};

// Exclusive scan of in[0, n) into out[0, n] (out[n] = the total; in == out
// scans in place); one CTA.
template <class Op>
__global__ void __launch_bounds__(LL_SNT) ll_scan(const typename Op::T *in, typename Op::T *out, int n) {
    using T = typename Op::T;
    __shared__ T s[LL_SNT];
    const int tid = threadIdx.x;
    const int per = (n + LL_SNT - 1) / LL_SNT;
    const int lo = min(n, tid * per), hi = min(n, lo + per);
    T acc = Op::id();
    for (int k = lo; k < hi; ++k) acc = Op::op(acc, in[k]);
    s[tid] = acc;
    __syncthreads();
    for (int d = 1; d < LL_SNT; d <<= 1) {  // inclusive Hillis-Steele over the chunk totals
        T v = s[tid];
        if (tid >= d) v = Op::op(s[tid - d], v);
        __syncthreads();
        s[tid] = v;
        __syncthreads();
    }
    T run = tid ? s[tid - 1] : Op::id();
    for (int k = lo; k < hi; ++k) {
        const T v = in[k];
        out[k] = run;
        run = Op::op(run, v);
    }
    if (tid == LL_SNT - 1) out[n] = s[LL_SNT - 1];
}

// ---------------------------------------------------------------- tokenizer
// tokenizer tables in smem: per byte the next states of states 0-3 / 4-7
// (bytes) and the full entries (bits 0-2 next state, TK_RING)
struct LLTok {
    unsigned lo[256], hi[256];
    uint8_t e[8 * 256];
};
// host: the tables from tk_entry
inline void ll_tok_build(LLTok &T) {
    for (int b = 0; b < 256; ++b) {
        unsigned lo = 0, hi = 0;
        for (int q = 0; q < 4; ++q) {
            lo |= (unsigned)(tk_entry(q, b) & 7u) << (8 * q);
            hi |= (unsigned)(tk_entry(q + 4, b) & 7u) << (8 * q);
        }
        T.lo[b] = lo;
        T.hi[b] = hi;
    }
    for (int k = 0; k < 8 * 256; ++k) T.e[k] = tk_entry(k >> 8, k & 255);
}
__device__ __forceinline__ void ll_tok_init(LLTok &T, const LLTok *g) {
    const uint4 *src = reinterpret_cast<const uint4 *>(g);
    uint4 *dst = reinterpret_cast<uint4 *>(&T);
    for (int k = threadIdx.x; k < (int)(sizeof(LLTok) / 16); k += blockDim.x) dst[k] = src[k];
    __syncthreads();
}

// per block: transfer map (the line's first block: the constant map of its
// image of TK_OUT0, so an unsegmented scan gives every block its entry
// state); any '\r' sends the line to the general routine
template <bool PRE>
__global__ void __launch_bounds__(LL_NT) ll_tok_map(LLWork W) {
    __shared__ __align__(16) LLTok T;
    if (PRE) ll_tok_init(T, W.tok);
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    LLine &L = W.ln[k.line];
    const uint8_t *s = W.in + L.gs + k.off;
    LLRd rd(W.in, W.in + W.n);
    unsigned v = 0x76543210u, cr = 0;
    for (int i = 0; i < k.len; ++i) {
        const unsigned c = rd(s + i);
        cr |= c == '\r';
        if (PRE) v = ll_apply(T.lo[c], T.hi[c], v);
    }
    if (cr) L.status = LL_FALLBACK;
    if (PRE) {
        if (k.head) v = 0x11111111u * (v & 7u);  // constant: the image of TK_OUT0
        W.map[b] = v;
    }
}

__device__ __forceinline__ unsigned ll_entry_state(const LLWork &W, const LLBlk &k, int b) {
    return k.head ? (unsigned)TK_OUT0 : (W.map[b] & 7u);  // scanned prefix: a constant map
}

// ring id of the token at s[i] ('%nn' or a digit); bounded by the line
__device__ __forceinline__ unsigned ll_ring_id(LLRd &rd, const uint8_t *s, int i, long long rem, bool &pct) {
    const unsigned c = rd(s + i);
    pct = c == '%';
    if (!pct) return c - '0';
    const unsigned d1 = rem > 1 ? rd(s + i + 1) : '0', d2 = rem > 2 ? rd(s + i + 2) : '0';
    return (d1 - '0') * 10u + (d2 - '0');
}

// ring tokens per block and the XOR parity of their ids; a tokenize error
// (a '%' without two digits is sticky, an open bracket at the end) -> fallback
__global__ void __launch_bounds__(LL_NT) ll_tok_count(LLWork W) {
    __shared__ __align__(16) LLTok T;
    ll_tok_init(T, W.tok);
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    LLine &L = W.ln[k.line];
    const long long len = L.ge - L.gs;
    const uint8_t *s = W.in + L.gs + k.off;
    unsigned st = ll_entry_state(W, k, b);
    int cnt = 0;
    uint4 par = make_uint4(0, 0, 0, 0);
    LLRd rd(W.in, W.in + W.n);
    for (int i = 0; i < k.len; ++i) {
        const unsigned e = T.e[(st << 8) | rd(s + i)];
        st = e & 7u;
        if (e & TK_RING) {
            bool pct;
            unsigned id = ll_ring_id(rd, s, i, len - k.off - i, pct);
            if (id >= 100) id = 0;  // (a malformed '%' token: the line falls back)
            const unsigned bit = 1u << (id & 31);
            if (id < 32) par.x ^= bit;
            else if (id < 64) par.y ^= bit;
            else if (id < 96) par.z ^= bit;
            else par.w ^= bit;
            ++cnt;
        }
    }
    if (k.last && st != TK_OUT0 && st != TK_OUT1) L.status = LL_FALLBACK;
    W.cnt[b] = cnt;
    W.par[b] = par;
}

__device__ __forceinline__ unsigned ll_par_bit(const uint4 &p, unsigned id) {
    const unsigned w = id < 32 ? p.x : id < 64 ? p.y : id < 96 ? p.z : p.w;
    return (w >> (id & 31)) & 1u;
}

// events of the block: line position, flags (id, '%nn', opens); an odd id
// count over the line (an unpaired ring) -> fallback
__global__ void __launch_bounds__(LL_NT) ll_tok_events(LLWork W) {
    __shared__ __align__(16) LLTok T;
    ll_tok_init(T, W.tok);
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    LLine &L = W.ln[k.line];
    const long long len = L.ge - L.gs;
    const uint8_t *s = W.in + L.gs + k.off;
    uint4 par = LLXor::op(W.par[b], W.par[L.blk0]);  // parity of the line before the block
    int ev = W.cnt[b];
    const int line_ev0 = W.cnt[L.blk0];
    if (k.head) {
        L.ev0 = ev;
        L.nev = W.cnt[L.blk0 + L.nblk] - ev;
    }
    unsigned st = ll_entry_state(W, k, b);
    LLRd rd(W.in, W.in + W.n);
    for (int i = 0; i < k.len; ++i) {
        const unsigned e = T.e[(st << 8) | rd(s + i)];
        st = e & 7u;
        if (e & TK_RING) {
            bool pct;
            unsigned id = ll_ring_id(rd, s, i, len - k.off - i, pct);
            if (id >= 100) id = 0;  // (a malformed '%' token: the line falls back)
            const unsigned open = ll_par_bit(par, id) ^ 1u;
            if (id < 32) par.x ^= 1u << id;
            else if (id < 64) par.y ^= 1u << (id - 32);
            else if (id < 96) par.z ^= 1u << (id - 64);
            else par.w ^= 1u << (id - 96);
            ZS_ASSERT(ev < W.ecap);
            W.epos[ev] = k.off + i;
            W.eflag[ev] = (uint16_t)(id | (pct ? 0x80u : 0u) | (open << 8) | (ev == line_ev0 ? 0x200u : 0u));
            ++ev;
        }
    }
    if (k.last && (par.x | par.y | par.z | par.w)) L.status = LL_FALLBACK;
}

// closing event -> its opening event (the nearest earlier event of the id)
// (launched for an upper bound of the events; the count is W.cnt[nb])
__global__ void __launch_bounds__(LL_NT) ll_pair(LLWork W, int n_bound) {
    const int e = blockIdx.x * LL_NT + threadIdx.x;
    if (e >= n_bound || e >= W.cnt[W.nb]) return;
    const unsigned f = W.eflag[e];
    if (f & 0x100u) {
        W.epart[e] = -1;
        return;
    }
    // an event closes when an odd number of same-id events precede it in its
    // line, so the search ends inside the line
    int j = e - 1;
    const unsigned id = f & 0x7fu;
    while (j >= 0 && (W.eflag[j] & 0x7fu) != id) --j;
    W.epart[e] = j;
}

// Colouring (smiles.py:163-183): rings in closing order, each the smallest
// colour k with lc[k] (the event index of k's latest close) < its opening
// event.  The events are cut into segments of LL_SEG, one thread each; a
// segment enters with a guessed lc[] (no closes: exact at a line start) and
// later passes check it against the left neighbour's exit:
//  * the segment's colours read the incoming lc[] only through its crossing
//    rings (closing in it, opened before it): entries older than the earliest
//    such opening u act as "free", so the incoming state normalised at u
//    decides whether the segment runs again;
//  * its exit is its own last closes for the colours it touched after its
//    last line start, and the incoming entries for the others (no line start
//    in it), so a neighbour's changed entries pass through without a re-run;
//    exits are normalised at U (the earliest crossing-ring opening of all
//    later segments, ll_umin), below which no later segment looks, so old
//    entries stop travelling.
// A pass in which no exit changed ends the iteration.  Colour 100
// (RingIdOverflow) marks the ring 0xff; its line falls back (ll_rlen).
constexpr int LL_SEG = 128;
constexpr int LL_NCOL = 100;
// ints per segment.  exits: lc[100], n (entries from n on are -1);
// assumed: lc[100] (normalised at u), u, head, touched[4], U, n
constexpr int LL_CS = 112;
enum : int { LLC_N = 100, LLC_U = 100, LLC_HEAD = 101, LLC_T = 102, LLC_UU = 106, LLC_AN = 107 };

// (lm[k] is read only for k < nc, every such entry written first; nvcc cannot
// see that through the lambdas)
#pragma nv_diag_suppress 549
__global__ void __launch_bounds__(LL_NT) ll_colour(LLWork W, int n_bound, int pass, int *exits, int *assumed) {
    const int sg = blockIdx.x * LL_NT + threadIdx.x;
    const int a = sg * LL_SEG;
    const int n_ev = min(n_bound, W.cnt[W.nb]);
    if (a >= n_ev) return;
    const int b = min(n_ev, a + LL_SEG);
    int *ex = exits + (size_t)sg * LL_CS, *as = assumed + (size_t)sg * LL_CS;
    // lc: colours 0-7 in registers, the rest in local memory; entries from
    // nc on are -1
    int lr[8], lm[LL_NCOL - 8];
#pragma unroll
    for (int j = 0; j < 8; ++j) lr[j] = -1;
    int nc = 0;
    auto get = [&](int k) {
        if (k >= 8) return lm[k - 8];
        int v = -1;
#pragma unroll
        for (int j = 0; j < 8; ++j) v = k == j ? lr[j] : v;
        return v;
    };
    auto set = [&](int k, int v) {
#pragma unroll
        for (int j = 0; j < 8; ++j) lr[j] = k == j ? v : lr[j];
        if (k >= 8) lm[k - 8] = v;
    };
    const int U = pass > 0 ? as[LLC_UU] : -1;  // (pass 0: U is not known yet)
    if (pass > 0) {
        const int u = as[LLC_U], an = as[LLC_AN];
        const int *prev = exits + (size_t)(sg - 1) * LL_CS;
        const int pn = u < a || !as[LLC_HEAD] ? *(volatile const int *)&prev[LLC_N] : 0;
        auto pv = [&](int k) { return k < pn ? *(volatile const int *)&prev[k] : -1; };
        bool same = true;
        if (u < a)
            for (int k = 0; k < max(pn, an); ++k) {
                const int v = pv(k);
                same &= (v > u ? v : -1) == (k < an ? as[k] : -1);
            }
        if (same) {
            // colours unchanged: the exit is the own closes (touched colours,
            // or every colour after a line start) and the incoming entries
            const bool head = as[LLC_HEAD] != 0;
            const int en = ex[LLC_N], n = head ? en : max(en, pn);
            bool diff = false;
            for (int k = 0; k < n; ++k) {
                const bool own = head || ((as[LLC_T + (k >> 5)] >> (k & 31)) & 1);
                const int v0 = own ? (k < en ? ex[k] : -1) : pv(k);
                const int v = v0 > U ? v0 : -1;
                diff |= (k < en ? ex[k] : -1) != v;
                ex[k] = v;
            }
            if (n != en) ex[LLC_N] = n;
            if (diff) *W.changed = 1;
            return;
        }
        for (int k = 0; k < pn; ++k) {
            const int v = pv(k);
            set(k, v);
            as[k] = v > u ? v : -1;
        }
        nc = pn;
        as[LLC_AN] = pn;
    }
    // the walk, 16 events per step from vector loads; pass 0 also finds u:
    // the earliest opening before the segment among the rings closing in it
    // up to its first line start (a: none)
    unsigned t0 = 0, t1 = 0, t2 = 0, t3 = 0, head = 0;  // colours touched since the last line start
    int u = a;
    for (int base = a; base < b; base += 16) {
        uint16_t fl[16];
        int pt[16];
        if (base + 16 <= b) {
            const uint4 f0 = *reinterpret_cast<const uint4 *>(W.eflag + base);
            const uint4 f1 = *reinterpret_cast<const uint4 *>(W.eflag + base + 8);
            const unsigned fw[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
            for (int j = 0; j < 16; ++j) fl[j] = (uint16_t)(fw[j >> 1] >> (16 * (j & 1)));
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int4 v = *reinterpret_cast<const int4 *>(W.epart + base + 4 * q);
                pt[4 * q] = v.x;
                pt[4 * q + 1] = v.y;
                pt[4 * q + 2] = v.z;
                pt[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                fl[j] = base + j < b ? W.eflag[base + j] : 0;
                pt[j] = base + j < b ? W.epart[base + j] : -1;
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int e = base + j;
            if (e >= b) break;
            if (fl[j] & 0x200u) {
#pragma unroll
                for (int q = 0; q < 8; ++q) lr[q] = -1;
                nc = 0;
                t0 = t1 = t2 = t3 = 0;
                head = 1;
            }
            const int o = pt[j];
            if (o < 0) continue;  // opens a ring
            ZS_ASSERT(o < e);
            if (!head) u = min(u, o);
            int k = 8;
#pragma unroll
            for (int q = 7; q >= 0; --q) k = lr[q] < o ? q : k;  // (lr[q] = -1 beyond nc: free)
            if (k == 8) {
                while (k < nc && lm[k - 8] > o) ++k;
                if (k == nc && nc < LL_NCOL) lm[k - 8] = -1;
            }
            nc = max(nc, min(k + 1, LL_NCOL));
            if (k < LL_NCOL) {
                set(k, e);
                const unsigned bit = 1u << (k & 31);
                if (k < 32) t0 |= bit;
                else if (k < 64) t1 |= bit;
                else if (k < 96) t2 |= bit;
                else t3 |= bit;
            }
            W.ecol[e] = W.ecol[o] = (uint8_t)(k < LL_NCOL ? k : 0xff);
        }
    }
    if (pass == 0) {
        as[LLC_U] = u;
        as[LLC_AN] = 0;
    }
    as[LLC_HEAD] = (int)head;
    as[LLC_T] = (int)t0;
    as[LLC_T + 1] = (int)t1;
    as[LLC_T + 2] = (int)t2;
    as[LLC_T + 3] = (int)t3;
    const int en = pass > 0 ? ex[LLC_N] : 0;
    bool diff = false;
    for (int k = 0; k < max(nc, en); ++k) {
        const int g = k < nc ? get(k) : -1;
        const int v = g > U ? g : -1;
        diff |= (k < en ? ex[k] : -1) != v;
        ex[k] = v;
    }
    ex[LLC_N] = max(nc, en);
    if (pass > 0 && diff) *W.changed = 1;
}

#pragma nv_diag_default 549

// U of every segment: the minimum u of the segments after it (unsegmented:
// a later line's u lies past every event of this line, which then all
// normalise away, as they may); one CTA
__global__ void __launch_bounds__(LL_SNT) ll_umin(LLWork W, int n_bound, int *assumed) {
    __shared__ int s[LL_SNT];
    const int n_ev = min(n_bound, W.cnt[W.nb]);
    const int nseg = (n_ev + LL_SEG - 1) / LL_SEG;
    const int tid = threadIdx.x;
    const int per = (nseg + LL_SNT - 1) / LL_SNT;
    const int lo = min(nseg, tid * per), hi = min(nseg, lo + per);
    int m = 0x7fffffff;
    for (int k = lo; k < hi; ++k) m = min(m, assumed[(size_t)k * LL_CS + LLC_U]);
    s[tid] = m;
    __syncthreads();
    for (int d = 1; d < LL_SNT; d <<= 1) {  // inclusive suffix min over the chunk minima
        int v = s[tid];
        if (tid + d < LL_SNT) v = min(v, s[tid + d]);
        __syncthreads();
        s[tid] = v;
        __syncthreads();
    }
    int run = tid + 1 < LL_SNT ? s[tid + 1] : 0x7fffffff;  // min over the chunks after this one
    for (int k = hi - 1; k >= lo; --k) {
        assumed[(size_t)k * LL_CS + LLC_UU] = run;
        run = min(run, assumed[(size_t)k * LL_CS + LLC_U]);
    }
}

// ---------------------------------------------------------------- rewrite
// Units of a block: the bytes from its first byte not covered by a '%nn'
// token of the previous block, and the ring tokens that start in it (a token
// may run into the next block).
__device__ __forceinline__ int ll_skip(const LLWork &W, const LLBlk &k, int ev_first) {
    if (!W.preprocess || k.head || ev_first <= W.ln[k.line].ev0) return 0;
    const int j = ev_first - 1;
    const int end = W.epos[j] + ((W.eflag[j] & 0x80u) ? 3 : 1);
    return max(0, end - k.off);
}

__device__ __forceinline__ int ll_newlen(unsigned col) { return col < 10 ? 1 : 3; }

__global__ void __launch_bounds__(LL_NT) ll_rlen(LLWork W) {
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    LLine &L = W.ln[k.line];
    if (L.status != LL_OK) {
        W.rlen[b] = 0;
        return;
    }
    int r = k.len;
    if (W.preprocess) {
        const int ea = W.cnt[b], eb = W.cnt[b + 1];
        r -= ll_skip(W, k, ea);
        for (int e = ea; e < eb; ++e) {
            if (W.ecol[e] == 0xff) L.status = LL_FALLBACK;  // > 100 overlapping rings
            const int ol = (W.eflag[e] & 0x80u) ? 3 : 1;
            r += ll_newlen(W.ecol[e]) - min(ol, k.off + k.len - W.epos[e]);
        }
    }
    W.rlen[b] = r;
}

__global__ void __launch_bounds__(LL_NT) ll_rewrite(LLWork W) {
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    const LLine &L = W.ln[k.line];
    if (L.status != LL_OK) return;
    const uint8_t *s = W.in + L.gs;
    uint8_t *o = W.R + W.rlen[b];
    LLRd rd(W.in, W.in + W.n);
    LLWr wr;
    int e = W.preprocess ? W.cnt[b] : 0;
    const int eb = W.preprocess ? W.cnt[b + 1] : 0;
    int p = k.off + (W.preprocess ? ll_skip(W, k, e) : 0);
    const int end = k.off + k.len;
    int next = e < eb ? W.epos[e] : 0x7fffffff;
    while (p < end) {
        if (p == next) {
            const unsigned col = W.ecol[e];
            if (col < 10) {
                wr.put(o++, '0' + col);
            } else {
                wr.put(o++, '%');
                wr.put(o++, '0' + col / 10);
                wr.put(o++, '0' + col % 10);
            }
            p += (W.eflag[e] & 0x80u) ? 3 : 1;
            ++e;
            next = e < eb ? W.epos[e] : 0x7fffffff;
        } else {
            wr.put(o++, rd(s + p));
            ++p;
        }
    }
    ZS_ASSERT(o - W.R <= W.rcap && (int)(o - W.R) == W.rlen[b + 1]);
    wr.flush();
}

// ---------------------------------------------------------------- parse
// block b's range in R: [rlen[b], rlen[b + 1]) (scanned offsets); the line's
// [rlen[blk0], rlen[blk0 + nblk])
__device__ __forceinline__ unsigned ll_dec(unsigned e, unsigned c) {
    return ((e >> 16) & 0xffu) | (c & (unsigned)((int)e >> 31));
}

__global__ void __launch_bounds__(LL_NT) ll_parse(LLWork W) {
    extern __shared__ uint32_t s_pa[];
    __shared__ uint8_t s_cm[256];
    for (int k = threadIdx.x; k < W.pa_words; k += LL_NT) s_pa[k] = W.pa[k];
    for (int k = threadIdx.x; k < 256; k += LL_NT) s_cm[k] = W.cmap[k];
    __syncthreads();
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    const LLine &L = W.ln[k.line];
    if (L.status != LL_OK) return;
    const int lo = W.rlen[b], hi = W.rlen[b + 1], lend = W.rlen[L.blk0 + L.nblk];
    unsigned st = 0;
    LLRd rd = ll_rd(W.R);
    if (!k.last)  // guessed entry: warm-up from the line-end state
        for (int p = min(hi + LL_WARM, lend) - 1; p >= hi; --p) st = s_pa[(st + s_cm[rd(W.R + p)]) >> 2] & 0xffffu;
    W.pin[b] = st;
    LLWr wr;
    for (int p = hi - 1; p >= lo; --p) {
        const unsigned c = rd(W.R + p);
        const unsigned e = s_pa[(st + s_cm[c]) >> 2];
        st = e & 0xffffu;
        wr.put(W.D + p, ll_dec(e, c));
    }
    wr.flush();
    W.pout[b] = st;
}

// a block whose entry differs from its right neighbour's exit is parsed again
// from the true state next to the assumed one until the two states meet
__global__ void __launch_bounds__(LL_NT) ll_parse_fix(LLWork W) {
    extern __shared__ uint32_t s_pa[];
    __shared__ uint8_t s_cm[256];
    for (int k = threadIdx.x; k < W.pa_words; k += LL_NT) s_pa[k] = W.pa[k];
    for (int k = threadIdx.x; k < 256; k += LL_NT) s_cm[k] = W.cmap[k];
    __syncthreads();
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    const LLine &L = W.ln[k.line];
    if (L.status != LL_OK || k.last) return;
    const unsigned truth = *(volatile unsigned *)&W.pout[b + 1];
    unsigned so = W.pin[b];
    if (truth == so) return;
    const int lo = W.rlen[b], hi = W.rlen[b + 1];
    unsigned sn = truth;
    bool met = false;
    for (int p = hi - 1; p >= lo; --p) {
        const unsigned c = W.R[p];
        const unsigned eo = s_pa[(so + s_cm[c]) >> 2], en = s_pa[(sn + s_cm[c]) >> 2];
        so = eo & 0xffffu;
        sn = en & 0xffffu;
        W.D[p] = (uint8_t)ll_dec(en, c);
        if (sn == so) {
            met = true;
            break;
        }
    }
    W.pin[b] = truth;
    if (!met && W.pout[b] != sn) {
        W.pout[b] = sn;
        *W.changed = 1;
    }
}

// ---------------------------------------------------------------- emit
// one decision at p: output bytes (2 for an escape), positions covered
__device__ __forceinline__ void ll_step(const LLWork &W, LLRd &rd, const uint8_t *xl, int &p, int &out,
                                        int &esc) {
    const unsigned c = rd(W.D + p);
    if (c == 0x20u) {
        out += 2;
        ++esc;
        ++p;
    } else {
        ++out;
        p += xl[c];
    }
}

__global__ void __launch_bounds__(LL_NT) ll_emit_count(LLWork W) {
    __shared__ uint8_t xl[256];
    for (int k = threadIdx.x; k < 256; k += LL_NT) xl[k] = W.explen[k];
    __syncthreads();
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    const LLine &L = W.ln[k.line];
    if (L.status != LL_OK) {
        W.ocnt[b] = W.oesc[b] = 0;
        return;
    }
    const int lo = W.rlen[b], hi = W.rlen[b + 1];
    int p = lo, out = 0, esc = 0;  // guess: a decision starts at the block's first byte
    LLRd rd = ll_rd(W.D);
    while (p < hi) ll_step(W, rd, xl, p, out, esc);
    W.g[b] = lo;
    W.x[b] = p;
    W.ocnt[b] = out + (k.last ? 1 : 0);  // the line's '\n'
    W.oesc[b] = esc;
}

// a block entered off its left neighbour's exit walks the true path next to
// the guessed one (advancing the one behind) until they meet
__global__ void __launch_bounds__(LL_NT) ll_emit_fix(LLWork W) {
    __shared__ uint8_t xl[256];
    for (int k = threadIdx.x; k < 256; k += LL_NT) xl[k] = W.explen[k];
    __syncthreads();
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    const LLine &L = W.ln[k.line];
    if (L.status != LL_OK || k.head) return;
    const int truth = *(volatile int *)&W.x[b - 1];
    int gp = W.g[b];
    if (truth == gp) return;
    const int hi = W.rlen[b + 1];
    int a = truth, da = 0, ea = 0, db = 0, eb = 0;
    LLRd rd = ll_rd(W.D);
    while (a != gp && min(a, gp) < hi) {
        if (a < gp) ll_step(W, rd, xl, a, da, ea);
        else ll_step(W, rd, xl, gp, db, eb);
    }
    W.ocnt[b] += da - db;
    W.oesc[b] += ea - eb;
    W.g[b] = truth;
    if (a != gp) {  // never met: the exit moves
        W.x[b] = a;
        *W.changed = 1;
    }
}

__global__ void __launch_bounds__(LL_NT) ll_emit_write(LLWork W) {
    __shared__ uint8_t xl[256];
    for (int k = threadIdx.x; k < 256; k += LL_NT) xl[k] = W.explen[k];
    __syncthreads();
    const int b = blockIdx.x * LL_NT + threadIdx.x;
    if (b >= W.nb) return;
    const LLBlk k = ll_blk(W, b);
    LLine &L = W.ln[k.line];
    if (L.status != LL_OK) return;
    const int hi = W.rlen[b + 1];
    uint8_t *o = W.O + W.ooff[b];
    int p = W.g[b];
    LLRd rdd = ll_rd(W.D), rdr = ll_rd(W.R);
    LLWr wr;
    while (p < hi) {
        const unsigned c = rdd(W.D + p);
        if (c == 0x20u) {
            wr.put(o++, 0x20);
            wr.put(o++, rdr(W.R + p));
            ++p;
        } else {
            wr.put(o++, c);
            p += xl[c];
        }
    }
    if (k.last) wr.put(o, '\n');
    ZS_ASSERT(o + (k.last ? 1 : 0) - W.O == W.ooff[b + 1] && o - W.O < W.ocap);
    wr.flush();
    if (W.oesc[b]) atomicAdd((unsigned long long *)&L.esc, (unsigned long long)W.oesc[b]);
    if (k.head) {
        L.obase = W.ooff[b];
        L.cost = (long long)W.ooff[L.blk0 + L.nblk] - W.ooff[b] - 1;
    }
}

// ---------------------------------------------------------------- place
// after compress_cx (mode 1): each coded line to the offset it reserved
__global__ void __launch_bounds__(LL_NT) ll_place(const LLine *ln, int n_ll, const uint8_t *O, uint8_t *out,
                                                  long long out_cap) {
    const LLine &L = ln[blockIdx.x];
    if (L.status != LL_OK || L.nblk == 0 || L.dst < 0) return;
    const long long len = L.cost + 1;
    if (L.dst + len > out_cap) return;
    const uint8_t *src = O + L.obase;
    uint8_t *dst = out + L.dst;
    const long long step = (long long)gridDim.y * LL_NT;
    for (long long i = (long long)blockIdx.y * LL_NT + threadIdx.x; i < len; i += step) dst[i] = src[i];
}

}  // namespace zs
