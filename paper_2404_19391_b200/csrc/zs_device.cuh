// zs_device.cuh -- sm_100a device code for the ZSMILES per-line codec.
//
// Layout of the hot path:
//   * The input buffer stays resident in HBM.  It is cut into fixed TILE-byte
//     tiles; a line belongs to the tile in which it STARTS.  One persistent
//     CTA per SM takes tiles in order from an atomic ticket.
//   * Per tile the CTA stages [tile_start-16, tile_end+EXTRA) in shared memory
//     (16-byte vector loads), finds its line starts (newline scan + block
//     scan -> a compact queue), and processes lines thread-per-line from the
//     queue: CR policy, ring renumbering (in place in smem), then the
//     min-cost parse.
//   * The parse runs right-to-left over a reversed-pattern Aho-Corasick DFA
//     held in shared memory: one 16-bit table lookup per byte yields the next
//     state and the set of dictionary match lengths starting at that byte;
//     the DP keeps the next W costs in registers as packed keys
//     (cost<<3)-position, so "cheapest, then longest" (numba_impl.py:50) is a
//     single signed min.  Decisions (the chosen code byte, 0x20 = escape) are
//     written per byte into smem.
//   * Tile output size -> decoupled look-back over tiles (single pass, no
//     line-offset array in HBM) -> the forward emit writes compressed records
//     into a smem staging buffer -> coalesced 16-byte stores to HBM.
//   * Decompression uses the same tile/look-back skeleton with a table-driven
//     size/validate pass and expansion pass.
//
// Lines that do not fit the smem window (longer than EXTRA past the tile, or
// lines that grow under renumbering) take a "global" path in the same kernel:
// scratch from a bump arena in HBM and the reference-shaped trie walk.
#pragma once
#include <stdint.h>

namespace zs {

// ----------------------------------------------------------------------------
// constants
// ----------------------------------------------------------------------------
constexpr int NT = 512;                 // threads per CTA
constexpr int NWARP = NT / 32;
// Per-thread chunk of the tile for the newline scans and the emit walks.
// 68 bytes = 17 words: an odd word stride puts the 32 lanes of a warp on 32
// different shared-memory banks (a 64-byte stride would be a 16-way conflict).
constexpr int CHUNK = 68;
constexpr int TILE = CHUNK * NT;        // 34816 bytes of line-start ownership per tile
constexpr int EXTRA = 4096;             // window overhang past the tile end
constexpr int HEAD = 16;                // bytes staged before the tile start
constexpr int WIN = HEAD + TILE + EXTRA;  // staged window (multiple of 16)
constexpr int QCAP = 2048;              // line queue capacity per round
constexpr int OUTCAP = 20480;           // compress staging (~0.4 B/B typical; else direct)
constexpr int DOUTCAP = 3 * TILE;       // decompress staging
constexpr int NCOL = 97;                // DFA columns: bytes 0x20..0x7f, other
constexpr int FAST_W = 8;               // max pattern length on the fast path
constexpr int FAST_STATES = 256;        // max DFA states on the fast path
constexpr int T2_MASKS = 16;            // cost-window transducer: mask indices per window
constexpr int T2_WINDOWS = 1024;        // ... and windows (4 B entries: <= 64 KB)

// decision-byte sentinels (never valid codes: codes are 0x21-0x7e, 0x80-0xff)
constexpr uint8_t D_ESC = 0x20;   // escape: emit 0x20 + literal
constexpr uint8_t D_END = 0x0A;   // end of (preprocessed) line
constexpr uint8_t D_DROP = 0x0D;  // line dropped (lenient CR) or strict error
constexpr uint8_t D_GLOBAL = 0x0B;  // line processed in the HBM arena

// tile flags for the look-back
enum : unsigned { F_AGG = 1u, F_INC = 2u };

enum ErrKind {
    E_NONE = 0, E_CR = 1, E_BRACKET = 2, E_PERCENT = 3, E_UNPAIRED = 4, E_OVERFLOW = 5,
    E_UNKNOWN = 6, E_TRUNC = 7
};

struct Tables {
    // fast path: reversed-pattern AC DFA, [n_states][NCOL] u16 = next | mask<<8
    const uint16_t *dfa;
    const uint8_t *codes;   // [n_states][FAST_W] code of the match of length L+1
    int n_states;
    int fast;               // 1 if the DFA path serves this dictionary
    // cost-window transducer (fast path, when built): dfa2 entries carry a
    // mask index instead of the mask; t2[window][mask index] = next window |
    // L << 12 | (cost delta + 16) << 16
    const uint16_t *dfa2;
    const uint32_t *t2;
    int n_windows;
    // generic path (reference layout): dense trie in HBM
    const int32_t *children;  // [n_nodes][256]
    const int16_t *term_code;
    int n_nodes;
    int max_len;
    // decode
    const uint8_t *exp_len;   // [256], 0 = invalid code
    const uint16_t *exp_off;  // [257]
    const uint8_t *exp_flat;
    int n_flat;
    int max_exp;  // longest expansion (<= 8 enables the unrolled copy)
};

struct Ctl {                    // zeroed before every launch
    unsigned long long ticket;
    unsigned long long total_out;
    unsigned long long lines;
    unsigned long long escapes;
    unsigned long long skipped;
    unsigned long long flagged;
    unsigned long long err_key;    // (line_idx << 24) | tile ; ~0 = none
    unsigned long long arena_used;
    unsigned long long overflow;   // output or arena capacity exceeded
    unsigned long long in_lines;   // lines seen (records in)
    unsigned long long ll_n;       // long lines recorded (compress_cx, Job.ll_mode 0)
    unsigned long long phase[8];   // per-phase SM cycles (thread 0), when Job.timing
};

// A line longer than compress_cx's staged window ("long line", zs_ll.cuh):
// recorded by compress_cx (ge), sorted by ge on the host, then coded by the
// block-parallel long-line kernels before compress_cx runs again and takes
// its output size from here.
struct LLine {
    long long ge;     // global offset of the terminating '\n' (n: the virtual one at EOF)
    long long gs;     // global offset of the first byte
    long long obase;  // output bytes (payload + '\n') in the long-line workspace
    long long dst;    // output offset compress_cx reserved for the line; -1 = none
    long long cost;   // payload bytes (without the '\n')
    long long esc;    // escapes
    int blk0, nblk;   // 256-byte blocks [blk0, blk0 + nblk) of the line
    int ev0, nev;     // ring-token events [ev0, ev0 + nev) (preprocess)
    int status;       // LL_OK, or LL_FALLBACK: the general routine codes the line
    int pad;
};
enum : int { LL_OK = 0, LL_FALLBACK = 1 };

struct TileState {
    unsigned int flag;
    unsigned int pad;
    unsigned long long agg_out, agg_lines, inc_out, inc_lines;
};

struct TileErr {
    int kind;
    int code;
    long long offset;
    unsigned long long ids[2];
};

struct Job {
    const uint8_t *in;
    long long n;
    uint8_t *out;
    long long out_cap;
    int preprocess, lenient;
    long long n_tiles;
    Ctl *ctl;
    TileState *ts;
    TileErr *terr;
    uint8_t *arena;
    long long arena_cap;
    int timing;  // accumulate per-phase clock64 deltas into Ctl.phase
    // long lines (compress_cx): mode 0 records them in `ll` (up to ll_cap) and
    // flags Ctl.overflow bit 16; mode 1 takes the coded ones from `ll` (ll_n
    // entries sorted by ge); mode 2 codes every line in the kernel
    LLine *ll = nullptr;
    long long *tl = nullptr;  // per tile: global offset of its last '\n', -1 = none
    int ll_mode = 2, ll_n = 0, ll_cap = 0;
};

// Phase clocks and the other measurement hooks are compiled in only with
// -DZS_PHASES=1 (tools/phase_cx.py builds such a library); the production
// kernels carry no timing branches.
#ifndef ZS_PHASES
#define ZS_PHASES 0
#endif
constexpr bool kPhases = ZS_PHASES != 0;

// thread-0 phase clock: PHASE(k) adds the cycles since the last mark to phase k
struct PhaseClock {
    long long t;
    __device__ __forceinline__ void start() {
        if (kPhases) t = clock64();
    }
    __device__ __forceinline__ void mark(const Job &job, int k) {
        if (kPhases && job.timing != 2 && job.timing != 6 && job.timing && threadIdx.x == 0) {
            long long now = clock64();
            atomicAdd(&job.ctl->phase[k], (unsigned long long)(now - t));
            t = now;
        }
    }
};

// ----------------------------------------------------------------------------
// small helpers (host-callable too: tests/hostcheck runs the per-line
// routines on the CPU against the oracle)
// ----------------------------------------------------------------------------
#define ZS_HD __host__ __device__ __forceinline__

ZS_HD unsigned umin_(unsigned a, unsigned b) { return a < b ? a : b; }
ZS_HD int imin_(int a, int b) { return a < b ? a : b; }
ZS_HD int ffs64_(unsigned long long x) {
#ifdef __CUDA_ARCH__
    return __ffsll((long long)x);
#else
    return __builtin_ffsll((long long)x);
#endif
}

ZS_HD int dcol(unsigned b) { return (int)umin_(b - 0x20u, 96u); }

// Byte loads from a buffer that lives in shared memory on the device: the
// 32-bit shared address is formed once (a generic pointer re-derives the
// window base every access).  Host builds read through the pointer.
struct SmemBytes {
#ifdef __CUDA_ARCH__
    unsigned base;
    __device__ __forceinline__ explicit SmemBytes(const uint8_t *p)
        : base((unsigned)__cvta_generic_to_shared(p)) {}
    __device__ __forceinline__ unsigned ld(int i) const {
        unsigned v;
        asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(base + i));
        return v;
    }
#else
    const uint8_t *p;
    explicit SmemBytes(const uint8_t *q) : p(q) {}
    unsigned ld(int i) const { return p[i]; }
#endif
};

// Explicit shared-memory accesses through 32-bit addresses formed once (a
// generic pointer makes the compiler re-derive the shared window base,
// S2R SR_CgaCtaId + LEA, at many accesses under register pressure).  All are
// volatile so they keep program order with each other and with barriers.
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned ldsb(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned ldsh(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned ldsw(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void stsb(unsigned a, unsigned v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// warp-uniform loop condition (device: all 32 lanes must take part)
#ifdef __CUDA_ARCH__
#define ZS_ANY(p) __any_sync(0xffffffffu, (p))
#else
#define ZS_ANY(p) (p)
#endif

ZS_HD bool is_digit(unsigned b) { return b - '0' < 10u; }

// byte classes for the tokenizer (smiles.py:23-35, 83-137)
enum : uint8_t {
    C_OTHER = 0, C_ATOM = 1, C_BOND = 2, C_DIGIT = 3, C_PCT = 4, C_LBR = 5, C_RBR = 6,
    C_BOPEN = 7, C_BCLOSE = 8, C_DOT = 9, C_CR = 10
};

ZS_HD uint8_t tok_class(unsigned b) {
    if ((b | 0x20u) - 'a' < 26u || b == '*') return C_ATOM;
    if (b - '0' < 10u) return C_DIGIT;
    switch (b) {
    case '-': case '=': case '#': case '$': case ':': case '/': case '\\': case '~': return C_BOND;
    case '%': return C_PCT;
    case '[': return C_LBR;
    case ']': return C_RBR;
    case '(': return C_BOPEN;
    case ')': return C_BCLOSE;
    case '.': return C_DOT;
    case '\r': return C_CR;
    default: return C_OTHER;
    }
}

// block-wide exclusive scan of one value per thread (NT threads)
template <typename T>
__device__ __forceinline__ T block_exscan(T v, T *warp_tmp, T &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tmp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        T w = lane < NWARP ? warp_tmp[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NWARP) warp_tmp[lane] = w;  // inclusive per warp
    }
    __syncthreads();
    T base = wid ? warp_tmp[wid - 1] : T(0);
    total = warp_tmp[NWARP - 1];
    __syncthreads();
    return base + x - v;
}

// block-wide exclusive scan for a CTA of NTH threads (NTH / 32 <= 32)
template <typename T, int NTH>
__device__ __forceinline__ T block_exscan_n(T v, T *warp_tmp, T &total) {
    constexpr int NW = NTH / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tmp[wid] = x;
    __syncthreads();
    T base = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
        const T wv = warp_tmp[k];
        base += k < wid ? wv : T(0);
        tot += wv;
    }
    total = tot;
    __syncthreads();
    return base + x - v;
}

// ----------------------------------------------------------------------------
// decoupled look-back over tiles, one warp (ordered tickets guarantee
// progress).  Lanes inspect 32 predecessors per round trip: the nearest one
// with an inclusive prefix ends the walk, the aggregates before it are summed
// with a warp reduction.  Must be called by all 32 lanes of one warp.
// ----------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Publish this tile's aggregate (tile 0 publishes its inclusive prefix).
__device__ __forceinline__ void lookback_publish(TileState *ts, long long t,
                                                 unsigned long long agg_out,
                                                 unsigned long long agg_lines) {
    volatile TileState *vts = ts;
    if (t == 0) {
        vts[0].inc_out = agg_out;
        vts[0].inc_lines = agg_lines;
        __threadfence();
        atomicExch(&ts[0].flag, F_INC);
    } else {
        vts[t].agg_out = agg_out;
        vts[t].agg_lines = agg_lines;
        __threadfence();
        atomicExch(&ts[t].flag, F_AGG);
    }
}

// Resolve the exclusive prefix of tile t (all 32 lanes of one warp) and
// publish t's inclusive prefix.
__device__ __forceinline__ void lookback_resolve(TileState *ts, long long t,
                                                 unsigned long long agg_out,
                                                 unsigned long long agg_lines,
                                                 unsigned long long &pre_out,
                                                 unsigned long long &pre_lines) {
    volatile TileState *vts = ts;
    const int lane = threadIdx.x & 31;
    if (t == 0) {
        pre_out = 0;
        pre_lines = 0;
        return;
    }
    unsigned long long po = 0, pl = 0;
    long long j = t - 1;
    for (;;) {
        const long long idx = j - lane;
        unsigned f = idx >= 0 ? vts[idx].flag : F_INC;
        while (__any_sync(0xffffffffu, f == 0u))
            if (f == 0u) f = vts[idx].flag;
        __threadfence();
        const unsigned inc = __ballot_sync(0xffffffffu, f == F_INC);
        const int stop = inc ? __ffs(inc) - 1 : 32;  // lanes < stop: AGG; lane == stop: INC
        unsigned long long vo = 0, vl = 0;
        if (idx >= 0 && lane <= stop) {
            if (lane == stop) {
                vo = vts[idx].inc_out;
                vl = vts[idx].inc_lines;
            } else {
                vo = vts[idx].agg_out;
                vl = vts[idx].agg_lines;
            }
        }
        po += warp_sum(vo);
        pl += warp_sum(vl);
        if (inc) break;
        j -= 32;
    }
    if (lane == 0) {
        vts[t].inc_out = po + agg_out;
        vts[t].inc_lines = pl + agg_lines;
        __threadfence();
        atomicExch(&ts[t].flag, F_INC);
    }
    pre_out = po;
    pre_lines = pl;
}

__device__ __forceinline__ void lookback(TileState *ts, long long t, unsigned long long agg_out,
                                         unsigned long long agg_lines,
                                         unsigned long long &pre_out,
                                         unsigned long long &pre_lines) {
    if ((threadIdx.x & 31) == 0) lookback_publish(ts, t, agg_out, agg_lines);
    __syncwarp();
    lookback_resolve(ts, t, agg_out, agg_lines, pre_out, pre_lines);
}

// ----------------------------------------------------------------------------
// ring renumbering of one line (smiles.py:83-213), strict semantics.
//
// buf[0..n) is the line; marks[0..n] is per-byte scratch (0xff = not a ring
// token start, 0xfe = ring opened / colour pending, <100 = assigned colour).
// One forward pass tokenizes, pairs ids (occurrences alternate open/close)
// and colours each ring when it closes with the smallest id not used by a
// ring that closed inside it (closing-order greedy, smiles.py:162-180): a
// single backward scan from the closing token finds the opener (the most
// recent pending token with the same id) and collects those colours.
// Returns E_NONE and the new length in *new_len (the rewrite is in place
// when no ring token grows), E_CR if a '\r' is present anywhere, another
// E_* on a tokenize/pair/colour error (err_off / ids filled), or -1 when the
// line grows (caller re-runs it out of place with out != buf).
// ----------------------------------------------------------------------------
__host__ __device__ int preprocess_line(const uint8_t *buf, int n, uint8_t *marks, uint8_t *out,
                               int *new_len, int *err_off, unsigned long long ids[2],
                               bool cr_is_error = true) {
    uint64_t open0 = 0, open1 = 0;  // currently open ring ids
    bool ring_ok = false;
    int nrings = 0, grow = 0;
    int err = E_NONE, eoff = -1;
    int i = 0;
    while (i < n) {
        unsigned b = buf[i];
        uint8_t c = tok_class(b);
        if (c == C_CR && !cr_is_error) c = C_OTHER;
        marks[i] = 0xff;
        int rid = -1, tlen = 1;
        if (c == C_ATOM || c == C_BOND) {
            ring_ok = true;
        } else if (c == C_DIGIT) {
            if (ring_ok) rid = (int)(b - '0');
        } else if (c == C_PCT) {
            if (i + 2 >= n || !is_digit(buf[i + 1]) || !is_digit(buf[i + 2])) {
                err = E_PERCENT; eoff = i;
                break;
            }
            marks[i + 1] = 0xff;
            marks[i + 2] = 0xff;
            tlen = 3;
            if (ring_ok) rid = (int)(buf[i + 1] - '0') * 10 + (int)(buf[i + 2] - '0');
        } else if (c == C_LBR) {
            int j = i + 1;
            while (j < n && buf[j] != ']') {
                if (cr_is_error && buf[j] == '\r') { err = E_CR; break; }
                marks[j] = 0xff;
                ++j;
            }
            if (err) break;
            if (j >= n) { err = E_BRACKET; eoff = i; break; }
            marks[j] = 0xff;
            tlen = j + 1 - i;
            ring_ok = true;
        } else if (c == C_CR) {
            err = E_CR;
            break;
        } else {
            ring_ok = false;  // ( ) . and any other byte
        }
        if (rid >= 0) {
            // ring closure token
            uint64_t bit = 1ull << (rid & 63);
            bool is_open = rid < 64 ? (open0 & bit) : (open1 & bit);
            if (!is_open) {
                marks[i] = 0xfe;
                if (rid < 64) open0 |= bit; else open1 |= bit;
            } else {
                if (rid < 64) open0 &= ~bit; else open1 &= ~bit;
                uint64_t used0 = 0, used1 = 0;
                int o = i - 1;
                for (;; --o) {
                    uint8_t m = marks[o];
                    if (m == 0xfe) {
                        int r2 = buf[o] == '%' ? (buf[o + 1] - '0') * 10 + (buf[o + 2] - '0')
                                               : buf[o] - '0';
                        if (r2 == rid) break;
                    } else if (m < 100) {
                        if (m < 64) used0 |= 1ull << m; else used1 |= 1ull << (m - 64);
                    }
                }
                int col = used0 != ~0ull ? ffs64_(~used0) - 1
                                         : 64 + (used1 != ~0ull ? ffs64_(~used1) - 1 : 64);
                if (col > 99) { err = E_OVERFLOW; break; }
                marks[o] = (uint8_t)col;
                marks[i] = (uint8_t)col;
                // an endpoint grows only when a 1-byte id takes a colour >= 10
                // (the two endpoints may differ: '1' pairs with '%01')
                if (col >= 10) grow |= (buf[o] != '%') | (tlen == 1);
                nrings++;
            }
            ring_ok = true;
        }
        i += tlen;
    }
    if (err == E_NONE && (open0 | open1)) {
        err = E_UNPAIRED;
        ids[0] = open0;
        ids[1] = open1;
    }
    if (cr_is_error && err != E_NONE && err != E_CR) {
        // CR anywhere in the line takes precedence (pipeline.py:102-107)
        for (int k = 0; k < n; ++k)
            if (buf[k] == '\r') { err = E_CR; break; }
    }
    if (err != E_NONE) {
        *err_off = eoff;
        return err;
    }
    if (nrings == 0) {
        if (out != buf)
            for (int k = 0; k < n; ++k) out[k] = buf[k];
        *new_len = n;
        return E_NONE;
    }
    if (grow && out == buf) return -1;  // needs an out-of-place rewrite
    // rewrite: tokens keep order; every ring token takes its colour text
    int w = 0;
    for (int r = 0; r < n;) {
        uint8_t m = marks[r];
        if (m < 100) {
            int ol = buf[r] == '%' ? 3 : 1;
            if (m < 10) {
                out[w++] = (uint8_t)('0' + m);
            } else {
                out[w++] = '%';
                out[w++] = (uint8_t)('0' + m / 10);
                out[w++] = (uint8_t)('0' + m % 10);
            }
            r += ol;
        } else {
            out[w++] = buf[r++];
        }
    }
    *new_len = w;
    return E_NONE;
}

// ----------------------------------------------------------------------------
// ring renumbering, fast path (the common case), in three steps:
//
//  1. tokenize: one tight pass over the bytes (class LUT in smem).  Ring
//     tokens are threaded into a forward chain kept in `marks`: marks[pos]
//     = distance to the next chain node (0 = last; 255 = a hop node that is
//     not a token, inserted when the gap exceeds 254).
//  2. pair + colour: walk the chain (~6 nodes per line).  Open rings live in
//     4 register slots (id, position); the smallest free colour comes from
//     lc[k] = position where colour k last closed (k is taken by a ring
//     closed inside (o, c) iff lc[k] > o).  Single-digit tokens are
//     rewritten in place; a '%nn' token gets its digit in s[pos+1] and the
//     line is compacted in step 3.
//  3. compaction (only with '%nn' ring tokens): walk the chain again,
//     shifting the bytes between tokens left.
//
// Same semantics as preprocess_line for lines with at most 4 rings open at
// once and colours < 8; otherwise RN_FALLBACK (the caller restores the line
// from HBM and runs preprocess_line).  On any return other than E_NONE the
// line bytes may be partially rewritten.
// ----------------------------------------------------------------------------
constexpr int RN_FALLBACK = -4;

// Tokenizer transducer (smiles.py:83-137 as an 8-state machine).  Entry =
// tk[state << 8 | byte]: bits 0-2 next state, TK_RING = a ring-closure token
// starts here, TK_CR = '\r', TK_ENTER_BR / TK_ENTER_PCT = this byte is a '['
// opening a bracket atom / a '%' starting a %nn token (outside brackets).
enum : unsigned {
    TK_OUT0 = 0, TK_OUT1 = 1,  // outside brackets; ring_ok = 0 / 1
    TK_IN = 2,                 // inside a bracket atom
    TK_ERR = 3,                // '%' not followed by two digits (sticky)
    TK_P1R = 4, TK_P2R = 5,    // after '%' / '%d' of a ring-closure %nn token
    TK_P1O = 6, TK_P2O = 7,    // ... of an Other %nn token
    TK_RING = 8, TK_CR = 16, TK_ENTER_BR = 32, TK_ENTER_PCT = 64
};

ZS_HD uint8_t tk_entry(unsigned st, unsigned b) {
    const uint8_t c = tok_class(b);
    const unsigned cr = c == C_CR ? TK_CR : 0u;
    switch (st) {
    case TK_OUT0:
    case TK_OUT1: {
        const bool ok = st == TK_OUT1;
        switch (c) {
        case C_LBR: return TK_IN | TK_ENTER_BR;
        case C_PCT: return (ok ? TK_P1R | TK_RING : TK_P1O) | TK_ENTER_PCT;
        case C_DIGIT: return ok ? TK_OUT1 | TK_RING : TK_OUT0;
        case C_ATOM:
        case C_BOND: return TK_OUT1;
        default: return TK_OUT0 | cr;  // ( ) . stray ] and any other byte
        }
    }
    case TK_IN: return b == ']' ? TK_OUT1 : TK_IN | cr;
    case TK_P1R: return c == C_DIGIT ? TK_P2R : TK_ERR | cr;
    case TK_P2R: return c == C_DIGIT ? TK_OUT1 : TK_ERR | cr;
    case TK_P1O: return c == C_DIGIT ? TK_P2O : TK_ERR | cr;
    case TK_P2O: return c == C_DIGIT ? TK_OUT0 : TK_ERR | cr;
    default: return TK_ERR | cr;
    }
}
enum : uint8_t { K_OKP = 1, K_DIG = 2, K_PCT = 4, K_LBR = 8, K_CR = 16, K_SPECIAL = K_PCT | K_LBR | K_CR };

ZS_HD uint8_t tok_bits(unsigned b) {
    uint8_t c = tok_class(b);
    return c == C_ATOM || c == C_BOND ? K_OKP : c == C_DIGIT ? K_DIG : c == C_PCT ? K_PCT
         : c == C_LBR ? K_LBR : c == C_CR ? K_CR : 0;
}

// next ring token after chain node i (step = marks[i] != 0); 255 = hop of 254
ZS_HD int chain_next(const uint8_t *marks, int i, unsigned step) {
    while (step == 255) {
        i += 254;
        step = marks[i];
    }
    return i + step;
}

// All 32 lanes of a warp must call renumber_fast together (lanes with
// nothing to do pass n = 0): its loops are warp-uniform (ZS_ANY) so the lanes
// stay converged trip by trip under independent thread scheduling.
ZS_HD int renumber_fast(uint8_t *s, int n, const uint8_t *lut, uint8_t *marks,
                        int *new_len, int *err_off, unsigned long long ids[2]) {
    int res = E_NONE;
    // ---- 1. tokenize (one table lookup per byte) ----
    // Ring-token positions go to a u16 list in the line's scratch (marks,
    // 2-byte aligned): a predicated store per byte, no branch.  A line with
    // more ring tokens than the list holds (> ~n/2) takes the fallback.
    uint16_t *list = reinterpret_cast<uint16_t *>(reinterpret_cast<uintptr_t>(marks + 1) & ~(uintptr_t)1);
    const int cap = (n - 1) / 2;
    int cnt = 0, br = -1, pct = -1, n_pct = 0;
    unsigned st = TK_OUT0, crs = 0;
    const SmemBytes sb(s), tk(lut);
    for (int i = 0; ZS_ANY(i < n); ++i) {
        if (i >= n) continue;
        const unsigned e = tk.ld((st << 8) | sb.ld(i));
        st = e & 7u;
        crs |= e;
        br = (e & TK_ENTER_BR) ? i : br;
        pct = (e & TK_ENTER_PCT) ? i : pct;
        const bool ring = e & TK_RING;
        n_pct += ring & ((e & TK_ENTER_PCT) != 0);
        if (ring && cnt < cap) list[cnt] = (uint16_t)i;
        cnt += ring;
    }
    if (crs & TK_CR) {
        res = E_CR;  // '\r' anywhere in the line takes precedence (pipeline.py:102-107)
    } else if (st == TK_ERR || st >= TK_P1R) {
        *err_off = pct;  // '%' without two digits (the first such '%' wins: ERR is sticky)
        res = E_PERCENT;
    } else if (st == TK_IN) {
        *err_off = br;  // '[' never closed
        res = E_BRACKET;
    } else if (cnt > cap) {
        res = RN_FALLBACK;
    }
    // ---- 2. pair + colour along the list ----
    unsigned oid = 0xffffffffu;  // 4 slots: open ring id per byte, 0xff = free
    int opos[4] = {0, 0, 0, 0};
    int lc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) lc[k] = -1;
    const int ntok = res == E_NONE ? cnt : 0;
    for (int t = 0; ZS_ANY(t < ntok && res == E_NONE); ++t) {
        if (t >= ntok || res != E_NONE) continue;
        const int i = list[t];
        const bool pct_tok = sb.ld(i) == '%';
        const unsigned rid = pct_tok ? (sb.ld(i + 1) - '0') * 10u + (sb.ld(i + 2) - '0') : sb.ld(i) - '0';
        int slot = -1, free_slot = -1;
#pragma unroll
        for (int k = 3; k >= 0; --k) {
            const unsigned v = (oid >> (8 * k)) & 0xffu;
            if (v == rid) slot = k;
            if (v == 0xffu) free_slot = k;
        }
        if (slot < 0) {
            if (free_slot < 0) {
                res = RN_FALLBACK;
                continue;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k == free_slot) opos[k] = i;
            oid = (oid & ~(0xffu << (8 * free_slot))) | (rid << (8 * free_slot));
        } else {
            int o = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k == slot) o = opos[k];
            oid |= 0xffu << (8 * slot);
            int col = 8;
#pragma unroll
            for (int k = 7; k >= 0; --k)
                if (lc[k] <= o) col = k;
            if (col == 8) {
                res = RN_FALLBACK;
                continue;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k == col) lc[k] = i;
            // colour digits: 1-byte tokens in place, '%nn' tokens in their
            // first digit slot (compacted below)
            s[o + (s[o] == '%')] = (uint8_t)('0' + col);
            s[i + pct_tok] = (uint8_t)('0' + col);
        }
    }
    if (res == E_NONE && oid != 0xffffffffu) {
        ids[0] = ids[1] = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned v = (oid >> (8 * k)) & 0xffu;
            if (v != 0xffu) ids[v >> 6] |= 1ull << (v & 63);
        }
        res = E_UNPAIRED;
    }
    // ---- 3. compaction of '%nn' ring tokens (rare: no warp-uniform loop) ----
    *new_len = n;
    if (res == E_NONE && n_pct) {
        int w = list[0], r = list[0];
        for (int t = 0; t < cnt; ++t) {
            const int i = list[t];
            while (r < i) s[w++] = s[r++];
            if (s[i] == '%') {
                s[w++] = s[i + 1];
                r = i + 3;
            }
        }
        while (r < n) s[w++] = s[r++];
        *new_len = w;
    }
    return res;
}

// ----------------------------------------------------------------------------
// Bitmap variant of renumber_fast for the in-place compress kernel: the
// ring-token starts are set in a shared bitmap (bit = window position,
// atomicOr since neighbouring lines share words) instead of a per-line list,
// so the line needs no scratch bytes.  bit0 = window position of s[0].
// Same contract as renumber_fast (all 32 lanes call together).
// ----------------------------------------------------------------------------
ZS_HD void bm_set(unsigned *bm, int pos) {
#ifdef __CUDA_ARCH__
    atomicOr(&bm[pos >> 5], 1u << (pos & 31));
#else
    bm[pos >> 5] |= 1u << (pos & 31);
#endif
}

// next set bit at or after pos within [pos, end); -1 if none
ZS_HD int bm_next(const unsigned *bm, int pos, int end) {
    while (pos < end) {
        unsigned w = bm[pos >> 5] >> (pos & 31);
        if (w) {
            const int q = pos + ffs64_(w) - 1;
            return q < end ? q : -1;
        }
        pos = (pos | 31) + 1;
    }
    return -1;
}

ZS_HD int renumber_bm(uint8_t *s, int n, const uint8_t *lut, unsigned *rbits, int bit0,
                      int *new_len, int *err_off, unsigned long long ids[2]) {
    int res = E_NONE;
    // ---- 1. tokenize (one table lookup per byte); mark ring-token starts ----
    int cnt = 0, br = -1, pct = -1, n_pct = 0;
    unsigned st = TK_OUT0, crs = 0;
    const SmemBytes sb(s), tk(lut);
    for (int i = 0; ZS_ANY(i < n); ++i) {
        if (i >= n) continue;
        const unsigned e = tk.ld((st << 8) | sb.ld(i));
        st = e & 7u;
        crs |= e;
        br = (e & TK_ENTER_BR) ? i : br;
        pct = (e & TK_ENTER_PCT) ? i : pct;
        const bool ring = e & TK_RING;
        n_pct += ring & ((e & TK_ENTER_PCT) != 0);
        if (ring) bm_set(rbits, bit0 + i);
        cnt += ring;
    }
    if (crs & TK_CR) {
        res = E_CR;  // '\r' anywhere in the line takes precedence (pipeline.py:102-107)
    } else if (st == TK_ERR || st >= TK_P1R) {
        *err_off = pct;  // '%' without two digits (the first such '%' wins: ERR is sticky)
        res = E_PERCENT;
    } else if (st == TK_IN) {
        *err_off = br;  // '[' never closed
        res = E_BRACKET;
    }
    // ---- 2. pair + colour, tokens in order ----
    unsigned oid = 0xffffffffu;  // 4 slots: open ring id per byte, 0xff = free
    int opos[4] = {0, 0, 0, 0};
    int lc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) lc[k] = -1;
    const int ntok = res == E_NONE ? cnt : 0;
    int cur = bit0 - 1;
    for (int t = 0; ZS_ANY(t < ntok && res == E_NONE); ++t) {
        if (t >= ntok || res != E_NONE) continue;
        cur = bm_next(rbits, cur + 1, bit0 + n);
        const int i = cur - bit0;
        const bool pct_tok = sb.ld(i) == '%';
        const unsigned rid = pct_tok ? (sb.ld(i + 1) - '0') * 10u + (sb.ld(i + 2) - '0') : sb.ld(i) - '0';
        int slot = -1, free_slot = -1;
#pragma unroll
        for (int k = 3; k >= 0; --k) {
            const unsigned v = (oid >> (8 * k)) & 0xffu;
            if (v == rid) slot = k;
            if (v == 0xffu) free_slot = k;
        }
        if (slot < 0) {
            if (free_slot < 0) {
                res = RN_FALLBACK;
                continue;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k == free_slot) opos[k] = i;
            oid = (oid & ~(0xffu << (8 * free_slot))) | (rid << (8 * free_slot));
        } else {
            int o = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k == slot) o = opos[k];
            oid |= 0xffu << (8 * slot);
            int col = 8;
#pragma unroll
            for (int k = 7; k >= 0; --k)
                if (lc[k] <= o) col = k;
            if (col == 8) {
                res = RN_FALLBACK;
                continue;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k == col) lc[k] = i;
            s[o + (s[o] == '%')] = (uint8_t)('0' + col);
            s[i + pct_tok] = (uint8_t)('0' + col);
        }
    }
    if (res == E_NONE && oid != 0xffffffffu) {
        ids[0] = ids[1] = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned v = (oid >> (8 * k)) & 0xffu;
            if (v != 0xffu) ids[v >> 6] |= 1ull << (v & 63);
        }
        res = E_UNPAIRED;
    }
    // ---- 3. compaction of '%nn' ring tokens (rare) ----
    *new_len = n;
    if (res == E_NONE && n_pct) {
        int w = -1, r = 0;
        for (int q = bm_next(rbits, bit0, bit0 + n); q >= 0; q = bm_next(rbits, q + 1, bit0 + n)) {
            const int i = q - bit0;
            if (w < 0) w = r = i;
            while (r < i) s[w++] = s[r++];
            if (s[i] == '%') {
                s[w++] = s[i + 1];
                r = i + 3;
            }
        }
        while (r < n) s[w++] = s[r++];
        *new_len = w;
    }
    return res;
}

// dp_t2 writing its decisions over the line bytes (each byte is read once,
// right to left, before its decision replaces it).  Escapes keep the literal
// byte and set its bit in `ebits` (bit0 = window position of s[0]).
ZS_HD int dp_t2_inplace(uint8_t *s, int n, const uint16_t *dfa2, const uint32_t *t2,
                        const uint8_t *codes, unsigned *ebits, int bit0) {
    unsigned st = 0, wi = 0;
    int cost = 0;
    for (int i = n - 1; i >= 0; --i) {
        const unsigned b = s[i];
        const unsigned e = dfa2[st * NCOL + dcol(b)];
        st = e & 0xffu;
        const unsigned x = t2[wi * T2_MASKS + (e >> 8)];
        wi = x & 0xfffu;
        const unsigned L = (x >> 12) & 15u;
        cost += (int)(x >> 16) - 16;
        if (L) s[i] = codes[st * FAST_W + L - 1];
        else bm_set(ebits, bit0 + i);
    }
    return cost;
}

// ----------------------------------------------------------------------------
// min-cost parse, fast path: reversed AC DFA in smem, W <= 8.
//
// key(j) = (cost[j] << 3) - j.  Among candidates j in (i, i+W], a smaller key
// means cheaper, and at equal cost the larger j (= longer match), which is
// exactly the reference's replacement rule (numba_impl.py:50).  The escape
// edge (cost 2 + cost[i+1]) loses every tie because it shares j = i+1 with
// the length-1 match only, which is strictly cheaper.
// s[0..n) line bytes, dec[0..n] decisions out.  Returns cost[0].
// ----------------------------------------------------------------------------
template <int W>
ZS_HD int dp_fast(const uint8_t *s, int n, uint8_t *dec,
                                       const uint16_t *dfa, const uint8_t *codes) {
    constexpr int INF = 0x3fffffff;
    int k[W + 1];
#pragma unroll
    for (int L = 1; L <= W; ++L) k[L] = INF;
    // position n: cost 0
    int key = -n;
    int st = 0;
    dec[n] = D_END;
    for (int i = n - 1; i >= 0; --i) {
        // shift window: k[L] = key of position i+L
#pragma unroll
        for (int L = W; L > 1; --L) k[L] = k[L - 1];
        k[1] = key;
        unsigned b = s[i];
        unsigned e = dfa[st * NCOL + dcol(b)];
        st = e & 0xffu;
        int mm = INF;
#pragma unroll
        for (int L = 1; L <= W; ++L)
            if (e & (0x100u << (L - 1))) mm = imin_(mm, k[L]);
        int esc = k[1] + (2 << 3);
        int best = imin_(esc, mm + (1 << 3));
        int t = best + i + W;
        int L = W - (t & 7);
        key = (t & ~7) - i;
        uint8_t code = codes[st * FAST_W + L - 1];
        dec[i] = esc < mm + (1 << 3) ? D_ESC : code;
    }
    return key >> 3;  // position 0: key = cost[0] << 3
}

// ----------------------------------------------------------------------------
// min-cost parse through the cost-window transducer: per byte one AC-DFA
// lookup (next state, match-mask index) and one t2 lookup (next relative cost
// window, chosen length, cost delta).  Same decisions as dp_fast by
// construction (build_t2 enumerates exactly dp_fast's step).  Returns cost[0].
// ----------------------------------------------------------------------------
ZS_HD int dp_t2(const uint8_t *s, int n, uint8_t *dec, const uint16_t *dfa2, const uint32_t *t2,
                const uint8_t *codes) {
    unsigned st = 0, wi = 0;
    int cost = 0;
    dec[n] = D_END;
    for (int i = n - 1; i >= 0; --i) {
        const unsigned b = s[i];
        const unsigned e = dfa2[st * NCOL + dcol(b)];
        st = e & 0xffu;
        const unsigned x = t2[wi * T2_MASKS + (e >> 8)];
        wi = x & 0xfffu;
        const unsigned L = (x >> 12) & 15u;
        cost += (int)(x >> 16) - 16;
        dec[i] = L ? codes[st * FAST_W + L - 1] : D_ESC;
    }
    return cost;
}

// ----------------------------------------------------------------------------
// min-cost parse, generic path: the reference trie walk (numba_impl.py:37-56)
// over the dense HBM trie; keys (cost<<7)-j in a 128-entry ring buffer so any
// pattern length <= 64 works.  s/dec may live in smem or HBM.
// ----------------------------------------------------------------------------
__device__ long long dp_generic(const uint8_t *s, long long n, uint8_t *dec, const Tables &tb,
                                long long *ring /* 128 entries */) {
    ring[n & 127] = -n;  // key of position n: cost 0
    dec[n] = D_END;
    for (long long i = n - 1; i >= 0; --i) {
        long long best = ring[(i + 1) & 127] + (2ll << 7);
        int bc = -1;
        int node = 0;
        for (long long j = i; j < n; ++j) {
            node = __ldg(&tb.children[(long long)node * 256 + s[j]]);
            if (node < 0) break;
            int tc = __ldg(&tb.term_code[node]);
            if (tc < 0) continue;
            long long cand = ring[(j + 1) & 127] + (1ll << 7);
            if (cand < best) {  // keys encode "cheaper, then longer"
                best = cand;
                bc = tc;
            }
        }
        long long t = best + i + 127;
        ring[i & 127] = (t & ~127ll) - i;
        dec[i] = bc < 0 ? D_ESC : (uint8_t)bc;
    }
    return ring[0] >> 7;
}

}  // namespace zs
