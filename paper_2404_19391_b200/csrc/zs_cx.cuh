// zs_cx.cuh -- lane-chunk compress kernel (the encode hot path).
//
// Three persistent 256-thread CTAs per SM take 19,968-byte tiles in ticket
// order.  A tile owns the lines whose terminating '\n' lies inside it (their
// first bytes may sit in the 2 KB staged before the tile).  Every lane owns
// a contiguous run of whole lines, ~78 bytes, cut at the newline nearest to
// its chunk boundary, and walks it in straight loops that all lanes of a
// warp execute in lock step (no per-line queues, sorting or barriers):
//
//   P1  newline bitmap of the staged window (block-cooperative SWAR), lane
//       ranges from the nearest-newline cuts (two block scans)
//   P2  tokenizer (smiles.py:83-137 as an 8-state table transducer): CR and
//       tokenize errors per line, ring-token starts OR'ed into the bitmap
//   P3  ring pairing + colouring (smiles.py:140-213) walking the bitmap's
//       events: open rings in 4 register slots, colours 0-9 from per-colour
//       last-close positions; '%nn' lines are compacted in place with the
//       freed bytes left as a gap of escape-only filler before the '\n'
//   --  rare lines (drops, strict errors, lines the fast path cannot renumber)
//       are rewritten to escape-only filler and handled by one thread each
//       (general routine, HBM arena); lines longer than the staged window are
//       recorded for the long-line kernels (zs_ll.cuh) and placed by them
//   P4  min-cost parse right to left across the lane's lines
//       (numba_impl.py:32-56): per byte one AC-DFA lookup and one lookup in
//       the cost-window transducer; '\n' is a DFA column whose transducer
//       entry resets the window and emits the record separator, so the walk
//       never branches on line ends.  Decisions overwrite the bytes in place.
//   P5  lane output bytes -> block scan -> decoupled look-back publish
//   P6  forward walk of the decisions (numba_impl.py:57-69) into an smem
//       staging buffer, then aligned 16-byte stores at the resolved offset.
//
// Escape decisions are the byte 0x20 (never a code); the emit re-reads the
// literal from the input in HBM.  `rbits` marks the newlines (P1), `gbits`
// the ring-token starts P2 found (P3 walks them), `fbits` filler and
// arena-marker positions (P6).
#pragma once
#include "zs_kernels.cuh"
#ifdef ZS_CHECKS
#include <cassert>
#define ZS_ASSERT(c) assert(c)
#else
#define ZS_ASSERT(c) ((void)0)
#endif

namespace zs {

constexpr int CX_NT = 256;
constexpr int CX_NW = CX_NT / 32;
constexpr int CX_CC = 78;                         // bytes of line ends per lane (tile 19,968 B)
constexpr int CX_TILE = CX_NT * CX_CC;
constexpr int CX_HEAD = 2048;                     // staged before the tile
constexpr int CX_WIN = CX_HEAD + CX_TILE;         // multiple of 32 (bitmap words)
constexpr int CX_WORDS = CX_WIN / 32 + 4;         // bitmap words (multiple of 4: keeps the carve 16-aligned)
constexpr int CX_NCOL = 119;                      // dcol: umin(b - 10, 118); 0 = '\n'
constexpr int CX_NLMASK = 15;                     // transducer mask slot of '\n'
constexpr int CX_CODES = 20;                      // code-slot row stride (0 escape, 1-8 match, 9 '\n'; 5 words:
                                                  // rows of random states spread over the 32 banks)
constexpr int CX_LUTS = 260;                      // tokenizer LUT row stride (65 words)
constexpr int CX_T2S = 18;                        // transducer row stride in u16 (9 words, same reason)
constexpr int CX_OUTCAP = 11264;                  // staging (tile output up to ratio ~0.55)
constexpr int CX_RARE = 64;                       // rare lines per tile
constexpr int CX_JOBS = 16;                       // '%nn' compactions per warp and tile
constexpr int CX_WARM = 32;                       // P4 warm-up bytes right of a slice (speculative entry)
constexpr int CX_XLONG = 4 * CX_CC;               // P4 uses byte-exact slices when a line-lane range is longer
constexpr int CX_PWARM = 8;                       // PA: warm-up bytes of a slice's guessed P4 / P6 entry
static_assert((CX_WIN + CX_NT) / CX_NT + 31 <= 128, "a P3 slice spans at most 4 bitmap words");

// rare-line kinds
enum : int { RK_DROP = 1, RK_ARENA = 2, RK_STRICT = 3 };

struct CxRare {
    int ls, le;        // window positions: first byte, terminating '\n'
    int kind;          // RK_*
    int lane;
    int local;         // line index within the lane
    int err;           // E_* (strict errors)
    unsigned aoff;     // arena offset / 16 (RK_ARENA)
    int out;           // output bytes of the arena line incl. its '\n' (RK_ARENA)
    int glob;          // the line starts before the window (only its '\n' at le is staged)
    long long gs;      // global offset of the line's first byte (RK_ARENA)
    int ll;            // RK_ARENA coded by the long-line kernels: its Job.ll entry; -1 = none
};

__host__ __device__ inline int cx_align16(int x) { return (x + 15) & ~15; }

// Shared-memory layout: the fixed-size buffers first, at compile-time
// offsets, then the dictionary tables (their sizes depend on the dictionary;
// the host passes the table offsets as kernel parameters).  Constant offsets
// keep the compiler from rebuilding buffer addresses inside the hot loops.
constexpr int CX_O_WIN = 0;
constexpr int CX_O_FB = CX_O_WIN + ((CX_WIN + 32 + 15) & ~15);
// rbits / gbits are dead once P4 starts: P6 stages its output from their
// start on (CX_STAGE bytes), so dictionaries with a ratio up to ~0.8 still
// emit through shared memory
constexpr int CX_O_RB = CX_O_FB + CX_WORDS * 4;
constexpr int CX_O_EB = CX_O_RB + CX_WORDS * 4;
constexpr int CX_O_OUT = CX_O_EB + CX_WORDS * 4;
constexpr int CX_STAGE = CX_O_OUT + CX_OUTCAP - CX_O_RB;
constexpr int CX_O_RARE = CX_O_OUT + CX_OUTCAP;
constexpr int CX_O_LA = CX_O_RARE + CX_RARE * (int)sizeof(CxRare);
constexpr int CX_O_LB = CX_O_LA + CX_NT * 4;
constexpr int CX_O_LC = CX_O_LB + CX_NT * 4;
constexpr int CX_O_LF = CX_O_LC + CX_NT * 4;      // per line-lane: first in-window line byte | glob << 30
constexpr int CX_O_JOBS = CX_O_LF + CX_NT * 4;
constexpr int CX_O_NJOBS = CX_O_JOBS + CX_NW * CX_JOBS * 16;
constexpr int CX_POOL = 1536;                     // P3 (PA): lines with ring events per tile, sorted
constexpr int CX_HIST = 64;                       // P3 (PA): event-count buckets
constexpr int CX_O_POOL = (CX_O_NJOBS + CX_NW * 4 + 15) & ~15;
constexpr int CX_O_HIST = CX_O_POOL + CX_POOL * 4;
constexpr int CX_O_CODES = (CX_O_HIST + CX_HIST * 4 + 15) & ~15;  // code slots, when they fit here
constexpr int CX_CODES_CAP = 256 * CX_CODES;                        // (transducer DFAs: <= 256 states)
constexpr int CX_O_DFA = CX_O_CODES + CX_CODES_CAP;

// Per kernel variant: resident CTAs per SM and where the dictionary tables
// start.  The default kernel (product automaton, line-lane phases) needs
// neither the P3 line pool / buckets (slices only) nor the code slots
// (DFA + transducer only), so its tables follow the job lists and three CTAs
// fit an SM: barriers of one CTA are covered by two others.
template <bool PA, bool SL>
__host__ __device__ constexpr int cx_ctas() { return (PA && !SL) ? 3 : 2; }
template <bool PA, bool SL>
__host__ __device__ constexpr int cx_o_tab() { return (PA && !SL) ? CX_O_POOL : PA ? CX_O_CODES : CX_O_DFA; }
static_assert(CX_O_JOBS % 16 == 0, "int4 job slots");

struct CxLayout {
    int o_t2, o_codes, bytes;
};

__host__ __device__ inline CxLayout cx_layout(int ns, int nw, int nc) {
    CxLayout L;
    L.o_t2 = CX_O_DFA + cx_align16(ns * nc * 2);
    const int end_t2 = L.o_t2 + cx_align16(nw * CX_T2S * 2);
    const bool fixed = ns * CX_CODES <= CX_CODES_CAP;  // compile-time offset in the parse loop
    L.o_codes = fixed ? CX_O_CODES : end_t2;
    L.bytes = fixed ? end_t2 : end_t2 + cx_align16(ns * CX_CODES);
    return L;
}

__host__ __device__ inline int cx_smem_bytes(int ns, int nw, int nc) { return cx_layout(ns, nw, nc).bytes; }

// device tables of the lane-chunk kernel (built by build_cx, zs_api.cu): the
// minimised reversed-pattern DFA over byte-class columns, the cost-window
// transducer, code slots per state and the byte -> column map
struct CxTables {
    const uint16_t *dfa;   // [states][cols] = next | mask index << 8
    const uint16_t *t2;    // [windows][16] = next window | L << 9 | (cost delta + 4) << 13
    const uint8_t *codes;  // [states][16]
    const uint8_t *cmap;   // [256]
    int ns, nw, nc;
    int o_t2, o_codes;     // smem offsets (cx_layout)
    int p4x;               // 1: byte-exact parse slices (default), 0: parse the lane's line range
    int kw;                // 1: key-window parse (patterns up to 16 bytes; dfa = u32 [states][nc/2])
    int o_ring;            // kw: per-thread key rings (cx_kw_ring_bytes) at this smem offset
    const uint32_t *pa;    // compress_cx<true>: parse automaton [ns][nc] (build_pa); cmap = column * 4
};

// shared memory of compress_cx<true>: the fixed buffers, then the parse automaton
__host__ __device__ inline int cx_pa_smem_bytes(int ns, int nc, bool slices) {
    return (slices ? cx_o_tab<true, true>() : cx_o_tab<true, false>()) + cx_align16(ns * nc * 4);
}

// kw: a 32-entry key ring per thread (stride 33 words: conflict-free banks)
constexpr int CX_KW_RING = 33;
__host__ __device__ inline int cx_kw_ring_bytes() { return CX_NT * CX_KW_RING * 4; }

struct CxSmem {
    uint16_t *dfa;
    uint16_t *t2;
    uint8_t *codes;
    uint8_t *explen;
    uint8_t *lut;
    uint8_t *win;
    unsigned *rbits, *gbits, *fbits;  // newlines (P1), ring-token starts (P2), filler (P6)
    uint8_t *out;
    CxRare *rare;
    int *lane_a, *lane_b, *lane_c, *lane_f;
    int4 *jobs;   // [warp][CX_JOBS] (ls, q, owner lane, local line index)
    int *njobs;   // [warp]
    uint32_t *pool;  // [CX_POOL] lines with ring events: first event | '\n' << 16 (P3, PA)
    int *hist;       // [CX_HIST] event-count buckets (P3, PA)
};

__device__ inline CxSmem cx_carve(uint8_t *p, int o_t2, int o_codes, int o_tab) {
    CxSmem S;
    S.win = p + CX_O_WIN;
    S.rbits = reinterpret_cast<unsigned *>(p + CX_O_RB);
    S.gbits = reinterpret_cast<unsigned *>(p + CX_O_EB);
    S.fbits = reinterpret_cast<unsigned *>(p + CX_O_FB);
    S.out = p + CX_O_RB;  // P6 staging: rbits + gbits + the out buffer (CX_STAGE bytes)
    S.rare = reinterpret_cast<CxRare *>(p + CX_O_RARE);
    S.lane_a = reinterpret_cast<int *>(p + CX_O_LA);
    S.lane_b = reinterpret_cast<int *>(p + CX_O_LB);
    S.lane_c = reinterpret_cast<int *>(p + CX_O_LC);
    S.lane_f = reinterpret_cast<int *>(p + CX_O_LF);
    S.jobs = reinterpret_cast<int4 *>(p + CX_O_JOBS);
    S.njobs = reinterpret_cast<int *>(p + CX_O_NJOBS);
    S.pool = reinterpret_cast<uint32_t *>(p + CX_O_POOL);
    S.hist = reinterpret_cast<int *>(p + CX_O_HIST);
    S.dfa = reinterpret_cast<uint16_t *>(p + o_tab);
    S.t2 = reinterpret_cast<uint16_t *>(p + o_t2);
    S.codes = p + o_codes;
    return S;
}

// explicit 32-bit shared addresses in the hot loops (a generic pointer makes
// the compiler rebuild the shared window base inside every loop trip)
__device__ __forceinline__ unsigned cx_lb(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned cx_lh(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned cx_lw(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void cx_sb(unsigned a, unsigned v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cx_or(unsigned a, unsigned v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned cx_bit(const unsigned *bm, int p) { return (bm[p >> 5] >> (p & 31)) & 1u; }
__device__ __forceinline__ void cx_set(unsigned *bm, int p) { atomicOr(&bm[p >> 5], 1u << (p & 31)); }
__device__ __forceinline__ void cx_clr(unsigned *bm, int p) { atomicAnd(&bm[p >> 5], ~(1u << (p & 31))); }

// set bits of bm in window positions [a, b]
__device__ __forceinline__ int cx_popc_range(const unsigned *bm, int a, int b) {
    int n = 0;
    for (int w = a >> 5; a <= b && w <= (b >> 5); ++w) {
        unsigned m = bm[w];
        if (w == (a >> 5)) m &= 0xffffffffu << (a & 31);
        if (w == (b >> 5) && (b & 31) != 31) m &= (2u << (b & 31)) - 1u;
        n += __popc(m);
    }
    return n;
}

// first set bit at position >= p (bm bits beyond the window are never set;
// callers bound the search by a position known to be set)
__device__ __forceinline__ int cx_next(const unsigned *bm, int p) {
    int w = p >> 5;
    unsigned m = bm[w] & (0xffffffffu << (p & 31));
    while (!m) m = bm[++w];
    return (w << 5) + __ffs(m) - 1;
}

// block-wide inclusive max / min scans (CX_NT threads); tmp: CX_NW ints
template <bool MAX>
__device__ __forceinline__ int cx_block_scan_mm(int v, int *tmp, bool exclusive, int ident) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = MAX ? max(x, y) : min(x, y);
    }
    if (lane == 31) tmp[wid] = x;
    __syncthreads();
    int pre = ident;
    for (int k = 0; k < wid; ++k) pre = MAX ? max(pre, tmp[k]) : min(pre, tmp[k]);
    int ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = ident;
    ex = MAX ? max(pre, ex) : min(pre, ex);
    const int inc = MAX ? max(pre, x) : min(pre, x);
    __syncthreads();
    return exclusive ? ex : inc;
}

// suffix min scan (from the right) via a reversed index
__device__ __forceinline__ int cx_block_suffix_min(int v, int *tmp) {
    // lane order reversed: thread t holds v of t; compute min over t' >= t
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_down_sync(0xffffffffu, x, o);
        if (lane + o < 32) x = min(x, y);
    }
    if (lane == 0) tmp[wid] = x;
    __syncthreads();
    int post = 0x7fffffff;
    for (int k = wid + 1; k < CX_NW; ++k) post = min(post, tmp[k]);
    const int r = min(post, x);
    __syncthreads();
    return r;
}

// emit one arena line (compress_line_global output) at o[w...]; returns escapes
__device__ __forceinline__ unsigned cx_emit_arena(const Job &job, const uint8_t *explen, unsigned aoff,
                                                  uint8_t *o, unsigned long long &w, long long raw_gs) {
    unsigned esc = 0;
    const uint8_t *blk = job.arena + ((long long)aoff << 4);
    const ArenaHdr *h = reinterpret_cast<const ArenaHdr *>(blk);
    const uint8_t *bytes = h->bytes_off < 0 ? job.in + raw_gs : job.arena + h->bytes_off;
    const uint8_t *dec = job.arena + h->dec_off;
    for (long long i = 0; i < h->n_pre;) {
        const uint8_t c = dec[i];
        if (c == D_ESC) {
            o[w++] = 0x20;
            o[w++] = bytes[i];
            ++esc;
            ++i;
        } else {
            ZS_ASSERT(explen[c] != 0);
            o[w++] = c;
            i += explen[c];
        }
    }
    o[w++] = '\n';
    return esc;
}

// P6 walk of one lane range [p0, p1] into o at w (STAGED: o is the smem
// staging buffer).  A decision byte 0x20 is an escape (literal re-read from
// the input in HBM) unless `fbits` marks the position as filler or as an
// arena line's marker.
template <bool STAGED>
__device__ __forceinline__ unsigned cx_emit_range(const Job &job, const CxSmem &S, long long ws, int p0, int p1,
                                                  uint8_t *o, unsigned long long w, int n_rare) {
    unsigned esc = 0;
    const uint8_t *__restrict__ win = S.win;
    const uint8_t *__restrict__ explen = S.explen;
    if constexpr (STAGED) {
        // explicit 32-bit shared addresses: with generic pointers the compiler
        // rebuilds the shared window base (S2R SR_CgaCtaId, LEA) every code
        const unsigned wb = (unsigned)__cvta_generic_to_shared(win), eb = (unsigned)__cvta_generic_to_shared(explen);
        const unsigned ob = (unsigned)__cvta_generic_to_shared(o);
        unsigned ww = (unsigned)w;
        auto lb = [](unsigned a) {  // pure load: the window and explen do not change during the walk
            unsigned v;
            asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
            return v;
        };
        for (int p = p0; p <= p1;) {
            const unsigned c = lb(wb + (unsigned)p);
            if (c == 0x20) {
                w = ww;
                if (cx_bit(S.fbits, p)) {
                    for (int r = 0; r < n_rare; ++r)  // an arena line's marker?
                        if (S.rare[r].kind == RK_ARENA && (S.rare[r].glob ? S.rare[r].le : S.rare[r].ls) == p) {
                            const unsigned long long w0 = w;
                            ZS_ASSERT(S.rare[r].ll < 0);  // tiles with long lines emit direct
                            esc += cx_emit_arena(job, S.explen, S.rare[r].aoff, o, w, S.rare[r].gs);
                            ZS_ASSERT(w - w0 == (unsigned long long)S.rare[r].out);
                        }
                } else {
                    o[w] = 0x20;
                    o[w + 1] = job.in[ws + p];
                    w += 2;
                    ++esc;
                }
                ww = (unsigned)w;
                ZS_ASSERT(ww <= (unsigned)CX_STAGE);
                ++p;
            } else {
                ZS_ASSERT(ww < (unsigned)CX_STAGE);
                asm volatile("st.shared.u8 [%0], %1;" ::"r"(ob + ww), "r"(c) : "memory");
                ++ww;
                p += (int)lb(eb + c);
            }
        }
        return esc;
    } else {
        for (int p = p0; p <= p1;) {
            const unsigned c = win[p];
            if (c == 0x20) {
                if (cx_bit(S.fbits, p)) {
                    for (int r = 0; r < n_rare; ++r)  // an arena line's marker?
                        if (S.rare[r].kind == RK_ARENA && (S.rare[r].glob ? S.rare[r].le : S.rare[r].ls) == p) {
                            if (S.rare[r].ll >= 0) {  // long line: its bytes are placed by ll_place
                                LLine &L = job.ll[S.rare[r].ll];
                                L.dst = (long long)w;
                                w += (unsigned long long)S.rare[r].out;
                                esc += (unsigned)L.esc;
                            } else {
                                esc += cx_emit_arena(job, S.explen, S.rare[r].aoff, o, w, S.rare[r].gs);
                            }
                        }
                } else {
                    o[w] = 0x20;
                    o[w + 1] = job.in[ws + p];
                    w += 2;
                    ++esc;
                }
                ++p;
            } else {
                o[w++] = (uint8_t)c;
                p += explen[c];
            }
        }
        return esc;
    }
}

// ---- asynchronous bulk copies (TMA engine) into shared memory ----
__device__ __forceinline__ unsigned cx_saddr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cx_mbar_init(uint64_t *mbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cx_saddr(mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one thread: arm the mbarrier with `bytes` and copy global [src, src+bytes)
// to shared dst in pieces (src, dst 16-byte aligned, bytes a multiple of 16)
__device__ __forceinline__ void cx_bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *mbar) {
    const unsigned mb = cx_saddr(mbar), d = cx_saddr(dst);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic accesses first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    constexpr unsigned PIECE = 8192;
    for (unsigned o = 0; o < bytes; o += PIECE) {
        const unsigned nb = bytes - o < PIECE ? bytes - o : PIECE;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(d + o), "l"(reinterpret_cast<const char *>(src) + o), "r"(nb), "r"(mb)
                     : "memory");
    }
}
__device__ __forceinline__ void cx_mbar_wait(uint64_t *mbar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(cx_saddr(mbar)), "r"(parity) : "memory");
}

// Stage window bytes [ws, ws+len) (positions before the buffer read as '\n'
// so offset 0 is a line start; positions past the end as '\n').  Interior
// windows of a 16-byte aligned buffer arrive by one bulk copy (TMA) that
// thread 0 issued (returns true: wait on the mbarrier); windows of an
// unaligned buffer are read as aligned 16-byte chunks and shifted into place
// in registers; the first and last windows of a buffer bytewise.
__device__ __forceinline__ bool cx_load_window(const uint8_t *in, long long n, long long ws, int len, uint8_t *win,
                                               uint64_t *mbar) {
    const unsigned mis = (unsigned)((reinterpret_cast<uintptr_t>(in) + (uintptr_t)ws) & 15);
    const bool interior = ws >= 0 && ws + len <= n && (len & 15) == 0;
    if (interior && mis == 0) {
        if (threadIdx.x == 0) cx_bulk_load(win, in + ws, (unsigned)len, mbar);
        return true;
    }
    if (interior && ws + len + 16 <= n) {
        const uint4 *src = reinterpret_cast<const uint4 *>(in + ws - mis);
        uint4 *dst = reinterpret_cast<uint4 *>(win);
        const unsigned sel = 0x3210u + 0x1111u * (mis & 3);  // byte shift within a word pair
        const unsigned q = mis >> 2;
        for (int k = threadIdx.x; k < len / 16; k += CX_NT) {
            const uint4 a = __ldcs(src + k), b = __ldcs(src + k + 1);
            const unsigned w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint4 v;
            // q is the same for every thread: the branches do not diverge
            if (q == 0) v = make_uint4(__byte_perm(w[0], w[1], sel), __byte_perm(w[1], w[2], sel),
                                       __byte_perm(w[2], w[3], sel), __byte_perm(w[3], w[4], sel));
            else if (q == 1) v = make_uint4(__byte_perm(w[1], w[2], sel), __byte_perm(w[2], w[3], sel),
                                            __byte_perm(w[3], w[4], sel), __byte_perm(w[4], w[5], sel));
            else if (q == 2) v = make_uint4(__byte_perm(w[2], w[3], sel), __byte_perm(w[3], w[4], sel),
                                            __byte_perm(w[4], w[5], sel), __byte_perm(w[5], w[6], sel));
            else v = make_uint4(__byte_perm(w[3], w[4], sel), __byte_perm(w[4], w[5], sel),
                                __byte_perm(w[5], w[6], sel), __byte_perm(w[6], w[7], sel));
            dst[k] = v;
        }
        return false;
    }
    for (int k = threadIdx.x; k < len; k += CX_NT) {
        const long long g = ws + k;
        win[k] = g < 0 ? (uint8_t)'\n' : (g < n ? __ldcs(in + g) : (uint8_t)'\n');
    }
    return false;
}

// Staged tile output -> HBM: bytes until dst is 16-byte aligned, then 16-byte
// stores, each built from the two aligned 16-byte staging chunks it spans.
__device__ __forceinline__ void cx_store_out(uint8_t *dst, const uint8_t *src, int len) {
    const int head = min(len, (int)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
    if ((int)threadIdx.x < head) dst[threadIdx.x] = src[threadIdx.x];
    const int nvec = (len - head) >> 4;
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + head);
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);  // src is 16-byte aligned
    const unsigned sel = 0x3210u + 0x1111u * (head & 3), q = (unsigned)head >> 2;
    for (int k = threadIdx.x; k < nvec; k += CX_NT) {
        if (head == 0) {
            d4[k] = s4[k];
            continue;
        }
        const uint4 a = s4[k], b = s4[k + 1];  // bytes head + 16k .. head + 16k + 15
        const unsigned w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        uint4 v;
        if (q == 0) v = make_uint4(__byte_perm(w[0], w[1], sel), __byte_perm(w[1], w[2], sel),
                                   __byte_perm(w[2], w[3], sel), __byte_perm(w[3], w[4], sel));
        else if (q == 1) v = make_uint4(__byte_perm(w[1], w[2], sel), __byte_perm(w[2], w[3], sel),
                                        __byte_perm(w[3], w[4], sel), __byte_perm(w[4], w[5], sel));
        else if (q == 2) v = make_uint4(__byte_perm(w[2], w[3], sel), __byte_perm(w[3], w[4], sel),
                                        __byte_perm(w[4], w[5], sel), __byte_perm(w[5], w[6], sel));
        else v = make_uint4(__byte_perm(w[3], w[4], sel), __byte_perm(w[4], w[5], sel),
                            __byte_perm(w[5], w[6], sel), __byte_perm(w[6], w[7], sel));
        d4[k] = v;
    }
    for (int k = head + (nvec << 4) + threadIdx.x; k < len; k += CX_NT) dst[k] = src[k];
}

// record a rare line (returns false when the tile's list is full)
__device__ __forceinline__ void cx_rare(const CxSmem &S, int *n, int ls, int le, int kind, int lane, int local,
                                        int err, int glob) {
    const int r = atomicAdd(n, 1);
    if (r < CX_RARE) {
        CxRare &R = S.rare[r];
        R.ls = ls;
        R.le = le;
        R.kind = kind;
        R.lane = lane;
        R.local = local;
        R.err = err;
        R.aoff = 0;
        R.glob = glob;
        R.gs = 0;
        R.ll = -1;
    }
}

// clear the bits of window positions [a, b]
__device__ __forceinline__ void cx_clear_bits(unsigned *bm, int a, int b) {
    for (int w = a >> 5; a <= b && w <= (b >> 5); ++w) {
        unsigned m = 0xffffffffu;
        if (w == (a >> 5)) m &= 0xffffffffu << (a & 31);
        if (w == (b >> 5) && (b & 31) != 31) m &= (2u << (b & 31)) - 1u;
        atomicAnd(&bm[w], ~m);
    }
}

// last newline before position q (rbits: newlines only), or lo - 1 if none at or after lo
__device__ __forceinline__ int cx_prev_nl(const unsigned *rb, int q, int lo) {
    int w = q >> 5;
    unsigned m = rb[w] & ((1u << (q & 31)) - 1u);
    while (!m && w > (lo >> 5)) m = rb[--w];
    const int p = m ? (w << 5) + 31 - __clz(m) : lo - 1;
    return p < lo ? lo - 1 : p;
}

// PA: the parse runs the product automaton (one lookup per byte) instead of
// the DFA + cost-window transducer + code slots.
// SL: every phase on byte-exact slices (P2 and P4 entered by guess and
// repaired up to where the guessed and the true walks meet, P3 over lines
// bucket-sorted by event count, P6 by path entry guess + repair): balanced
// lanes, but a block barrier between phases (measured slower on C2 than the
// barrier-free line-lane pipeline; kept as a mode)
template <bool PA, bool SL>
__global__ void __launch_bounds__(CX_NT, (cx_ctas<PA, SL>())) compress_cx(Job job, Tables tb, CxTables ct) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int s_tmp[CX_NW];
    __shared__ unsigned long long s_tmp64[CX_NW];
    __shared__ long long s_tile;
    __shared__ int s_head_nl, s_last_nl, s_nrare, s_err_ord, s_r0, s_r2, s_nfe;
    __shared__ unsigned s_esc, s_skip, s_flag, s_inl, s_has_ll, s_cr;
    __shared__ unsigned long long s_pre_out, s_pre_lines;
    __shared__ __align__(8) uint64_t s_mbar;  // window bulk copies
    unsigned mbar_phase = 0;

    // tokenizer transducer (static: constant addresses); rows of CX_LUTS bytes so
    // the same byte in different states falls in different banks
    __shared__ __align__(16) uint8_t s_lut[8 * CX_LUTS];
    __shared__ __align__(16) uint8_t s_explen[256];
    __shared__ __align__(16) uint8_t s_exp0[256];  // first byte of each code's expansion (P4 re-parse)
    __shared__ __align__(16) uint8_t s_cmap[256];
    CxSmem S = cx_carve(smem, ct.o_t2, ct.o_codes, cx_o_tab<PA, SL>());
    S.lut = s_lut;
    S.explen = s_explen;
    {
        if (PA) {
            uint32_t *dst = reinterpret_cast<uint32_t *>(S.dfa);
            for (int k = threadIdx.x; k < ct.ns * ct.nc; k += CX_NT) dst[k] = ct.pa[k];
        } else {
            const uint4 *src = reinterpret_cast<const uint4 *>(ct.dfa);
            uint4 *dst = reinterpret_cast<uint4 *>(S.dfa);
            for (int k = threadIdx.x; k < cx_align16(ct.ns * ct.nc * 2) / 16; k += CX_NT) dst[k] = src[k];
            for (int k = threadIdx.x; k < ct.nw * CX_T2S; k += CX_NT) S.t2[k] = ct.t2[k];
            for (int k = threadIdx.x; k < ct.ns * CX_CODES; k += CX_NT) S.codes[k] = ct.codes[k];
        }
        for (int k = threadIdx.x; k < 256; k += CX_NT) s_cmap[k] = ct.cmap[k];
        for (int k = threadIdx.x; k < 256; k += CX_NT) S.explen[k] = k == '\n' ? 1 : tb.exp_len[k];
        for (int k = threadIdx.x; k < 256; k += CX_NT)
            s_exp0[k] = k == '\n' ? (uint8_t)'\n' : (tb.exp_len[k] ? tb.exp_flat[tb.exp_off[k]] : (uint8_t)k);
        for (int k = threadIdx.x; k < 8 * 256; k += CX_NT) {
            const unsigned st = k >> 8, b = k & 255;
            uint8_t e = tk_entry(st, b) & ~(TK_ENTER_BR | TK_ENTER_PCT);  // bits 5/6: line-end errors only
            if (b == '\n') {  // line end: back to TK_OUT0; flag an open bracket / a bad '%'
                e = 128u;
                if (job.preprocess && st == TK_IN) e |= 0x20u;
                if (job.preprocess && (st == TK_ERR || st >= TK_P1R)) e |= 0x40u;
            }
            S.lut[st * CX_LUTS + b] = e;
        }
    }
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    if (tid == 0) {
        s_esc = 0;
        cx_mbar_init(&s_mbar);
    }
    PhaseClock pc;
    pc.start();

    for (;;) {
        __syncthreads();
        if (tid == 0) {
            if (s_esc) atomicAdd(&job.ctl->escapes, (unsigned long long)s_esc);  // previous tile
            s_tile = (long long)atomicAdd(&job.ctl->ticket, 1ull);
            s_nrare = 0;
            s_err_ord = 0x7fffffff;
            s_r0 = s_r2 = 0x7fffffff;
            s_esc = s_skip = s_flag = s_has_ll = s_cr = 0;
        }
        __syncthreads();
        const long long t = s_tile;
        if (t >= job.n_tiles) break;
        const long long T0 = t * (long long)CX_TILE;
        const long long T1 = min(job.n, T0 + CX_TILE);
        const long long ws = T0 - CX_HEAD;
        const int tile_end = (int)(T1 - ws);
        const bool bulk = cx_load_window(job.in, job.n, ws, cx_align16(tile_end), S.win, &s_mbar);
        for (int k = tid; k < CX_WORDS; k += CX_NT) S.gbits[k] = S.fbits[k] = 0u;
        S.lane_b[tid] = 0;  // lane output adjustments (compaction gaps, arena lines)
        if (SL && tid < CX_HIST) S.hist[tid] = 0;  // P3 buckets
        if (lane == 0) S.njobs[tid >> 5] = 0;
        if (bulk) {
            cx_mbar_wait(&s_mbar, mbar_phase);
            mbar_phase ^= 1u;
        }
        __syncthreads();
        // the final tile closes a last line without '\n' with a virtual one
        int win_end = tile_end;
        if (T1 == job.n && S.win[tile_end - 1] != '\n') {
            win_end = tile_end + 1;
            if (tid == 0) S.win[tile_end] = '\n';
        }
        // ---- P1: newline bitmap of [0, win_end); without renumbering also
        // whether the window holds a '\r' (none: P2 has nothing to find) ----
        for (int wd = tid; wd < CX_WORDS; wd += CX_NT) {
            unsigned m = 0, cr = 0;
            const int b0 = wd * 32;
            if (b0 < win_end) {
                const unsigned *w4 = reinterpret_cast<const unsigned *>(S.win + b0);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const unsigned x = w4[k] ^ 0x0a0a0a0au;
                    const unsigned z = ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);
                    const unsigned nib = ((z >> 7) & 1u) | ((z >> 14) & 2u) | ((z >> 21) & 4u) | ((z >> 28) & 8u);
                    m |= nib << (4 * k);
                    if (!job.preprocess) {
                        const unsigned y = w4[k] ^ 0x0d0d0d0du;
                        unsigned zc = ~(((y & 0x7f7f7f7fu) + 0x7f7f7f7fu) | y | 0x7f7f7f7fu);
                        if (b0 + 4 * k + 4 > win_end)  // bytes past the window end are not data
                            zc &= b0 + 4 * k >= win_end ? 0u : 0xffffffffu >> (8 * (b0 + 4 * k + 4 - win_end));
                        cr |= zc;
                    }
                }
                if (b0 + 32 > win_end) m &= (1u << (win_end - b0)) - 1u;
            }
            S.rbits[wd] = m;
            if (cr) s_cr = 1;
        }
        __syncthreads();
        const int c0 = CX_HEAD + tid * CX_CC;
        const int c1 = min(c0 + CX_CC, win_end);
        int first_nl = 0x7fffffff, last_nl = -1;
        for (int wd = c0 >> 5; c0 < c1 && wd <= (c1 - 1) >> 5; ++wd) {
            unsigned m = S.rbits[wd];
            const int b0 = wd * 32;
            if (b0 < c0) m &= 0xffffffffu << (c0 - b0);
            if (b0 + 32 > c1) m &= (1u << (c1 - b0)) - 1u;
            if (m) {
                if (first_nl == 0x7fffffff) first_nl = b0 + __ffs(m) - 1;
                last_nl = b0 + 31 - __clz(m);
            }
        }
        if (tid < 32) {
            // last '\n' before the tile (in the staged head); -1: none
            int best = -1;
            for (int wd = (CX_HEAD >> 5) - 1 - lane; wd >= 0; wd -= 32) {
                const unsigned m = S.rbits[wd];
                best = max(best, m ? wd * 32 + 31 - __clz(m) : -1);
            }
            best = __reduce_max_sync(0xffffffffu, best);
            if (lane == 0) s_head_nl = best;
        }
        const int Lx = cx_block_scan_mm<true>(last_nl, s_tmp, true, -1);  // last '\n' before c0
        const int Rx = cx_block_suffix_min(first_nl, s_tmp);             // first '\n' at/after c0
        if (tid == CX_NT - 1) s_last_nl = max(Lx, last_nl);              // the tile's last '\n'
        const int head_nl = s_head_nl;
        // cut before lane tid: the newline nearest to c0 (lane 0: the head newline)
        int cut;
        {
            const int L = Lx >= 0 ? Lx : head_nl;
            if (tid == 0 || Rx == 0x7fffffff) cut = L;
            else if (L < 0) cut = Rx;
            else cut = (Rx - c0 < c0 - L) ? Rx : L;
        }
        S.lane_a[tid] = cut;
        __syncthreads();
        if (tid == 0 && job.tl) job.tl[t] = s_last_nl >= CX_HEAD ? ws + s_last_nl : -1;
        pc.mark(job, 0);  // load, newline bitmap, lane cuts
        // lane range (cut, end]; end = next lane's cut (last lane: the tile's last '\n')
        const int end = tid + 1 < CX_NT ? S.lane_a[tid + 1] : s_last_nl;
        // a line that starts before the window is owned by the lane whose
        // range holds its '\n' (the tile's first newline): a "global" line
        const bool glob = cut < 0 && end >= CX_HEAD;
        int start = cut + 1;
        int gpos = -1;
        if (end < CX_HEAD) start = end + 1;  // no line of this tile
        if (glob) {
            gpos = cx_next(S.rbits, CX_HEAD);
            start = gpos;
        }
        const int first = glob ? gpos + 1 : start;  // first byte of the first in-window line
        S.lane_f[tid] = first | (glob ? 1 << 30 : 0);
        if (kPhases && job.timing == 2) {  // debug: lane range statistics
            const int len = max(0, end - start + 1);
            const int wmax = __reduce_max_sync(0xffffffffu, len);
            const int wsum = __reduce_add_sync(0xffffffffu, len);
            if (lane == 0) {
                atomicAdd(&job.ctl->phase[0], (unsigned long long)wmax);
                atomicAdd(&job.ctl->phase[1], (unsigned long long)wsum);
                atomicAdd(&job.ctl->phase[2], 1ull);
            }
        }

        // P2 -> P3 -> P4 run per warp without block barriers: a lane only
        // touches its own range (bitmap words shared with a neighbour are
        // updated atomically).  Rare lines are turned into escape-only filler
        // by their owner right away (the parse prices a filler byte at exactly
        // 2); their general-routine work waits until after the parse.
        int sub = 0;  // parse cost of the lane's filler bytes (2 each)
        auto filler = [&](int a, int b) {  // window positions [a, b]
            for (int j = a; j <= b; ++j) {
                S.win[j] = 0x01;
                cx_set(S.fbits, j);
            }
            sub += 2 * (b - a + 1);
        };
        // ---- P2: tokenizer; CR / tokenize errors; ring-token bits ----
        // LUT entry: bits 0-2 next state, 3 ring token, 4 '\r', 7 line end;
        // a line end's bits 5/6 flag an unclosed '[' / a bad '%' (preprocess).
        // The fast walk only ORs the flags together; a lane whose range holds
        // a CR or a tokenize error walks it again with the per-line handling.
        // Ring-token bits gather in a register per 32-byte bitmap word.
        int nlines = glob ? 1 : 0;
        // Long line-lane ranges (long lines): P2 and P4 walk byte-exact slices
        // instead (they pay a warm-up of up to CX_WARM bytes per lane, worth
        // it only when a line-lane range is much longer than a slice).  Every
        // warp derives the same decision from lane_a.
        bool long_ranges = false;
        bool p2_regular = true;  // P2 ended with the per-line walks (no final block barrier)
        if (ct.p4x) {
            int mx = 0;
            for (int k = lane; k < CX_NT; k += 32)
                mx = max(mx, (k + 1 < CX_NT ? S.lane_a[k + 1] : s_last_nl) - S.lane_a[k]);
            long_ranges = __reduce_max_sync(0xffffffffu, mx) > CX_XLONG;
        }
        {
            const uint8_t *__restrict__ lut = S.lut;
            const unsigned *__restrict__ w32 = reinterpret_cast<const unsigned *>(S.win);
            unsigned st = TK_OUT0, crs = 0, rmask = 0, flags = 0;
            int ls = first;
            auto step_fast = [&](int p, unsigned b) {
                const unsigned e = lut[st * CX_LUTS + b];
                rmask |= ((e >> 3) & 1u) << (p & 31);
                flags |= e;
                nlines += e >> 7;
                st = e & 7u;
            };
            // one tokenizer step at window position p (byte b), per-line errors
            auto step = [&](int p, unsigned b) {
                const unsigned e = lut[st * CX_LUTS + b];
                rmask |= ((e >> 3) & 1u) << (p & 31);
                const bool nl = e & 128u;
                if (nl && ((e & 0x60u) | (crs & TK_CR))) {
                    const int k = (crs & TK_CR) ? E_CR : (e & 0x40u) ? E_PERCENT : E_BRACKET;
                    if (k == E_CR || !job.lenient) {
                        // dropped (lenient CR) or a strict error: filler
                        cx_rare(S, &s_nrare, ls, p, job.lenient ? RK_DROP : RK_STRICT, tid, nlines, k, 0);
                        filler(ls, p);
                    } else {
                        atomicAdd(&s_flag, 1u);  // lenient: the raw line is compressed
                    }
                    if (job.preprocess) {  // P3 does not renumber it: drop its ring-token bits
                        cx_clear_bits(S.gbits, ls, p);
                        rmask &= ls > (p & ~31) ? (1u << (ls & 31)) - 1u : 0u;  // this word's, not flushed yet
                    }
                }
                nlines += nl;
                ls = nl ? p + 1 : ls;
                crs = nl ? 0u : (crs | e);
                st = e & 7u;
            };
            auto flush = [&](int p) {  // ring bits of the bitmap word holding p
                if (rmask && job.preprocess) atomicOr(&S.gbits[p >> 5], rmask);
                rmask = 0;
            };
            auto walk = [&](auto &&stepfn) {
                int p = first;
                // bytes up to a word boundary, then whole words, then the tail
                const int w0 = (first + 3) & ~3, w1 = (end + 1) & ~3;
                if (w0 < w1) {
                    for (; p < w0; ++p) stepfn(p, S.win[p]);
                    if (p > first && (p & 31) == 0) flush(p - 1);
                    unsigned cur = w32[p >> 2];
                    for (; p < w1; p += 4) {
                        const unsigned nxt = w32[(p >> 2) + 1];  // prefetch (the window has slack after it)
                        stepfn(p, cur & 0xffu);
                        stepfn(p + 1, (cur >> 8) & 0xffu);
                        stepfn(p + 2, (cur >> 16) & 0xffu);
                        stepfn(p + 3, cur >> 24);
                        if (((p + 3) & 31) == 31) flush(p);
                        cur = nxt;
                    }
                }
                for (; p <= end; ++p) {
                    stepfn(p, S.win[p]);
                    if ((p & 31) == 31) flush(p);
                }
                flush(end);
            };
            // the fast walk: whole words of 4 bytes; per word the four LUT
            // entries are combined once for the flags, the ring-token nibble
            // and the newline count
            auto walk_fast_range = [&](const int first, const int end) {
                int p = first;
                const int w0 = (first + 3) & ~3, w1 = (end + 1) & ~3;
                if (w0 < w1) {
                    for (; p < w0; ++p) step_fast(p, S.win[p]);
                    if (p > first && (p & 31) == 0) flush(p - 1);
                    unsigned cur = w32[p >> 2];
                    for (; p < w1; p += 4) {
                        const unsigned nxt = w32[(p >> 2) + 1];  // prefetch (the window has slack after it)
                        const unsigned e0 = lut[st * CX_LUTS + (cur & 0xffu)];
                        const unsigned e1 = lut[(e0 & 7u) * CX_LUTS + ((cur >> 8) & 0xffu)];
                        const unsigned e2 = lut[(e1 & 7u) * CX_LUTS + ((cur >> 16) & 0xffu)];
                        const unsigned e3 = lut[(e2 & 7u) * CX_LUTS + (cur >> 24)];
                        st = e3 & 7u;
                        const unsigned ew = e0 | (e1 << 8) | (e2 << 16) | (e3 << 24);
                        flags |= ew;
                        nlines += __popc(ew & 0x80808080u);
                        const unsigned rn = (((ew >> 3) & 0x01010101u) * 0x01020408u) >> 24;  // ring bits, byte k -> bit k
                        rmask |= (rn & 15u) << (p & 31);
                        if (((p + 3) & 31) == 31) flush(p);
                        cur = nxt;
                    }
                }
                for (; p <= end; ++p) {
                    step_fast(p, S.win[p]);
                    if ((p & 31) == 31) flush(p);
                }
                flush(end);
                flags |= (flags >> 8) | (flags >> 16) | (flags >> 24);
            };
            bool &regular = p2_regular;
            if (SL || long_ranges) {
                // ---- P2 on byte-exact slices ----
                // A slice is entered in the tokenizer state a newline leaves
                // (found within CX_WARM bytes to its left, or the region start),
                // else in the state of a warm-up from TK_OUT0; such a guess is
                // checked against the left neighbour's exit state and the slice
                // walked again (its ring bits cleared first) until none
                // differs.  A CR or a tokenize error anywhere sends every
                // line-lane through the per-line walk below instead.
                nlines += cx_popc_range(S.rbits, first, end);  // the bitmap holds only newlines yet
                if (first <= end) atomicMin(&s_r2, first);
                if (start <= end) atomicMin(&s_r0, start);  // P4 / P6 slices
                __syncthreads();
                const int R0 = s_r2, R1 = s_last_nl;
                const int sz = R1 >= R0 ? (R1 - R0 + CX_NT) / CX_NT : 0;
                const int s0 = R0 + tid * sz, e0 = min(R1, s0 + sz - 1);
                bool spec = false;
                unsigned spec_state = TK_OUT0;
                const int nl_keep = nlines;
                flags = 0;
                st = TK_OUT0;
                if (sz > 0 && s0 <= e0) {
                    if (SL && s0 > R0 && S.win[s0 - 1] != '\n') {
                        spec = true;  // guess TK_OUT0, repaired below up to where the walks meet
                    } else if (s0 > R0 && S.win[s0 - 1] != '\n') {
                        const int lim = max(R0, s0 - CX_WARM);
                        int p = s0 - 1;
                        while (p > lim && S.win[p] != '\n') --p;
                        if (S.win[p] == '\n') ++p;
                        else spec = p > R0;  // R0 is a line start
                        for (; p < s0; ++p) st = lut[st * CX_LUTS + S.win[p]] & 7u;
                        spec_state = st;
                    }
                    walk_fast_range(s0, e0);
                }
                S.lane_c[tid] = (int)st;  // exit state (read by the right neighbour)
                __syncthreads();
                for (;;) {
                    bool need = false;
                    unsigned truth = 0;
                    if (spec) {
                        truth = (unsigned)S.lane_c[tid - 1];
                        need = truth != spec_state;
                    }
                    if (!__syncthreads_or(need)) break;
                    if (SL && need) {
                        // walk again from the true entry state next to the guessed
                        // one until the two states meet; fix the ring bits of the
                        // bytes where they differ
                        unsigned so = spec_state, sn = truth;
                        int p = s0;
                        for (; p <= e0; ++p) {
                            const unsigned b = S.win[p];
                            const unsigned eo = lut[so * CX_LUTS + b], en = lut[sn * CX_LUTS + b];
                            so = eo & 7u;
                            sn = en & 7u;
                            flags |= en;
                            if (((eo ^ en) & 8u) && job.preprocess) {
                                if (en & 8u) atomicOr(&S.gbits[p >> 5], 1u << (p & 31));
                                else atomicAnd(&S.gbits[p >> 5], ~(1u << (p & 31)));
                            }
                            if (so == sn) break;
                        }
                        spec_state = truth;
                        if (p > e0) S.lane_c[tid] = (int)sn;
                    } else if (need) {
                        cx_clear_bits(S.gbits, s0, e0);
                        st = truth;
                        flags = 0;
                        walk_fast_range(s0, e0);
                        spec_state = truth;
                        S.lane_c[tid] = (int)st;
                    }
                    __syncthreads();
                }
                nlines = nl_keep;
                regular = __syncthreads_or((flags & 0x70u) != 0u) != 0;
                if (regular) {  // rare: per-line walks over the line-lanes (ring bits are set again, idempotently)
                    nlines = glob ? 1 : 0;
                    st = TK_OUT0;
                    flags = 0;
                    rmask = 0;
                }
            }
            if (regular && first <= end && !job.preprocess && !s_cr) {
                // without renumbering the tokenizer only looks for '\r' (line
                // ends flag no errors), and the window has none: count lines
                nlines += cx_popc_range(S.rbits, first, end);
            } else if (regular && first <= end) {
                walk_fast_range(first, end);
                if (flags & 0x70u) {  // a CR or a tokenize error in the range (rare)
                    nlines = glob ? 1 : 0;
                    st = TK_OUT0;
                    walk(step);
                }
            }
        }
        if (glob) {
            cx_rare(S, &s_nrare, gpos, gpos, RK_ARENA, tid, 0, 0, 1);
            filler(gpos, gpos);
        }
        pc.mark(job, 1);  // warp 0: tokenizer

        // ---- P3: ring pairing + colouring (smiles.py:140-213) ----
        // One straight-line step per event (ring token or '\n') so the lanes
        // of a warp stay converged: open rings in 4 register slots (id,
        // position), colours 0-3 from their last close positions (a ring
        // takes the smallest colour not closed inside it).  Lines beyond that
        // (5+ open rings, colour >= 4, a colour digit that is not an identity
        // code) go to the general routine.
        if (job.preprocess) {
            // Ring-token events only (gbits); a line's bounds come from the
            // newline bitmap when its first event arrives, and lines without
            // events cost nothing.  P2 already turned its error lines into
            // filler or raw lines and dropped their ring bits.
            const uint8_t *win = S.win;
            int ls = -1, le = -1;  // the line being renumbered: [ls, le], le its '\n'
            unsigned oid = 0xffffffffu;  // 4 slots: open ring id per byte, 0xff = free
            int op0 = 0, op1 = 0, op2 = 0, op3 = 0;
            int lc0 = -1, lc1 = -1, lc2 = -1, lc3 = -1;
            unsigned n_pct = 0;
            bool fail = false;
            auto finish = [&]() {  // special handling at the line's end (smiles.py:151-159, 196-202)
                if (!((fail | (oid != 0xffffffffu) | (n_pct != 0)) && (!kPhases || job.timing < 3))) return;
                const int q = le;
                // the line-lane owning the line (P3 slices: not this lane) and the
                // line's index in it
                int own = tid, local;
                if (SL) {
                    int lo = 0, hi = CX_NT - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (S.lane_a[mid] < ls) lo = mid;
                        else hi = mid - 1;
                    }
                    own = lo;
                    const int f = S.lane_f[own], f0 = f & ((1 << 30) - 1);
                    local = (f >> 30) + (ls > f0 ? cx_popc_range(S.rbits, f0, ls - 1) : 0);
                } else {
                    local = (glob ? 1 : 0) + (ls > first ? cx_popc_range(S.rbits, first, ls - 1) : 0);
                }
                auto fill = [&](int a, int b) {
                    if (SL) {
                        for (int j = a; j <= b; ++j) {
                            S.win[j] = 0x01;
                            cx_set(S.fbits, j);
                        }
                        atomicAdd(&S.lane_b[own], -2 * (b - a + 1));
                    } else {
                        filler(a, b);
                    }
                };
                if (fail) {
                    cx_rare(S, &s_nrare, ls, q, RK_ARENA, own, local, 0, 0);
                    fill(ls, q);
                } else if (oid != 0xffffffffu) {
                    // ring ids left open (smiles.py:151-159)
                    if (job.lenient) {
                        for (int j = ls; j < q; ++j) S.win[j] = job.in[ws + j];
                        atomicAdd(&s_flag, 1u);
                    } else {
                        cx_rare(S, &s_nrare, ls, q, RK_STRICT, own, local, E_UNPAIRED, 0);
                        fill(ls, q);
                    }
                } else {
                    // '%nn' ring tokens: compacted below by a whole warp (PA: one
                    // job list per CTA, spread over the warps after P3)
                    const int jn = atomicAdd(&S.njobs[SL ? 0 : tid >> 5], 1);
                    if (jn < (SL ? CX_NW * CX_JOBS : CX_JOBS)) {
                        S.jobs[SL ? jn : (tid >> 5) * CX_JOBS + jn] = make_int4(ls, q, own, local);
                    } else {
                        cx_rare(S, &s_nrare, ls, q, RK_ARENA, own, local, 0, 0);
                        fill(ls, q);
                    }
                }
            };
            // PA: byte-exact slices of the tile's lines: a lane renumbers the
            // lines whose first ring event lies in its slice (to their end), so
            // every lane walks about the same number of events.  The lines of
            // other line-lanes must be through P2 (ring bits final) first.
            int p3a = first, p3b = end, p3lo = first;
            if (SL) {
                if (p2_regular) __syncthreads();  // P2's per-line walks of every warp done (else P2 ended on a barrier)
                const int R0 = s_r2, R1 = s_last_nl;
                const int sz = R1 >= R0 ? (R1 - R0 + CX_NT) / CX_NT : 0;
                p3a = R0 + tid * sz;
                p3b = sz > 0 ? min(R1, p3a + sz - 1) : p3a - 1;
                p3lo = R0;
            }
            // one ring event of the current line (smiles.py:140-180 restated
            // over 4 open-ring slots and the per-colour last-close positions)
            auto ring_event = [&](int q) {
                ZS_ASSERT(q >= 0 && q < le && q < CX_WIN);
                const unsigned c = win[q];
                ZS_ASSERT(c == '%' || (c >= '0' && c <= '9'));
                const bool pct = c == '%';
                const unsigned rid = pct ? (win[q + 1] - '0') * 10u + (win[q + 2] - '0') : c - '0';
                n_pct += pct;
                const unsigned v0 = oid & 0xffu, v1 = (oid >> 8) & 0xffu, v2 = (oid >> 16) & 0xffu, v3 = oid >> 24;
                const int slot = v0 == rid ? 0 : v1 == rid ? 1 : v2 == rid ? 2 : v3 == rid ? 3 : -1;
                if (slot < 0) {
                    const int fs = v0 == 0xffu ? 0 : v1 == 0xffu ? 1 : v2 == 0xffu ? 2 : v3 == 0xffu ? 3 : -1;
                    fail |= fs < 0;
                    op0 = fs == 0 ? q : op0;
                    op1 = fs == 1 ? q : op1;
                    op2 = fs == 2 ? q : op2;
                    op3 = fs == 3 ? q : op3;
                    oid = fs < 0 ? oid : (oid & ~(0xffu << (8 * fs))) | (rid << (8 * fs));
                } else {
                    const int o = slot == 0 ? op0 : slot == 1 ? op1 : slot == 2 ? op2 : op3;
                    oid |= 0xffu << (8 * slot);
                    const int col = lc0 <= o ? 0 : lc1 <= o ? 1 : lc2 <= o ? 2 : lc3 <= o ? 3 : 4;
                    const bool ok = col < 4 && S.explen['0' + col] != 0;
                    fail |= !ok;
                    if (ok && !fail) {
                        lc0 = col == 0 ? q : lc0;
                        lc1 = col == 1 ? q : lc1;
                        lc2 = col == 2 ? q : lc2;
                        lc3 = col == 3 ? q : lc3;
                        S.win[o + (win[o] == '%')] = (uint8_t)('0' + col);
                        S.win[q + pct] = (uint8_t)('0' + col);
                    }
                }
            };
            if (SL && (!kPhases || job.timing != 4)) {
                // Line-first ring events of the slice (an event whose previous
                // newline-or-event mark is a newline): with X = newlines |
                // events, ~X + (newlines << 1) carries each newline's bit up to
                // the next mark; the marks it reaches that are events start a
                // line.  Each line is renumbered by one lane, event by event;
                // a tile has ~1.7 such lines per lane and their event counts
                // vary, so the lines are bucket-sorted by event count
                // (descending) and lane t takes sorted lines t, t + CX_NT, ...:
                // the lanes of a warp walk lines of about the same length.
                unsigned nfe = 0;
                const int w0 = p3a >> 5, w1 = p3b >> 5;
                unsigned cin = 1;  // the last mark before word w0 is a newline (or the region start)
                if (p3a <= p3b) {
                    for (int v = w0 - 1; v >= (p3lo >> 5); --v) {
                        unsigned xm = S.rbits[v] | S.gbits[v];
                        if (v == (p3lo >> 5)) xm &= 0xffffffffu << (p3lo & 31);
                        if (xm) {
                            cin = (S.rbits[v] >> (31 - __clz(xm))) & 1u;
                            break;
                        }
                    }
                }
                unsigned fe_w[4];  // line-first event bits of the slice's words (<= 4 words)
                #pragma unroll
                for (int k = 0; k < 4; ++k) {
                    fe_w[k] = 0;
                    const int w = w0 + k;
                    if (p3a <= p3b && w <= w1) {
                        const unsigned N = S.rbits[w], E = S.gbits[w], X = N | E;
                        const unsigned fe = ((~X) + (N << 1) + cin) & E;
                        unsigned m = 0xffffffffu;
                        if (w == w0) m &= 0xffffffffu << (p3a & 31);
                        if (w == w1 && (p3b & 31) != 31) m &= (2u << (p3b & 31)) - 1u;
                        fe_w[k] = fe & m;
                        nfe += __popc(fe_w[k]);
                        cin = X ? (N >> (31 - __clz(X))) & 1u : cin;
                    }
                }
                // bucket-sort the lines by (about) their event count,
                // descending: the events between a line-first event and the
                // next one in the slice (the slice's last line: to the slice
                // end) -- only the order depends on it
                auto keys = [&](auto &&fn) {
                    int prev = -1;
                    #pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        unsigned m = fe_w[k];
                        while (m) {
                            const int q0 = ((w0 + k) << 5) + __ffs(m) - 1;
                            m &= m - 1u;
                            if (prev >= 0) fn(prev, cx_popc_range(S.gbits, prev, q0 - 1));
                            prev = q0;
                        }
                    }
                    if (prev >= 0) fn(prev, cx_popc_range(S.gbits, prev, p3b));
                };
                int nfe_all;
                {
                    keys([&](int, int ne) { atomicAdd(&S.hist[CX_HIST - 1 - min(ne, CX_HIST - 1)], 1); });
                    __syncthreads();
                    if (tid < 32) {  // exclusive scan of the 64 buckets
                        const int h0 = S.hist[2 * lane], h1 = S.hist[2 * lane + 1];
                        int x = h0 + h1;
                        #pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int y = __shfl_up_sync(0xffffffffu, x, o);
                            if (lane >= o) x += y;
                        }
                        S.hist[2 * lane] = x - h0 - h1;
                        S.hist[2 * lane + 1] = x - h1;
                        if (lane == 31) s_nfe = x;
                    }
                    __syncthreads();
                    nfe_all = s_nfe;
                }
                const bool pooled = nfe_all <= CX_POOL;
                if (pooled)
                    keys([&](int q0, int ne) {
                        const int at = atomicAdd(&S.hist[CX_HIST - 1 - min(ne, CX_HIST - 1)], 1);
                        ZS_ASSERT(at >= 0 && at < nfe_all);
                        S.pool[at] = (uint32_t)q0;
                    });
                __syncthreads();
                if (pooled) {
                    for (int i = tid; i < nfe_all; i += CX_NT) {
                        const int q0 = (int)S.pool[i];
                        le = cx_next(S.rbits, q0);
                        ZS_ASSERT(q0 >= p3lo && q0 < le && le <= s_last_nl && S.win[le] == '\n');
                        ls = cx_prev_nl(S.rbits, q0, p3lo) + 1;
                        oid = 0xffffffffu;
                        lc0 = lc1 = lc2 = lc3 = -1;
                        n_pct = 0;
                        fail = false;
                        int ew = q0 >> 5;
                        const int ew_last = le >> 5;
                        unsigned em = S.gbits[ew] & (0xffffffffu << (q0 & 31));
                        for (;;) {
                            while (!em && ew < ew_last) em = S.gbits[++ew];
                            const int q = em ? (ew << 5) + __ffs(em) - 1 : 0x7fffffff;
                            if (q > le) break;
                            em &= em - 1u;
                            ring_event(q);
                        }
                        finish();
                    }
                    le = -1;
                } else if (p3a <= p3b) {
                    // (more line-first events than the queue holds: this lane
                    // walks the lines that start in its slice itself)
                    #pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        unsigned m = fe_w[k];
                        while (m) {
                            const int q0 = ((w0 + k) << 5) + __ffs(m) - 1;
                            m &= m - 1u;
                            le = cx_next(S.rbits, q0);
                            ls = cx_prev_nl(S.rbits, q0, p3lo) + 1;
                            oid = 0xffffffffu;
                            lc0 = lc1 = lc2 = lc3 = -1;
                            n_pct = 0;
                            fail = false;
                            int ew = q0 >> 5;
                            unsigned em = S.gbits[ew] & (0xffffffffu << (q0 & 31));
                            for (;;) {
                                while (!em && ew < (le >> 5)) em = S.gbits[++ew];
                                if (!em) break;
                                const int qq = (ew << 5) + __ffs(em) - 1;
                                if (qq > le) break;
                                em &= em - 1u;
                                ring_event(qq);
                            }
                            finish();
                        }
                    }
                    le = -1;
                }
            }
            if (!SL && first <= end && (!kPhases || job.timing != 4)) {
                int ew = first >> 5;
                const int ew_last = end >> 5;
                unsigned em = S.gbits[ew] & (0xffffffffu << (first & 31));
                for (;;) {
                    while (!em && ew < ew_last) em = S.gbits[++ew];
                    if (!em) break;
                    const int q = (ew << 5) + __ffs(em) - 1;
                    if (q > end) break;
                    em &= em - 1u;
                    if (q > le) {  // the first event of a new line
                        if (le >= 0) finish();
                        le = cx_next(S.rbits, q);
                        ls = cx_prev_nl(S.rbits, q, first) + 1;
                        oid = 0xffffffffu;
                        lc0 = lc1 = lc2 = lc3 = -1;
                        n_pct = 0;
                        fail = false;
                    }
                    const unsigned c = win[q];
                    const bool pct = c == '%';
                    const unsigned rid = pct ? (win[q + 1] - '0') * 10u + (win[q + 2] - '0') : c - '0';
                    n_pct += pct;
                    const unsigned v0 = oid & 0xffu, v1 = (oid >> 8) & 0xffu, v2 = (oid >> 16) & 0xffu,
                                   v3 = oid >> 24;
                    const int slot = v0 == rid ? 0 : v1 == rid ? 1 : v2 == rid ? 2 : v3 == rid ? 3 : -1;
                    if (slot < 0) {
                        // opens a ring in the first free slot
                        const int fs = v0 == 0xffu ? 0 : v1 == 0xffu ? 1 : v2 == 0xffu ? 2 : v3 == 0xffu ? 3 : -1;
                        fail |= fs < 0;
                        op0 = fs == 0 ? q : op0;
                        op1 = fs == 1 ? q : op1;
                        op2 = fs == 2 ? q : op2;
                        op3 = fs == 3 ? q : op3;
                        oid = fs < 0 ? oid : (oid & ~(0xffu << (8 * fs))) | (rid << (8 * fs));
                    } else {
                        // closes the ring opened at o: the smallest colour not
                        // closed inside (o, q)
                        const int o = slot == 0 ? op0 : slot == 1 ? op1 : slot == 2 ? op2 : op3;
                        oid |= 0xffu << (8 * slot);
                        const int col = lc0 <= o ? 0 : lc1 <= o ? 1 : lc2 <= o ? 2 : lc3 <= o ? 3 : 4;
                        const bool ok = col < 4 && S.explen['0' + col] != 0;
                        fail |= !ok;
                        if (ok && !fail) {
                            lc0 = col == 0 ? q : lc0;
                            lc1 = col == 1 ? q : lc1;
                            lc2 = col == 2 ? q : lc2;
                            lc3 = col == 3 ? q : lc3;
                            S.win[o + (win[o] == '%')] = (uint8_t)('0' + col);
                            S.win[q + pct] = (uint8_t)('0' + col);
                        }
                    }
                }
                if (le >= 0) finish();
            }
            // ---- '%nn' compaction, the whole warp per line: a ring '%nn'
            // token keeps only its colour digit (at '%' + 1); the line's bytes
            // shift left and the freed bytes before its '\n' become escape
            // filler.  A byte that could be escaped in a shifted line (its
            // literal is re-read from HBM by position) sends the line to the
            // general routine instead.
            if (SL) __syncthreads();
            else __syncwarp();
            const int nj = SL ? min(S.njobs[0], CX_NW * CX_JOBS) : min(S.njobs[tid >> 5], CX_JOBS);
            for (int j = SL ? tid >> 5 : 0; j < nj; j += SL ? CX_NW : 1) {
                const int4 J = S.jobs[SL ? j : (tid >> 5) * CX_JOBS + j];
                const int jls = J.x, jq = J.y;
                int kept = 0;
                unsigned carry = 0;  // ring-'%' flags of the previous chunk's last two bytes
                bool risk = false;
                for (int c0b = jls; c0b < jq; c0b += 32) {
                    const int r = c0b + lane;
                    const bool valid = r < jq;
                    const unsigned b = valid ? S.win[r] : 0u;
                    const bool isp = valid && b == '%' && cx_bit(S.gbits, r);
                    const unsigned M = __ballot_sync(0xffffffffu, isp);
                    const unsigned M2 = (M << 2) | carry;
                    const bool drop = isp || ((M2 >> lane) & 1u);
                    const bool keep = valid && !drop;
                    risk |= keep && (b >= 0x80u || !S.explen[b]);
                    const unsigned K = __ballot_sync(0xffffffffu, keep);
                    __syncwarp();
                    if (keep) S.win[jls + kept + __popc(K & ((1u << lane) - 1u))] = (uint8_t)b;
                    __syncwarp();
                    kept += __popc(K);
                    carry = M >> 30;
                }
                const int gap0 = jls + kept;
                if (__any_sync(0xffffffffu, risk)) {
                    if (lane == 0) cx_rare(S, &s_nrare, jls, jq, RK_ARENA, J.z, J.w, 0, 0);
                    for (int r = jls + lane; r <= jq; r += 32) {
                        S.win[r] = 0x01;
                        cx_set(S.fbits, r);
                    }
                    if (lane == 0) atomicAdd(&S.lane_b[J.z], -2 * (jq - jls + 1));
                } else {
                    for (int r = gap0 + lane; r < jq; r += 32) {
                        S.win[r] = 0x01;  // escape-only filler
                        cx_set(S.fbits, r);
                    }
                    if (lane == 0) atomicAdd(&S.lane_b[J.z], -2 * (jq - gap0));
                }
            }
        }

        pc.mark(job, 2);  // warp 0: pairing
        // ---- P4: min-cost parse, right to left ----
        // Branch-free: code slot 0 of every state is 0x20, so an escape
        // decision writes the escape byte (its literal is re-read from HBM by
        // the emit).  Whole 4-byte words inside a range are read and written
        // with one 32-bit access each (the words at the range ends bytewise:
        // they are shared with the neighbouring lanes).
        //
        // Byte-exact slices (ct.p4x): the tile's owned bytes [R0, R1] are cut
        // into CX_NT equal slices, so every lane parses the same number of
        // bytes whatever the line lengths.  A slice's right end is entered
        // with the state a newline leaves (exact) or, when no newline lies
        // within CX_WARM bytes to its right, with the state of a K-byte
        // warm-up from a virtual line end (the (DFA state, cost window) pair
        // resynchronises within a few bytes).  After the parse every slice
        // publishes its exit state; a speculative entry that differs from
        // its right neighbour's exit is parsed again from the true state
        // (bytes rebuilt from the decisions), until none differs.  The
        // bias-corrected cost of each piece of a slice goes to the line-lane
        // that owns those bytes (lane_b), so P5 / P6 stay per line-lane.
        unsigned acc = 0;
        bool p4_exact = false;
        {
            const uint16_t *__restrict__ dfa = S.dfa;
            const uint16_t *__restrict__ t2 = S.t2;
            // transducer DFAs keep their code slots at a compile-time offset
            const uint8_t *__restrict__ codes = ct.kw ? S.codes : smem + CX_O_CODES;
            const int nc = ct.nc;
            uint8_t *win = S.win;
            unsigned st = 0, wi = 0;
            const unsigned pa_base = (unsigned)__cvta_generic_to_shared(S.dfa);
            auto step = [&](unsigned b) -> unsigned {
                if (PA) {  // st: the state's row offset in bytes (SL: no costs, P6 counts the output)
                    const unsigned e = cx_lw(pa_base + st + s_cmap[b]);
                    st = e & 0xffffu;
                    if (!SL) acc += (e >> 24) & 7u;
                    return ((e >> 16) & 0xffu) | (b & (unsigned)((int)e >> 31));
                }
                const unsigned e = dfa[st * nc + s_cmap[b]];
                st = e & 0xffu;
                const unsigned x = t2[wi * CX_T2S + (e >> 8)];
                wi = x & 0x1ffu;
                acc += x >> 13;
                const unsigned L = (x >> 9) & 15u;
                return L == 1 ? b : codes[st * CX_CODES + L];  // length 1: the identity code is the byte
            };
            // parse [lo, hi] right to left, decisions in place
            auto parse_range = [&](int lo, int hi) {
                if (lo > hi) return;
                const int lo_w = (lo + 3) & ~3;  // first whole word inside the range
                const int hi_w = (hi + 1) & ~3;  // end of the last whole word (exclusive)
                int i = hi;
                for (; i >= max(hi_w, lo); --i) win[i] = (uint8_t)step(win[i]);
                if (lo_w < hi_w) {
                    unsigned *w32 = reinterpret_cast<unsigned *>(win);
                    unsigned cur = w32[(hi_w >> 2) - 1];
                    for (int wd = (hi_w >> 2) - 1; wd >= (lo_w >> 2); --wd) {
                        const unsigned nxt = w32[wd - 1];  // prefetch (wd - 1 >= -1 words: slack before the window)
                        unsigned d = step(cur >> 24) << 24;
                        d |= step((cur >> 16) & 0xffu) << 16;
                        d |= step((cur >> 8) & 0xffu) << 8;
                        d |= step(cur & 0xffu);
                        w32[wd] = d;
                        cur = nxt;
                    }
                    i = lo_w - 1;
                }
                for (; i >= lo; --i) win[i] = (uint8_t)step(win[i]);
            };
            // the product-automaton parse always runs byte-exact slices (no
            // warm-up, so they pay on short lines too)
            p4_exact = SL || (long_ranges && (PA || !ct.kw));
            if (!PA && ct.kw) {
                // Key-window parse (dp_fast restated for W = 16): key(j) =
                // cost[j] * 16 - j, kept in a 32-entry ring per thread; the
                // cheapest candidate, longer on ties (numba_impl.py:50), wins.
                // A '\n' closes the line to its right (its cost + 1 for the
                // separator) and starts the next one with key = -position.
                const uint32_t *__restrict__ dfa32 = reinterpret_cast<const uint32_t *>(S.dfa);
                const int ncol = ct.nc >> 1;
                unsigned *ring = reinterpret_cast<unsigned *>(smem + ct.o_ring) + tid * CX_KW_RING;
                constexpr int INF = 0x3fffffff;
                // the range normally ends with its last line's '\n'; a rare
                // line's filler replaces that '\n', so the walk starts from a
                // virtual line end past the range (no separator byte of its own)
                int k1 = -(end + 1);  // key(i + 1)
                for (int L = 1; L <= 16; ++L) ring[(end + 1 + L) & 31] = (unsigned)INF;
                ring[(end + 1) & 31] = (unsigned)k1;
                bool virt = true;     // the line being parsed has no '\n' of its own
                unsigned long long tot = 0;
                for (int i = end; i >= start; --i) {
                    const unsigned b = win[i];
                    if (b == '\n') {
                        tot += (unsigned)(((k1 + i + 1) >> 4) + (virt ? 0 : 1));
                        virt = false;
                        k1 = -i;   // cost 0 at the line end
                        st = 0;
                        ring[i & 31] = (unsigned)(-i);
                        // positions right of the line end must never be candidates
                        for (int L = 1; L <= 16; ++L) ring[(i + L) & 31] = (unsigned)INF;
                        continue;  // the decision byte stays '\n'
                    }
                    const unsigned e = dfa32[st * ncol + s_cmap[b]];
                    st = e >> 16;
                    unsigned m = e & 0xffffu;
                    int mm = INF;
                    while (m) {
                        const int L = __ffs(m);
                        m &= m - 1u;
                        mm = min(mm, (int)ring[(i + L) & 31]);
                    }
                    const int esc = k1 + 32;
                    const int best = min(esc, mm + 16);
                    const int t = best + i + 16;
                    const int L = 16 - (t & 15);
                    k1 = (t & ~15) - i;
                    ring[i & 31] = (unsigned)k1;
                    win[i] = (uint8_t)(esc < mm + 16 ? 0x20u : (L == 1 ? b : codes[st * CX_CODES + L - 1]));
                }
                if (end >= start) tot += (unsigned)(((k1 + start) >> 4) + (virt ? 0 : 1));
                acc = (unsigned)(tot + 4ull * (unsigned)(end >= start ? end - start + 1 : 0));
            } else if (SL) {
                // One byte-exact slice per lane, parsed right to left in one
                // range.  A slice whose last byte is not a '\n' is entered in
                // the line-end state (a guess); after the pass the guess is
                // checked against the right neighbour's exit state and, where
                // it differs, the slice is parsed again from the true state
                // next to the guessed one until the two meet (a '\n' resets
                // both).  Costs are not kept: P6 counts the output.
                if (!long_ranges && start <= end) atomicMin(&s_r0, start);
                __syncthreads();  // P2 / P3 of every warp done (slices cross line-lanes)
                const int R0 = s_r0, R1 = s_last_nl;
                const int sz = R1 >= R0 ? (R1 - R0 + CX_NT) / CX_NT : 0;
                const int s0 = R0 + tid * sz, e0 = min(R1, s0 + sz - 1);
                const bool any = sz > 0 && s0 <= e0;
                const bool spec = any && win[e0] != '\n' && e0 < R1;  // (R1: nothing of the tile right of it)
                // the guess: the state after a short warm-up over the next slice's
                // first bytes from a virtual line end (the right neighbour
                // rewrites those bytes last; a stale read only changes the guess)
                if (spec)
                    for (int p = min(e0 + CX_PWARM, R1); p > e0; --p) step(win[p]);
                const unsigned guess = st;
                if (any) parse_range(s0, e0);
                S.lane_c[tid] = (int)st;  // exit state (read by the left neighbour)
                __syncthreads();
                unsigned assumed = guess;  // the entry state the slice's decisions were made from
                for (;;) {
                    const unsigned truth = spec ? (unsigned)S.lane_c[tid + 1] : 0u;
                    const bool need = spec && truth != assumed;
                    if (!__syncthreads_or(need)) break;  // (also: every lane has read)
                    if (need) {
                        unsigned so = assumed, sn = truth;
                        int p = e0;
                        for (; p >= s0; --p) {
                            const unsigned c = win[p];
                            const unsigned b = c == 0x20u ? (cx_bit(S.fbits, p) ? 0x01u : job.in[ws + p]) : s_exp0[c];
                            const unsigned col = s_cmap[b];
                            const unsigned eo = cx_lw(pa_base + so + col);
                            const unsigned en = cx_lw(pa_base + sn + col);
                            so = eo & 0xffffu;
                            sn = en & 0xffffu;
                            win[p] = (uint8_t)(((en >> 16) & 0xffu) | (b & (unsigned)((int)en >> 31)));
                            if (sn == so) break;
                        }
                        assumed = truth;
                        if (p < s0) S.lane_c[tid] = (int)sn;  // never met: the exit state changed
                    }
                    __syncthreads();
                }
            } else if (!p4_exact) {
                parse_range(start, end);
            } else {
                if (SL && !long_ranges && start <= end) atomicMin(&s_r0, start);
                __syncthreads();  // P2 / P3 of every warp done (slices cross line-lanes); R0 set
                const int R0 = s_r0, R1 = s_last_nl;
                const int sz = R1 >= R0 ? (R1 - R0 + CX_NT) / CX_NT : 0;
                const int s0 = R0 + tid * sz, e0 = min(R1, s0 + sz - 1);
                bool spec = false, found = false;
                unsigned spec_state = 0, racc = 0;
                int rlo = s0, rj = 0;
                if (sz > 0 && s0 <= e0) {
                    // entry state at e0
                    if (PA && win[e0] != '\n' && e0 < R1) {
                        // no warm-up: enter in the line-end state; a wrong guess
                        // is repaired below from the right neighbour's exit
                        // state, only up to where the two parses converge
                        spec = true;
                        spec_state = 0;
                    } else if (win[e0] != '\n' && e0 < R1) {
                        // every such entry is checked below, also when a newline was
                        // found (the check does not depend on when the right
                        // neighbour rewrites these bytes; it rewrites them last)
                        spec = true;
                        const int lim = min(e0 + CX_WARM, R1);
                        int p = e0 + 1;
                        while (p < lim && win[p] != '\n') ++p;  // R1 is a newline
                        found = win[p] == '\n';
                        if (!found) step('\n');                   // a virtual line end right of the warm-up
                        for (; p > e0; --p) step(win[p]);
                        spec_state = (wi << 16) | st;
                    }
                    __syncwarp();
                    // the line-lane owning e0: the last lane whose cut lies before it
                    int lo = 0, hi = CX_NT - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi + 1) >> 1;
                        if (S.lane_a[mid] < e0) lo = mid;
                        else hi = mid - 1;
                    }
                    int j = lo, h = e0;
                    bool first_piece = true;
                    for (;;) {
                        const int l = max(s0, S.lane_a[j] + 1);
                        acc = 0;
                        parse_range(l, h);
                        atomicAdd(&S.lane_b[j], (int)acc - 4 * (h - l + 1));
                        if (first_piece) {
                            racc = acc;
                            rlo = l;
                            rj = j;
                            first_piece = false;
                        }
                        if (l <= s0) break;
                        h = l - 1;
                        do {
                            --j;
                        } while (j > 0 && S.lane_a[j] >= h);
                    }
                } else {
                    __syncwarp();
                }
                S.lane_c[tid] = (int)((wi << 16) | st);  // exit state (read by the left neighbour)
                __syncthreads();
                // verify speculative entries against the right neighbour's exit
                for (int round = 0;; ++round) {
                    unsigned truth = 0;
                    bool need = false;
                    if (spec) {
                        truth = (unsigned)S.lane_c[tid + 1];
                        need = truth != spec_state;
                    }
                    if (kPhases && job.timing == 6 && round == 0) {  // debug: entries and first-round mismatches by warm-up kind
                        const unsigned F = 0xffffffffu;
                        if (lane == 0) {
                            atomicAdd(&job.ctl->phase[0], (unsigned long long)__popc(__ballot_sync(F, spec && found)));
                            atomicAdd(&job.ctl->phase[1], (unsigned long long)__popc(__ballot_sync(F, spec && !found)));
                            atomicAdd(&job.ctl->phase[2], (unsigned long long)__popc(__ballot_sync(F, need && found)));
                            atomicAdd(&job.ctl->phase[3], (unsigned long long)__popc(__ballot_sync(F, need && !found)));
                        } else {
                            __ballot_sync(F, spec && found);
                            __ballot_sync(F, spec && !found);
                            __ballot_sync(F, need && found);
                            __ballot_sync(F, need && !found);
                        }
                    }
                    if (!__syncthreads_or(need)) break;
                    if (PA && need) {
                        // Re-run the first piece from the true entry state next to
                        // the speculative run (both over the bytes rebuilt from the
                        // decisions) until the two states meet; from there on every
                        // decision and cost is the same.  A '\n' resets both, so
                        // the repair stays inside the piece.
                        unsigned so = spec_state, sn = truth;
                        int d = 0, p = e0;
                        for (; p >= rlo; --p) {
                            const unsigned c = win[p];
                            const unsigned b = c == 0x20u ? (cx_bit(S.fbits, p) ? 0x01u : job.in[ws + p]) : s_exp0[c];
                            const unsigned col = s_cmap[b];
                            const unsigned eo = cx_lw(pa_base + so + col);
                            const unsigned en = cx_lw(pa_base + sn + col);
                            so = eo & 0xffffu;
                            sn = en & 0xffffu;
                            d += (int)((en >> 24) & 7u) - (int)((eo >> 24) & 7u);
                            win[p] = (uint8_t)(((en >> 16) & 0xffu) | (b & (unsigned)((int)en >> 31)));
                            if (sn == so) break;
                        }
                        atomicAdd(&S.lane_b[rj], d);
                        spec_state = truth;
                        if (p < rlo && rlo == s0) S.lane_c[tid] = (int)sn;
                    } else if (need) {
                        // rebuild the piece's bytes from its decisions, parse it again
                        for (int p = rlo; p <= e0; ++p) {
                            const unsigned d = win[p];
                            unsigned b;
                            if (d == 0x20u) b = cx_bit(S.fbits, p) ? 0x01u : job.in[ws + p];
                            else b = s_exp0[d];
                            win[p] = (uint8_t)b;
                        }
                        st = truth & 0xffffu;
                        wi = truth >> 16;
                        acc = 0;
                        parse_range(rlo, e0);
                        atomicAdd(&S.lane_b[rj], (int)acc - (int)racc);
                        racc = acc;
                        spec_state = truth;
                        if (rlo == s0) S.lane_c[tid] = (int)((wi << 16) | st);
                    }
                    __syncthreads();
                }
                acc = 0;
            }
        }
        pc.mark(job, 3);  // warp 0: parse
        __syncthreads();
        pc.mark(job, 4);  // wait for the slowest warp
        const int n_rare = min(s_nrare, CX_RARE);
        if (tid == 0 && s_nrare > CX_RARE) atomicOr(&job.ctl->overflow, 8ull);  // host: general kernel
        // ---- rare lines: general routine (HBM arena), one thread each ----
        for (int r = tid; r < n_rare; r += CX_NT) {
            CxRare &R = S.rare[r];
            if (R.kind == RK_ARENA && R.glob && job.ll_mode == 0) {
                // a long line: recorded for the block-parallel long-line kernels
                // (the host runs them and this kernel again, in mode 1)
                const unsigned long long i = atomicAdd(&job.ctl->ll_n, 1ull);
                if (i < (unsigned long long)job.ll_cap) {
                    job.ll[i].ge = ws + R.le;
                    atomicOr(&job.ctl->overflow, 16ull);
                    R.kind = RK_DROP;
                }
            }
            if (R.kind == RK_ARENA) {
                ZS_ASSERT(R.ls >= 0 && R.ls <= R.le && R.le < CX_WIN);
                long long ge = ws + R.le, gs = ws + R.ls;
                if (R.glob) {
                    int i = -1;
                    if (job.ll_mode == 1) {  // coded by the long-line kernels?
                        int lo = 0, hi = job.ll_n - 1;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (job.ll[mid].ge < ge) lo = mid + 1;
                            else hi = mid;
                        }
                        if (job.ll_n > 0 && job.ll[lo].ge == ge) i = lo;
                    }
                    if (i >= 0) {
                        gs = job.ll[i].gs;
                        if (job.ll[i].status == LL_OK) {
                            R.gs = gs;
                            R.ll = i;
                            R.out = (int)job.ll[i].cost + 1;
                            atomicAdd(&S.lane_b[R.lane], R.out);
                            s_has_ll = 1;
                            continue;
                        }
                    } else {
                        gs = ge;
                        while (gs > 0 && job.in[gs - 1] != '\n') --gs;
                    }
                }
                unsigned aoff = 0;
                int kind = E_NONE, eoff = -1;
                unsigned long long ids[2] = {0, 0};
                const long long cost = compress_line_global(job, tb, gs, ge - gs, &aoff, &kind, &eoff, ids);
                R.gs = gs;
                if (kind == -2) {
                    R.kind = RK_DROP;  // arena exhausted: the host grows it and re-runs
                } else if (kind == E_CR || (kind > 0 && !job.lenient)) {
                    R.kind = job.lenient ? RK_DROP : RK_STRICT;
                    R.err = kind;
                } else {
                    if (kind == -3) atomicAdd(&s_flag, 1u);
                    R.aoff = aoff;
                    R.out = (int)cost + 1;
                    atomicAdd(&S.lane_b[R.lane], (int)cost + 1);
                }
            }
            if (R.kind == RK_DROP) atomicAdd(&s_skip, 1u);
            if (R.kind == RK_STRICT) s_err_ord = 0;  // ordinal resolved after the scan
        }
        __syncthreads();
        const int nbytes = (!p4_exact && end >= start) ? end - start + 1 : 0;  // exact slices: costs are in lane_b
        const long long my_out = (long long)acc - 4ll * nbytes - sub + S.lane_b[tid];
        int p6a = start, p6b = end;
        unsigned long long p6off, tile_out;
        unsigned tile_lines;
        if (SL) {
            // ---- P6a: output bytes per byte-exact slice ----
            // A slice's output starts at the first decision at or after its
            // first byte on the path the reference's forward walk takes
            // (numba_impl.py:57-69).  Guess: the slice's first byte; after the
            // count, the left neighbour's exit (its first path position past
            // its slice) is the truth, and a wrong guess is walked again next
            // to the guessed path until the two paths meet.
            const uint8_t *win = S.win;
            const int R0 = s_r0, R1 = s_last_nl;
            const int sz = R1 >= R0 ? (R1 - R0 + CX_NT) / CX_NT : 0;
            const int s0 = R0 + tid * sz, e0 = min(R1, s0 + sz - 1);
            const bool any = sz > 0 && s0 <= e0;
            auto marker_out = [&](int p) {
                int o = 0;
                for (int r = 0; r < n_rare; ++r)
                    if (S.rare[r].kind == RK_ARENA && (S.rare[r].glob ? S.rare[r].le : S.rare[r].ls) == p) o += S.rare[r].out;
                return o;
            };
            // output bytes of the decision at p; L = positions it covers
            auto out_at = [&](int p, int &L) -> unsigned {
                const unsigned d = win[p];
                if (d == 0x20u) {
                    L = 1;
                    return cx_bit(S.fbits, p) ? (unsigned)marker_out(p) : 2u;
                }
                L = S.explen[d];
                return 1u;
            };
            int c = s0, x = s0;
            unsigned cnt = 0;
            const bool spec = any && s0 > R0 && win[s0 - 1] != '\n';
            if (spec) {
                // guess: the path through a decision up to CX_PWARM bytes left
                // (exact when a line starts there)
                const int w = max(R0, s0 - CX_PWARM);
                int p = s0 - 1;
                while (p > w && win[p] != '\n') --p;
                c = win[p] == '\n' ? p + 1 : w;
                while (c < s0) c += win[c] == 0x20u ? 1 : S.explen[win[c]];
            }
            if (any) {
                int p = c;
                while (p <= e0) {
                    int L;
                    cnt += out_at(p, L);
                    p += L;
                }
                x = p;
            }
            __syncthreads();  // lane_a (the cuts) is free from here on
            S.lane_a[tid] = x;  // exit: first path position of the right neighbour's slice
            __syncthreads();
            for (;;) {
                const int truth = spec ? S.lane_a[tid - 1] : 0;
                const bool need = spec && truth != c;
                if (!__syncthreads_or(need)) break;
                if (need) {
                    int a = truth, b = c;
                    while (a != b && (a <= e0 || b <= e0)) {
                        int L;
                        if (a < b) {
                            cnt += out_at(a, L);
                            a += L;
                        } else {
                            cnt -= out_at(b, L);
                            b += L;
                        }
                    }
                    c = truth;
                    if (a != b) {  // the paths never met in the slice: new exit
                        x = a;
                        S.lane_a[tid] = x;
                    }
                }
                __syncthreads();
            }
            // ---- P5: tile output bytes and lines (one scan); publish ----
            unsigned long long tot;
            const unsigned long long ex = block_exscan_n<unsigned long long, CX_NT>(
                ((unsigned long long)cnt << 24) | (unsigned long long)nlines, s_tmp64, tot);
            p6off = ex >> 24;
            tile_out = tot >> 24;
            tile_lines = (unsigned)(tot & 0xffffffu);
            S.lane_c[tid] = (int)(ex & 0xffffffu);  // line-lane line bases (strict error ordinals)
            if (tid == 0) lookback_publish(job.ts, t, tile_out, (unsigned long long)tile_lines);
            p6a = c;
            p6b = any ? e0 : c - 1;
        } else {
            // ---- P5: tile output bytes and lines (one scan); publish ----
            unsigned long long tot;
            const unsigned long long ex = block_exscan_n<unsigned long long, CX_NT>(
                ((unsigned long long)my_out << 24) | (unsigned long long)nlines, s_tmp64, tot);
            const unsigned long long my_off = ex >> 24;
            tile_out = tot >> 24;
            tile_lines = (unsigned)(tot & 0xffffffu);
            S.lane_c[tid] = (int)(ex & 0xffffffu);  // lane line bases (strict error ordinals)
            if (tid == 0) lookback_publish(job.ts, t, tile_out, (unsigned long long)tile_lines);
            // ---- P6: emit (to staging now, or to HBM after the look-back) ----
            // Long-line tiles emit byte-exact slices: a slice starts at the first
            // decision at or after its first byte on the path the reference's
            // forward walk takes (numba_impl.py:57-69) -- found from a line start
            // within CX_WARM bytes to its left, or guessed from a walk started
            // CX_WARM bytes left and checked against the left neighbour's exit --
            // then counts its output bytes (one scan gives the slice offsets) and
            // emits them.
            p6off = my_off;
            if (long_ranges) {
                const uint8_t *win = S.win;
                const int R0 = s_r0, R1 = s_last_nl;
                const int sz = R1 >= R0 ? (R1 - R0 + CX_NT) / CX_NT : 0;
                const int s0 = R0 + tid * sz, e0 = min(R1, s0 + sz - 1);
                auto marker_out = [&](int p) {
                    int o = 0;
                    for (int r = 0; r < n_rare; ++r)
                        if (S.rare[r].kind == RK_ARENA && (S.rare[r].glob ? S.rare[r].le : S.rare[r].ls) == p) o += S.rare[r].out;
                    return o;
                };
                auto count = [&](int p, unsigned &cnt) {  // walk [p, e0]; returns the exit position
                    cnt = 0;
                    while (p <= e0) {
                        const unsigned d = win[p];
                        if (d == 0x20u) {
                            cnt += cx_bit(S.fbits, p) ? (unsigned)marker_out(p) : 2u;
                            ++p;
                        } else {
                            ++cnt;
                            p += S.explen[d];
                        }
                    }
                    return p;
                };
                int c = s0, x = s0;
                bool spec = false;
                unsigned cnt = 0;
                if (sz > 0 && s0 <= e0) {
                    if (s0 > R0 && win[s0 - 1] != '\n') {
                        const int w = max(R0, s0 - CX_WARM);
                        int p = s0 - 1;
                        while (p > w && win[p] != '\n') --p;
                        if (win[p] == '\n') {
                            c = p + 1;
                        } else {
                            c = w;
                            spec = w > R0;  // R0 starts the path
                        }
                        while (c < s0) c += win[c] == 0x20u ? 1 : S.explen[win[c]];
                    }
                    x = count(c, cnt);
                }
                __syncthreads();  // lane_a (the cuts) is free from here on
                S.lane_a[tid] = x;  // exit: first path position of the right neighbour's slice
                __syncthreads();
                for (;;) {
                    bool need = false;
                    int truth = 0;
                    if (spec) {
                        truth = S.lane_a[tid - 1];
                        need = truth != c;
                    }
                    if (!__syncthreads_or(need)) break;
                    if (need) {
                        c = truth;
                        x = count(c, cnt);
                        S.lane_a[tid] = x;
                    }
                    __syncthreads();
                }
                unsigned long long stot;
                p6off = block_exscan_n<unsigned long long, CX_NT>((unsigned long long)cnt, s_tmp64, stot);
                p6a = c;
                p6b = e0;
                if (!(sz > 0 && s0 <= e0)) p6b = p6a - 1;  // empty slice
            }
        }
        const bool staged = tile_out <= (unsigned long long)CX_STAGE && !s_has_ll;
        ZS_ASSERT(p6off <= tile_out);
        pc.mark(job, 5);  // output scan
        unsigned esc = 0;
        if (staged && p6a <= p6b)
            esc = cx_emit_range<true>(job, S, ws, p6a, p6b, S.out, p6off, n_rare);
        if (tid < 32) {
            unsigned long long po, pl;
            lookback_resolve(job.ts, t, tile_out, (unsigned long long)tile_lines, po, pl);
            if (tid == 0) {
                s_pre_out = po;
                s_pre_lines = pl;
            }
        }
        __syncthreads();
        pc.mark(job, 6);  // emit + look-back
        const unsigned long long pre_out = s_pre_out;
        const bool fits = pre_out + tile_out <= (unsigned long long)job.out_cap;
        if (!staged && fits && p6a <= p6b)
            esc = cx_emit_range<false>(job, S, ws, p6a, p6b, job.out, pre_out + p6off, n_rare);
        if (esc) atomicAdd(&s_esc, esc);
        if (tid == 0) {
            atomicAdd(&job.ctl->total_out, tile_out);
            atomicAdd(&job.ctl->lines, (unsigned long long)(tile_lines - s_skip));
            atomicAdd(&job.ctl->in_lines, (unsigned long long)tile_lines);
            if (s_skip && job.lenient) atomicAdd(&job.ctl->skipped, (unsigned long long)s_skip);
            if (s_flag) atomicAdd(&job.ctl->flagged, (unsigned long long)s_flag);
            if (!fits) atomicOr(&job.ctl->overflow, 1ull);
        }
        // ---- strict error: details of the tile's first bad line ----
        if (tid == 0 && s_err_ord != 0x7fffffff) {
            int ord = 0x7fffffff;
            long long gs = 0, ge = 0;
            int kind = E_NONE;
            for (int r = 0; r < n_rare; ++r) {
                const CxRare &R = S.rare[r];
                if (R.kind == RK_STRICT && S.lane_c[R.lane] + R.local < ord) {
                    ord = S.lane_c[R.lane] + R.local;
                    ge = ws + R.le;
                    gs = R.glob ? R.gs : ws + R.ls;
                    kind = R.err;
                }
            }
            TileErr e = {kind, 0, -1, {0, 0}};
            bool cr = false;
            for (long long k = gs; k < ge; ++k) cr |= job.in[k] == '\r';
            if (cr) {
                e.kind = E_CR;
            } else if (job.preprocess) {
                int nl2, eoff = -1;
                unsigned long long ids[2] = {0, 0};
                const long long n_l = ge - gs;
                const unsigned long long need = (4 * (unsigned long long)n_l + 19) & ~15ull;
                const unsigned long long a = atomicAdd(&job.ctl->arena_used, need);
                uint8_t *tmp = a + need <= (unsigned long long)job.arena_cap ? job.arena + a : nullptr;
                if (!tmp) atomicOr(&job.ctl->overflow, 2ull);
                const int k = tmp ? preprocess_line(job.in + gs, (int)n_l, tmp, tmp + n_l + 1, &nl2, &eoff, ids)
                                  : E_NONE;
                e.kind = k;
                e.offset = eoff;
                e.ids[0] = ids[0];
                e.ids[1] = ids[1];
            }
            job.terr[t] = e;
            __threadfence();
            atomicMin(&job.ctl->err_key, ((s_pre_lines + (unsigned long long)ord) << 24) |
                                             (unsigned long long)(t & 0xffffff));
        }
        if (fits && staged) cx_store_out(job.out + pre_out, S.out, (int)tile_out);
        pc.mark(job, 7);  // stats, store
    }
}

}  // namespace zs
