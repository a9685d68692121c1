// zs_kernels.cuh -- sm_100a kernels: fused single-pass tile kernels for the
// whole-buffer path and the thread-per-line parity-shim kernels.
#pragma once
#include "zs_device.cuh"

namespace zs {

// ----------------------------------------------------------------------------
// shared-memory carve-up for the compress tile kernel
// ----------------------------------------------------------------------------
struct CSmem {
    uint16_t *dfa;    // AC DFA (mask-index entries in transducer mode)
    uint32_t *t2;     // cost-window transducer (transducer mode only)
    uint8_t *codes;
    uint8_t *explen;
    uint8_t *win;
    uint8_t *dec;
    uint8_t *out;
    uint16_t *queue;  // line starts (window offsets) of the current round
    uint16_t *qlen;   // their lengths (0xffff = runs past the window)
    uint16_t *qsort;  // queue indices sorted by length, longest first
    unsigned *qoff;   // per line: payload size, then (scanned) tile output offset
    unsigned *chunk;  // per-thread-chunk output byte sums
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline int compress_smem_bytes(int n_states, int n_windows) {
    return align16(n_states * NCOL * 2) + n_windows * T2_MASKS * 4 + align16(n_states * FAST_W) +
           256 + align16(WIN + 16) +
           align16(WIN + 16) + align16(OUTCAP) + 3 * QCAP * 2 + QCAP * 4 + NT * 4;
}

__device__ inline CSmem carve_csmem(uint8_t *p, int ns, int nw) {
    CSmem S;
    S.dfa = reinterpret_cast<uint16_t *>(p); p += align16(ns * NCOL * 2);
    S.t2 = reinterpret_cast<uint32_t *>(p); p += nw * T2_MASKS * 4;
    S.codes = p; p += align16(ns * FAST_W);
    S.explen = p; p += 256;
    S.win = p; p += align16(WIN + 16);
    S.dec = p; p += align16(WIN + 16);
    S.out = p; p += align16(OUTCAP);
    S.queue = reinterpret_cast<uint16_t *>(p); p += QCAP * 2;
    S.qlen = reinterpret_cast<uint16_t *>(p); p += QCAP * 2;
    S.qsort = reinterpret_cast<uint16_t *>(p); p += QCAP * 2;
    S.qoff = reinterpret_cast<unsigned *>(p); p += QCAP * 4;
    S.chunk = reinterpret_cast<unsigned *>(p);
    return S;
}

// Copy the staged tile output to HBM: byte stores until dst is 16-byte
// aligned, then 16-byte vector stores assembled from smem bytes.
__device__ __forceinline__ void store_out(uint8_t *dst, const uint8_t *src, int len) {
    const int head = min(len, (int)((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15));
    if ((int)threadIdx.x < head) dst[threadIdx.x] = src[threadIdx.x];
    const int nvec = (len - head) >> 4;
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + head);
    for (int k = threadIdx.x; k < nvec; k += NT) {
        const uint8_t *q = src + head + 16 * k;
        uint4 v;
        v.x = q[0] | (q[1] << 8) | (q[2] << 16) | ((unsigned)q[3] << 24);
        v.y = q[4] | (q[5] << 8) | (q[6] << 16) | ((unsigned)q[7] << 24);
        v.z = q[8] | (q[9] << 8) | (q[10] << 16) | ((unsigned)q[11] << 24);
        v.w = q[12] | (q[13] << 8) | (q[14] << 16) | ((unsigned)q[15] << 24);
        d4[k] = v;
    }
    for (int k = head + (nvec << 4) + threadIdx.x; k < len; k += NT) dst[k] = src[k];
}


// Stage window bytes [ws, ws+len) of `in` into smem `win` (positions before
// the buffer start read as '\n' so offset 0 is a line start).
__device__ __forceinline__ void load_window(const uint8_t *in, long long n, long long ws, int len,
                                            uint8_t *win) {
    const bool aligned = ((reinterpret_cast<uintptr_t>(in) & 15) == 0) && ws >= 0 &&
                         ws + len <= n && (len & 15) == 0;
    if (aligned) {
        const uint4 *src = reinterpret_cast<const uint4 *>(in + ws);
        uint4 *dst = reinterpret_cast<uint4 *>(win);
        for (int k = threadIdx.x; k < len / 16; k += NT) dst[k] = __ldcs(src + k);
    } else {
        for (int k = threadIdx.x; k < len; k += NT) {
            long long g = ws + k;
            win[k] = g < 0 ? (uint8_t)'\n' : (g < n ? __ldcs(in + g) : (uint8_t)'\n');
        }
    }
}

// Each thread scans its CHUNK of the tile for line starts (a start is a
// position p in [T0, T1) whose previous byte is '\n').  Returns the count and,
// when `queue` is given, writes the window offsets of the starts whose
// ordinal falls in [q0, q1) at queue[ord - q0].
template <int CH = CHUNK>
__device__ __forceinline__ int scan_starts(const uint8_t *win, int tile_len, int base_ord,
                                           uint16_t *queue, int q0, int q1) {
    const int c0 = threadIdx.x * CH;
    const int c1 = min(c0 + CH, tile_len);
    if (c0 >= c1) return 0;
    // the predecessor bytes of the chunk's positions: window [a, b)
    const int a = HEAD + c0 - 1, b = HEAD + c1 - 1;
    int cnt = 0;
    for (int wa = a & ~3; wa < b; wa += 4) {
        const unsigned x = *reinterpret_cast<const unsigned *>(win + wa) ^ 0x0a0a0a0au;
        // exact per-byte zero test: bit 7 of each byte set iff byte == '\n'
        unsigned z = ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);
        if (wa < a) z &= 0xffffffffu << (8 * (a - wa));
        if (wa + 4 > b) z &= 0xffffffffu >> (8 * (wa + 4 - b));
        if (queue) {
            while (z) {
                const int pos = wa + ((__ffs(z) - 1) >> 3);
                const int ord = base_ord + cnt;
                if (ord >= q0 && ord < q1) queue[ord - q0] = (uint16_t)(pos + 1);
                ++cnt;
                z &= z - 1;
            }
        } else {
            cnt += __popc(z);
        }
    }
    return cnt;
}

// Find the end (window offset of '\n', or of EOF) of the line starting at
// window offset p; -1 if the line runs past the staged window.
__device__ __forceinline__ int find_end(const uint8_t *win, int p, int win_len, bool window_hits_eof) {
    for (int k = p; k < win_len; ++k)
        if (win[k] == '\n') return k;
    return window_hits_eof ? win_len : -1;
}

// arena block for a line processed out of smem:
// [ArenaHdr][pre bytes: 3n+3, 16-aligned][decisions: 3n+4]
struct ArenaHdr {
    long long n_pre;     // length of the (preprocessed) line
    long long bytes_off; // offset of the line bytes in the arena, -1 = in the input
    long long dec_off;   // offset of the decision bytes in the arena
    long long pad;
};

// Process one line in HBM (long line or one that grows under renumbering).
// Returns the payload size (cost[0]) and sets *kind to an error kind, or
// -2 when the arena is exhausted.
__device__ long long compress_line_global(const Job &job, const Tables &tb, long long gstart,
                                          long long n_l, unsigned *arena_off16, int *kind,
                                          int *eoff, unsigned long long ids[2]) {
    const uint8_t *src = job.in + gstart;
    long long need = (long long)sizeof(ArenaHdr) + ((3 * n_l + 3 + 15) & ~15ll) +
                     ((3 * n_l + 4 + 15) & ~15ll);
    unsigned long long a = atomicAdd((unsigned long long *)&job.ctl->arena_used,
                                     (unsigned long long)need);
    if ((long long)(a + need) > job.arena_cap) {
        atomicOr((unsigned long long *)&job.ctl->overflow, 2ull);
        *kind = -2;
        return 0;
    }
    uint8_t *blk = job.arena + a;
    ArenaHdr *h = reinterpret_cast<ArenaHdr *>(blk);
    uint8_t *pre = blk + sizeof(ArenaHdr);
    uint8_t *dec = pre + ((3 * n_l + 3 + 15) & ~15ll);
    h->dec_off = (long long)(dec - job.arena);
    *arena_off16 = (unsigned)(a >> 4);
    const uint8_t *line = src;
    long long n_pre = n_l;
    *kind = E_NONE;
    if (job.preprocess) {
        int nl2 = 0;
        int k = preprocess_line(src, (int)n_l, dec, pre, &nl2, eoff, ids);
        if (k != E_NONE) {
            *kind = k;
            if (k == E_CR || !job.lenient) return 0;
            // lenient: keep the raw line (pipeline.py:108-115)
            *kind = -3;  // flagged
        } else {
            line = pre;
            n_pre = nl2;
        }
    } else {
        for (long long q = 0; q < n_l; ++q)
            if (src[q] == '\r') { *kind = E_CR; return 0; }
    }
    h->n_pre = n_pre;
    h->bytes_off = line == src ? -1 : (long long)(pre - job.arena);
    // same decisions from every parse (tests/test_gpu_parity.py); the table
    // walks are L1/L2-resident, the dense trie walk costs HBM latency per step
    if (n_pre < (1ll << 30)) {
        if (tb.t2) return dp_t2(line, (int)n_pre, dec, tb.dfa2, tb.t2, tb.codes);
        if (tb.fast) return dp_fast<FAST_W>(line, (int)n_pre, dec, tb.dfa, tb.codes);
    }
    long long ring[128];
    return dp_generic(line, n_pre, dec, tb, ring);
}

// ----------------------------------------------------------------------------
// compress emit: one thread walks the positions of its CHUNK in a single flat
// loop (uniform trip structure across the warp).  At a line start the walk
// arms `nxt` at the line's first decision; every position equal to `nxt`
// emits its code (or escape + literal) and advances nxt by the code length;
// D_END emits the record separator.  Lines that started in the chunk are
// finished past the chunk end.
// ----------------------------------------------------------------------------
template <bool STAGED>
__device__ __forceinline__ unsigned emit_chunk(const Job &job, const CSmem &S, long long ws,
                                               int tile_len, unsigned long long w, uint8_t *o) {
    const int c0 = threadIdx.x * CHUNK;
    const int c1 = min(c0 + CHUNK, tile_len);
    unsigned esc = 0;
    int nxt = -1;
    // warp-uniform trip count (lanes finish their last line at different x)
    for (int x = c0; __any_sync(0xffffffffu, x < c1 || nxt >= 0); ++x) {
        const int p = HEAD + x;
        if (x < c1 && S.win[p - 1] == '\n') {
            const uint8_t first = S.dec[p];
            nxt = first == D_DROP || first == D_GLOBAL ? -1 : p;
            if (first == D_GLOBAL) {
                // out-of-smem line: its decisions live in the HBM arena
                const unsigned aoff = S.dec[p + 1] | (S.dec[p + 2] << 8) | (S.dec[p + 3] << 16) |
                                      ((unsigned)S.dec[p + 4] << 24);
                const uint8_t *blk = job.arena + ((long long)aoff << 4);
                const ArenaHdr *h = reinterpret_cast<const ArenaHdr *>(blk);
                const uint8_t *bytes = h->bytes_off < 0 ? job.in + ws + p : job.arena + h->bytes_off;
                const uint8_t *dec = job.arena + h->dec_off;
                uint8_t *og = job.out;  // direct mode is forced for such tiles
                for (long long i = 0; i < h->n_pre;) {
                    const uint8_t c = dec[i];
                    if (c == D_ESC) {
                        og[w++] = 0x20;
                        og[w++] = bytes[i];
                        ++esc;
                        ++i;
                    } else {
                        og[w++] = c;
                        i += S.explen[c];
                    }
                }
                og[w++] = '\n';
            }
        }
        if (p == nxt) {
            const uint8_t c = S.dec[p];
            if (c == D_END) {
                o[w++] = '\n';
                nxt = -1;
            } else if (c == D_ESC) {
                o[w++] = 0x20;
                o[w++] = S.win[p];
                ++esc;
                ++nxt;
            } else {
                o[w++] = c;
                nxt += S.explen[c];
            }
        }
    }
    return esc;
}

// ----------------------------------------------------------------------------
// compress emit, one line per lane (the tile's lines were parsed in one
// round): warps take the same length-sorted groups of 32 lines as the parse,
// so the lanes' decision walks have similar lengths.  w = the line's output
// offset (tile-local when staged).
// ----------------------------------------------------------------------------
__device__ __forceinline__ unsigned emit_lines(const Job &job, const CSmem &S, long long ws, int nq,
                                               int *grp, uint8_t *o, unsigned long long base) {
    unsigned esc = 0;
    for (;;) {
        int g = 0;
        if ((threadIdx.x & 31) == 0) g = atomicAdd(grp, 1);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g * 32 >= nq) break;
        const int r = g * 32 + (threadIdx.x & 31);
        __syncwarp();
        if (r < nq) {
            const int q = S.qsort[r];
            const int p = S.queue[q];
            unsigned long long w = base + S.qoff[q];
            const uint8_t first = S.dec[p];
            if (first == D_GLOBAL) {
                const unsigned aoff = S.dec[p + 1] | (S.dec[p + 2] << 8) | (S.dec[p + 3] << 16) |
                                      ((unsigned)S.dec[p + 4] << 24);
                const uint8_t *blk = job.arena + ((long long)aoff << 4);
                const ArenaHdr *h = reinterpret_cast<const ArenaHdr *>(blk);
                const uint8_t *bytes = h->bytes_off < 0 ? job.in + ws + p : job.arena + h->bytes_off;
                const uint8_t *dec = job.arena + h->dec_off;
                for (long long i = 0; i < h->n_pre;) {
                    const uint8_t c = dec[i];
                    if (c == D_ESC) {
                        o[w++] = 0x20;
                        o[w++] = bytes[i];
                        ++esc;
                        ++i;
                    } else {
                        o[w++] = c;
                        i += S.explen[c];
                    }
                }
                o[w++] = '\n';
            } else if (first != D_DROP) {
                for (int i = p;;) {
                    const uint8_t c = S.dec[i];
                    if (c == D_END) break;
                    if (c == D_ESC) {
                        o[w++] = 0x20;
                        o[w++] = S.win[i];
                        ++esc;
                        ++i;
                    } else {
                        o[w++] = c;
                        i += S.explen[c];
                    }
                }
                o[w++] = '\n';
            }
        }
        __syncwarp();
    }
    return esc;
}

// ----------------------------------------------------------------------------
// compress: one persistent CTA per SM, tiles in ticket order.
// W = fast-path window (max pattern length) or 0 for the generic trie walk.
// ----------------------------------------------------------------------------
template <int W, bool T2>
__global__ void __launch_bounds__(NT, 1) compress_tiles(Job job, Tables tb) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ unsigned long long s_tmp64[NWARP];
    __shared__ int s_tmp32[NWARP];
    __shared__ unsigned s_hist[256];
    __shared__ __align__(16) uint8_t s_lut[8 * 256];  // tokenizer transducer
    __shared__ long long s_tile;
    __shared__ int s_err_ord, s_global, s_grp;
    __shared__ unsigned long long s_wmax, s_wsum, s_wmin, s_ngrp, s_trn, s_tdp;
    __shared__ unsigned long long s_pre_out, s_pre_lines;
    __shared__ unsigned s_kept, s_esc, s_skip, s_flag;

    const CSmem S = carve_csmem(smem, W ? tb.n_states : 0, T2 ? tb.n_windows : 0);
    {
        const int ns = W ? tb.n_states : 0;
        if (W) {
            const uint4 *src = reinterpret_cast<const uint4 *>(T2 ? tb.dfa2 : tb.dfa);
            uint4 *dst = reinterpret_cast<uint4 *>(S.dfa);
            for (int k = threadIdx.x; k < align16(ns * NCOL * 2) / 16; k += NT) dst[k] = src[k];
            for (int k = threadIdx.x; k < ns * FAST_W; k += NT) S.codes[k] = tb.codes[k];
        }
        if (T2)
            for (int k = threadIdx.x; k < tb.n_windows * T2_MASKS; k += NT) S.t2[k] = tb.t2[k];
        for (int k = threadIdx.x; k < 256; k += NT) S.explen[k] = tb.exp_len[k];
        for (int k = threadIdx.x; k < 8 * 256; k += NT) s_lut[k] = tk_entry(k >> 8, k & 255);
    }
    const int tid = threadIdx.x;
    PhaseClock pc;
    pc.start();

    for (;;) {
        __syncthreads();
        pc.mark(job, 2);  // end of previous tile / table load
        if (tid == 0) {
            s_tile = (long long)atomicAdd(&job.ctl->ticket, 1ull);
            s_err_ord = 0x7fffffff;
            s_global = 0;
            s_kept = s_esc = s_skip = s_flag = 0;
        }
        __syncthreads();
        const long long t = s_tile;
        if (t >= job.n_tiles) break;
        const long long T0 = t * (long long)TILE;
        const int tile_len = (int)min((long long)TILE, job.n - T0);
        const long long ws = T0 - HEAD;
        const long long we = min(job.n, T0 + TILE + EXTRA);
        const int win_len = (int)(we - ws);
        const bool hits_eof = we == job.n;
        load_window(job.in, job.n, ws, align16(win_len), S.win);
        S.chunk[tid] = 0;
        __syncthreads();

        // ---- line starts: per-thread chunk counts -> block scan ----
        const int my_cnt = scan_starts(S.win, tile_len, 0, nullptr, 0, 0);
        int tile_lines;
        const int my_off = block_exscan<int>(my_cnt, s_tmp32, tile_lines);

        pc.mark(job, 2);  // ticket, window load, line-start scan
        // ---- parse phase, in rounds of QCAP lines ----
        for (int q0 = 0; q0 < tile_lines; q0 += QCAP) {
            const int nq = min(QCAP, tile_lines - q0);
            if (my_cnt) scan_starts(S.win, tile_len, my_off, S.queue, q0, q0 + nq);
            for (int k = tid; k < 256; k += NT) s_hist[k] = 0;
            __syncthreads();
            // line lengths and a counting sort by length (longest first) so
            // the 32 lines a warp parses together have similar lengths
            for (int q = tid; q < nq; q += NT) {
                const int p = S.queue[q];
                const int end = (q + 1 < nq) ? S.queue[q + 1] - 1 : find_end(S.win, p, win_len, hits_eof);
                const int len = end < 0 ? 0xffff : end - p;
                S.qlen[q] = (uint16_t)len;
                atomicAdd(&s_hist[255 - min(len, 255)], 1u);
            }
            __syncthreads();
            {
                unsigned h = tid < 256 ? s_hist[tid] : 0u;
                unsigned tot;
                const unsigned ex = block_exscan<unsigned>(h, reinterpret_cast<unsigned *>(s_tmp32), tot);
                if (tid < 256) s_hist[tid] = ex;
            }
            __syncthreads();
            for (int q = tid; q < nq; q += NT) {
                const int len = S.qlen[q];
                const unsigned r = atomicAdd(&s_hist[255 - min(len, 255)], 1u);
                S.qsort[r] = (uint16_t)q;
            }
            if (tid == 0) {
                s_grp = 0;
                s_wmax = s_wsum = s_ngrp = s_trn = s_tdp = 0;
                s_wmin = ~0ull;
            }
            __syncthreads();
            pc.mark(job, 2);  // queue, lengths, sort
            const long long wt0 = clock64();
            int my_groups = 0;
            // warps pull groups of 32 lines, longest first (LPT scheduling).
            // Independent thread scheduling does not reconverge lanes on its
            // own: every divergent step below ends in __syncwarp() so the 32
            // lanes enter the parse together.
            for (;;) {
                int g = 0;
                if ((tid & 31) == 0) g = atomicAdd(&s_grp, 1);
                g = __shfl_sync(0xffffffffu, g, 0);
                if (g * 32 >= nq) break;
                ++my_groups;
                const int r = g * 32 + (tid & 31);
                const bool valid = r < nq;
                int ord = 0, p = HEAD, qlen = 0, q = 0;
                if (valid) {
                    q = S.qsort[r];
                    ord = q0 + q;
                    p = S.queue[q];
                    qlen = S.qlen[q];
                }
                const int chunk_owner = (p - HEAD) / CHUNK;
                int kind = E_NONE;
                long long size = 0;
                bool global_line = valid && qlen == 0xffff;
                bool do_dp = valid && !global_line;
                uint8_t *s = S.win + p;
                uint8_t *d = S.dec + p;
                int n_l = qlen;
                // ---- CR policy + ring renumbering ----
                // renumber_fast is called by all 32 lanes (warp-uniform loops)
                int rn_k = E_NONE, rn_len = 0, rn_off = -1;
                unsigned long long rn_ids[2] = {0, 0};
                const bool rn = do_dp && job.preprocess;
                const long long tr0 = clock64();
                rn_k = renumber_fast(s, rn ? n_l : 0, s_lut, d, &rn_len, &rn_off, rn_ids);
                __syncwarp();
                if (kPhases && job.timing && (tid & 31) == 0) atomicAdd(&s_trn, (unsigned long long)(clock64() - tr0));
                if (do_dp) {
                    if (job.preprocess) {
                        int eoff = rn_off;
                        unsigned long long ids[2] = {rn_ids[0], rn_ids[1]};
                        int nlf = rn_len;
                        int k = rn_k;
                        if (k == E_NONE) {
                            n_l = nlf;
                        } else if (k == RN_FALLBACK) {
                            // pristine bytes, then the general routine
                            const uint8_t *g8 = job.in + ws + p;
                            for (int j = 0; j < n_l; ++j) s[j] = g8[j];
                            int nl2 = n_l;
                            k = preprocess_line(s, n_l, d, s, &nl2, &eoff, ids);
                            if (k == E_NONE) n_l = nl2;
                        }
                        if (k == -1) {
                            global_line = true;
                            do_dp = false;
                        } else if (k != E_NONE) {
                            if (k == E_CR) {
                                kind = E_CR;
                            } else if (job.lenient) {
                                // keep the raw line (pipeline.py:108-115)
                                const uint8_t *g8 = job.in + ws + p;
                                for (int j = 0; j < n_l; ++j) s[j] = g8[j];
                                atomicAdd(&s_flag, 1u);
                            } else {
                                kind = k;
                            }
                        }
                    } else {
                        for (int j = 0; j < n_l; ++j)
                            if (s[j] == '\r') { kind = E_CR; break; }
                    }
                    if (do_dp && kind != E_NONE) {
                        d[0] = D_DROP;
                        do_dp = false;
                        if (job.lenient) atomicAdd(&s_skip, 1u);
                        else atomicMin(&s_err_ord, ord);
                    }
                }
                __syncwarp();
                const long long td0 = clock64();
                // ---- min-cost parse (converged) ----
                if (do_dp) {
                    if constexpr (T2) {
                        size = dp_t2(s, n_l, d, S.dfa, S.t2, S.codes) + 1;
                    } else if constexpr (W > 0) {
                        size = dp_fast<W>(s, n_l, d, S.dfa, S.codes) + 1;
                    } else {
                        long long ring[128];
                        size = dp_generic(s, n_l, d, tb, ring) + 1;
                    }
                }
                __syncwarp();
                if (kPhases && job.timing && (tid & 31) == 0) atomicAdd(&s_tdp, (unsigned long long)(clock64() - td0));
                if (global_line) {
                    // line in HBM: find its end, process in the arena
                    const long long gs = ws + p;
                    long long ge = gs;
                    while (ge < job.n && job.in[ge] != '\n') ++ge;
                    unsigned aoff = 0;
                    int eoff = -1;
                    unsigned long long ids[2] = {0, 0};
                    long long cost = compress_line_global(job, tb, gs, ge - gs, &aoff, &kind, &eoff, ids);
                    s_global = 1;
                    if (kind == -2) {
                        d[0] = D_DROP;  // arena exhausted; host re-runs
                        kind = E_NONE;
                    } else if (kind == E_CR || (kind > 0 && !job.lenient)) {
                        d[0] = D_DROP;
                        if (job.lenient) atomicAdd(&s_skip, 1u);
                        else atomicMin(&s_err_ord, ord);
                    } else {
                        if (kind == -3) atomicAdd(&s_flag, 1u);
                        kind = E_NONE;
                        d[0] = D_GLOBAL;
                        d[1] = aoff & 0xff; d[2] = (aoff >> 8) & 0xff;
                        d[3] = (aoff >> 16) & 0xff; d[4] = (aoff >> 24) & 0xff;
                        size = cost + 1;
                    }
                }
                if (valid) S.qoff[q] = (unsigned)size;
                if (size) {
                    atomicAdd(&S.chunk[chunk_owner], (unsigned)size);
                    atomicAdd(&s_kept, 1u);
                }
                __syncwarp();
            }
            if (kPhases && job.timing && (tid & 31) == 0) {
                const unsigned long long dt = (unsigned long long)(clock64() - wt0);
                atomicMax(&s_wmax, dt);
                atomicMin(&s_wmin, dt);
                atomicAdd(&s_wsum, dt);
                atomicAdd(&s_ngrp, (unsigned long long)my_groups);
            }
            pc.mark(job, 6);  // thread 0's own parse work
            __syncthreads();
            pc.mark(job, 2);  // waiting for the slowest warp
            if (kPhases && job.timing && tid == 0) {
                atomicAdd(&job.ctl->phase[3], s_wmax);  // slot 3: max warp parse time
                atomicAdd(&job.ctl->phase[4], s_wmin);  // slot 4: min warp parse time
                atomicAdd(&job.ctl->phase[0], s_wsum / NWARP);  // slot 0: avg warp parse
                atomicAdd(&job.ctl->phase[1], s_ngrp);  // slot 1: groups per tile
                atomicAdd(&job.ctl->phase[5], s_trn / NWARP);  // slot 5: renumber per warp
                atomicAdd(&job.ctl->phase[7], s_tdp / NWARP);  // slot 7: parse per warp
            }
        }

        // ---- tile output size; publish the aggregate, emit to smem while
        // predecessors resolve, then the look-back ----
        unsigned long long tile_out;
        const unsigned long long my_out = S.chunk[tid];
        const unsigned long long my_out_off = block_exscan<unsigned long long>(my_out, s_tmp64, tile_out);
        const bool one_round = tile_lines <= QCAP;
        if (one_round) {
            // per-line output offsets: exclusive scan of S.qoff[0, tile_lines)
            const int per = (tile_lines + NT - 1) / NT;
            const int l0 = min(tid * per, tile_lines), l1 = min(l0 + per, tile_lines);
            unsigned sum = 0;
            for (int l = l0; l < l1; ++l) sum += S.qoff[l];
            unsigned tot;
            unsigned run = block_exscan<unsigned>(sum, reinterpret_cast<unsigned *>(s_tmp32), tot);
            for (int l = l0; l < l1; ++l) {
                const unsigned v = S.qoff[l];
                S.qoff[l] = run;
                run += v;
            }
            if (tid == 0) s_grp = 0;
            __syncthreads();
        }
        if (tid == 0) lookback_publish(job.ts, t, tile_out, (unsigned long long)tile_lines);
        const bool staged = !s_global && tile_out <= (unsigned long long)OUTCAP;
        if (staged) {
            const unsigned esc = one_round ? emit_lines(job, S, ws, tile_lines, &s_grp, S.out, 0)
                                           : emit_chunk<true>(job, S, ws, tile_len, my_out_off, S.out);
            if (esc) atomicAdd(&s_esc, esc);
        }
        pc.mark(job, 2);  // thread 0: publish + its own emit
        if (tid < 32) {
            unsigned long long po, pl;
            lookback_resolve(job.ts, t, tile_out, (unsigned long long)tile_lines, po, pl);
            if (tid == 0) {
                s_pre_out = po;
                s_pre_lines = pl;
            }
        }
        __syncthreads();
        pc.mark(job, 2);  // look-back resolve + wait for the slowest emitter
        const unsigned long long pre_out = s_pre_out;
        const bool fits = pre_out + tile_out <= (unsigned long long)job.out_cap;
        if (tid == 0) {
            atomicAdd(&job.ctl->total_out, tile_out);
            atomicAdd(&job.ctl->lines, (unsigned long long)s_kept);
            atomicAdd(&job.ctl->in_lines, (unsigned long long)tile_lines);
            if (s_skip) atomicAdd(&job.ctl->skipped, (unsigned long long)s_skip);
            if (s_flag) atomicAdd(&job.ctl->flagged, (unsigned long long)s_flag);
            if (!fits) atomicOr(&job.ctl->overflow, 1ull);
        }

        // ---- strict error: re-derive details of the first bad line ----
        if (tid == 0 && s_err_ord != 0x7fffffff) {
            int ord = s_err_ord, seen = 0, p = -1;
            for (int x = 0; x < tile_len && p < 0; ++x)
                if (S.win[HEAD + x - 1] == '\n') {
                    if (seen == ord) p = HEAD + x;
                    ++seen;
                }
            long long gs = ws + p, ge = gs;
            while (ge < job.n && job.in[ge] != '\n') ++ge;
            TileErr e = {E_CR, 0, -1, {0, 0}};
            bool cr = false;
            for (long long k = gs; k < ge; ++k) cr |= job.in[k] == '\r';
            if (!cr && job.preprocess) {
                // recompute from the pristine input (marks + output in HBM
                // scratch from the arena)
                int nl2, eoff = -1;
                unsigned long long ids[2] = {0, 0};
                const long long n_l = ge - gs;
                const unsigned long long need = (4 * (unsigned long long)n_l + 19) & ~15ull;
                unsigned long long a = atomicAdd(&job.ctl->arena_used, need);
                uint8_t *tmp = a + need <= (unsigned long long)job.arena_cap ? job.arena + a : nullptr;
                if (!tmp) atomicOr(&job.ctl->overflow, 2ull);
                int k = tmp ? preprocess_line(job.in + gs, (int)n_l, tmp, tmp + n_l + 1, &nl2, &eoff, ids)
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
        if (!fits) continue;

        // ---- store (staged) or emit straight to HBM (direct) ----
        if (staged) {
            store_out(job.out + pre_out, S.out, (int)tile_out);
            pc.mark(job, 2);
        } else {
            if (tid == 0) s_grp = 0;
            __syncthreads();
            const unsigned esc = one_round ? emit_lines(job, S, ws, tile_lines, &s_grp, job.out, pre_out)
                                           : emit_chunk<false>(job, S, ws, tile_len, pre_out + my_out_off, job.out);
            if (esc) atomicAdd(&s_esc, esc);
        }
        __syncthreads();
        if (tid == 0 && s_esc) atomicAdd(&job.ctl->escapes, (unsigned long long)s_esc);
    }
}

// ----------------------------------------------------------------------------
// decompress: same skeleton; size/validate pass then table expansion.
// ----------------------------------------------------------------------------
__device__ __forceinline__ int decode_size(const uint8_t *r, long long n, const uint8_t *explen,
                                           long long *m_out, long long *errpos, int *code,
                                           unsigned *esc) {
    long long m = 0;
    for (long long i = 0; i < n;) {
        unsigned b = r[i];
        if (b == 0x20) {
            if (i + 1 >= n) { *errpos = i; return E_TRUNC; }
            ++m;
            ++*esc;
            i += 2;
        } else {
            unsigned L = explen[b];
            if (!L) { *errpos = i; *code = (int)b; return E_UNKNOWN; }
            m += L;
            ++i;
        }
    }
    *m_out = m;
    return E_NONE;
}

__device__ __forceinline__ long long decode_fill(const uint8_t *r, long long n, const uint8_t *explen,
                                                 const uint16_t *expoff, const uint8_t *expflat,
                                                 uint8_t *o) {
    long long w = 0;
    for (long long i = 0; i < n;) {
        unsigned b = r[i];
        if (b == 0x20) {
            o[w++] = r[i + 1];
            i += 2;
        } else {
            unsigned L = explen[b];
            const uint8_t *e = expflat + expoff[b];
            for (unsigned k = 0; k < L; ++k) o[w + k] = e[k];
            w += L;
            ++i;
        }
    }
    return w;
}

// ============================================================================
// Byte-parallel decompress.  Each thread owns a fixed slice of the tile's
// compressed bytes (its CHUNK; the thread holding the tile end also takes
// the overhang of the last record) and walks it three times with a uniform
// trip count: (1) validate -- unknown codes and dangling escapes flag their
// record in a per-tile bitmap (rare atomics); (2) sum the output bytes of
// good records -> block scan -> the slice's output offset; (3) expand.
// The escape state at a slice start is the parity of the 0x20 run just
// before it (a 0x20 at an odd index of a run is a literal).  Records are
// framed by '\n' exactly as run_stream splits them (pipeline.py:49-74).
// ============================================================================
struct BpSmem {
    uint8_t *expflat;
    uint16_t *expoff;
    uint8_t *explen;
    uint8_t *win;
    uint8_t *out;
    unsigned *bad;   // bit per record ordinal of the tile
};

constexpr int BP_BADW = TILE / 32 + 2;

__host__ __device__ inline int bp_smem_bytes(int n_flat) {
    return align16(n_flat + 16) + align16(257 * 2) + 256 + align16(WIN + 16) + align16(DOUTCAP) +
           BP_BADW * 4;
}

__device__ inline BpSmem carve_bp(uint8_t *p, int n_flat) {
    BpSmem S;
    S.expflat = p; p += align16(n_flat + 16);
    S.expoff = reinterpret_cast<uint16_t *>(p); p += align16(257 * 2);
    S.explen = p; p += 256;
    S.win = p; p += align16(WIN + 16);
    S.out = p; p += align16(DOUTCAP);
    S.bad = reinterpret_cast<unsigned *>(p);
    return S;
}

// one compressed byte: window when resident, else HBM (long last record)
struct BpBytes {
    const uint8_t *win;
    const uint8_t *in;
    long long ws;
    int lim;  // window bytes [0, lim) are resident (incl. the EOF sentinel)
    __device__ __forceinline__ unsigned operator()(int p) const {
        return p < lim ? win[p] : in[ws + p];
    }
};

// One walk over a decompress slice.  MODE 0: validate (flag bad records);
// 1: count output bytes and escapes of good records; 2: expand to smem
// (staged) or HBM.  RES: every byte of the slice is in the smem window
// (bytes come 4 at a time from aligned words; p0 is word-aligned).
struct BpWalk {
    unsigned a_win, a_len, a_bad, a_off, a_flat, a_out;
    int p0, p1, tile_end, ord0;
    bool esc0, short_exp;
};

template <int MODE, bool RES>
__device__ __forceinline__ void bp_walk(const BpWalk &W, const BpSmem &S, const BpBytes &B,
                                        unsigned *bad, unsigned &sum, unsigned &nesc,
                                        uint8_t *o_glob, unsigned long long w) {
    int ord = W.ord0;
    unsigned esc = W.esc0;
    unsigned good = 0;
    if (MODE > 0 && ord >= 0) good = !((ldsw(W.a_bad + 4 * (ord >> 5)) >> (ord & 31)) & 1u);
    unsigned prev = W.p0 < W.p1 ? ldsb(W.a_win + W.p0 - 1) : 0u;
    unsigned word = 0;
    for (int p = W.p0; p < W.p1; ++p) {
        unsigned b;
        if (RES) {
            if (((p - W.p0) & 3) == 0) word = ldsw(W.a_win + p);  // p0 is 4-aligned
            b = word & 0xffu;
            word >>= 8;
        } else {
            b = B(p);
        }
        const unsigned start = (p < W.tile_end) & (prev == '\n');
        prev = b;
        ord += (int)start;
        esc &= start ^ 1u;
        if (MODE > 0 && start) good = !((ldsw(W.a_bad + 4 * (ord >> 5)) >> (ord & 31)) & 1u);
        const unsigned nl = b == '\n';
        const unsigned mark = (esc ^ 1u) & (nl ^ 1u) & (b == 0x20);
        const unsigned code = (esc ^ 1u) & (nl ^ 1u) & (mark ^ 1u);
        const unsigned L = ldsb(W.a_len + b);
        if (MODE == 0) {
            const unsigned err = (ord >= 0) & ((nl & esc) | (code & (L == 0)));
            if (err) atomicOr(&bad[ord >> 5], 1u << (ord & 31));
        } else {
            const unsigned add = code ? L : (mark ^ 1u);
            if (MODE == 1) {
                sum += good ? add : 0u;
                nesc += good & mark;
            } else if (good) {
                if (o_glob == nullptr) {
                    const unsigned ow = W.a_out + (unsigned)w;
                    if (!code) {
                        if (!mark) stsb(ow, b);  // literal or '\n'
                    } else {
                        const unsigned e = W.a_flat + ldsh(W.a_off + 2 * b);
                        if (W.short_exp) {
#pragma unroll
                            for (unsigned k = 0; k < 8; ++k)
                                if (k < L) stsb(ow + k, ldsb(e + k));
                        } else {
                            for (unsigned k = 0; k < L; ++k) stsb(ow + k, ldsb(e + k));
                        }
                    }
                } else {
                    if (!code) {
                        if (!mark) o_glob[w] = (uint8_t)b;
                    } else {
                        const uint8_t *e = S.expflat + S.expoff[b];
                        for (unsigned k = 0; k < L; ++k) o_glob[w + k] = e[k];
                    }
                }
                w += add;
            }
        }
        esc = mark;
    }
}

__global__ void __launch_bounds__(NT, 1) decompress_tiles_bp(Job job, Tables tb) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ unsigned long long s_tmp64[NWARP];
    __shared__ int s_tmp32[NWARP];
    __shared__ long long s_tile;
    __shared__ int s_last_end, s_first_start, s_nbad;
    __shared__ unsigned long long s_pre_out, s_pre_lines;
    __shared__ unsigned s_esc;

    const BpSmem S = carve_bp(smem, tb.n_flat);
    for (int k = threadIdx.x; k < tb.n_flat; k += NT) S.expflat[k] = tb.exp_flat[k];
    for (int k = threadIdx.x; k < 257; k += NT) S.expoff[k] = tb.exp_off[k];
    for (int k = threadIdx.x; k < 256; k += NT) S.explen[k] = tb.exp_len[k];
    const int tid = threadIdx.x;
    PhaseClock pc;
    pc.start();

    for (;;) {
        __syncthreads();
        pc.mark(job, 7);  // end of previous tile
        if (tid == 0) {
            s_tile = (long long)atomicAdd(&job.ctl->ticket, 1ull);
            s_nbad = 0;
            s_esc = 0;
            s_last_end = -1;
            s_first_start = 0x7fffffff;
        }
        __syncthreads();
        const long long t = s_tile;
        if (t >= job.n_tiles) break;
        const long long T0 = t * (long long)TILE;
        const int tile_len = (int)min((long long)TILE, job.n - T0);
        const long long ws = T0 - HEAD;
        const long long we = min(job.n, T0 + TILE + EXTRA);
        const int win_len = (int)(we - ws);
        const bool hits_eof = we == job.n;
        load_window(job.in, job.n, ws, align16(win_len), S.win);
        for (int k = tid; k < BP_BADW; k += NT) S.bad[k] = 0u;
        __syncthreads();
        if (tid == 0) S.win[win_len] = hits_eof ? '\n' : S.win[win_len];
        const int my_cnt = scan_starts(S.win, tile_len, 0, nullptr, 0, 0);
        int tile_lines;
        const int my_off = block_exscan<int>(my_cnt, s_tmp32, tile_lines);
        const int c0 = tid * CHUNK, c1 = min(c0 + CHUNK, tile_len);
        // the thread holding the tile end finishes the last record (overhang)
        const bool tail = c0 < tile_len && c1 == tile_len;
        if (tail && tile_lines > 0) {
            int e = HEAD + tile_len;
            // the last owned record ends at the first '\n' at or after the
            // tile end -- unless the tile's last byte is itself a '\n'
            if (S.win[HEAD + tile_len - 1] == '\n') {
                e = HEAD + tile_len - 1;
            } else {
                while (e < win_len && S.win[e] != '\n') ++e;
                if (e >= win_len && !hits_eof) {
                    long long g = ws + e;
                    while (g < job.n && job.in[g] != '\n') ++g;
                    e = (int)(g - ws);
                }
            }
            s_last_end = e;
        }
        __syncthreads();
        pc.mark(job, 0);  // ticket, load, start scan, last record end
        const int last_end = s_last_end;
        const BpBytes B{S.win, job.in, ws, hits_eof ? win_len + 1 : win_len};
        // my slice: [HEAD + c0, HEAD + c1), plus (tail) up to last_end inclusive
        const int p0 = HEAD + c0;
        const int p1 = tail ? last_end + 1 : HEAD + c1;
        const bool resident = last_end < (hits_eof ? win_len + 1 : win_len);
        // escape parity at the slice start
        bool esc0 = false;
        if (p0 < p1 && S.win[p0 - 1] != '\n') {
            int r = 0;
            while (p0 - 1 - r > 0 && S.win[p0 - 1 - r] == 0x20) ++r;
            esc0 = r & 1;
        }
        // Per-byte role, branch-free (selects + predicated stores):
        //   start : a record starts here (ord++, escape state reset)
        //   nl    : '\n' record end (outputs '\n' for a good record)
        //   lit   : escaped literal (outputs the byte)
        //   mark  : 0x20 escape marker (outputs nothing)
        //   code  : dictionary code (outputs explen bytes; explen 0 = error)
        // Non-resident tiles (last record longer than the window) read HBM
        // through B on the same path.
        const int tile_end = HEAD + tile_len;
        BpWalk W;
        W.a_win = sa(S.win);
        W.a_len = sa(S.explen);
        W.a_bad = sa(S.bad);
        W.a_off = sa(S.expoff);
        W.a_flat = sa(S.expflat);
        W.a_out = sa(S.out);
        W.p0 = p0;
        W.p1 = p1;
        W.tile_end = tile_end;
        W.ord0 = my_off - 1;
        W.esc0 = esc0;
        W.short_exp = tb.max_exp <= 8;
        unsigned dummy = 0, my_sum = 0, my_esc = 0;
        // ---- (1) validate ----
        if (resident) bp_walk<0, true>(W, S, B, S.bad, dummy, dummy, nullptr, 0);
        else bp_walk<0, false>(W, S, B, S.bad, dummy, dummy, nullptr, 0);
        __syncthreads();
        // ---- (2) output bytes of good records in my slice ----
        if (resident) bp_walk<1, true>(W, S, B, S.bad, my_sum, my_esc, nullptr, 0);
        else bp_walk<1, false>(W, S, B, S.bad, my_sum, my_esc, nullptr, 0);
        unsigned long long tile_out;
        const unsigned long long my_base = block_exscan<unsigned long long>(my_sum, s_tmp64, tile_out);
        if (my_esc) atomicAdd(&s_esc, my_esc);
        if (tid == 0) lookback_publish(job.ts, t, tile_out, (unsigned long long)tile_lines);
        const bool staged = resident && tile_out <= (unsigned long long)DOUTCAP;
        // ---- (3) expand: to smem now when staged, else to HBM after the look-back ----
        if (staged) bp_walk<2, true>(W, S, B, S.bad, dummy, dummy, nullptr, my_base);
        pc.mark(job, 3);  // thread 0's expand
        if (tid < 32) {
            unsigned long long po, pl;
            lookback_resolve(job.ts, t, tile_out, (unsigned long long)tile_lines, po, pl);
            if (tid == 0) {
                s_pre_out = po;
                s_pre_lines = pl;
            }
        }
        // bad records: count, and the stats/error details (rare, serial)
        {
            unsigned nb = 0;
            for (int k = tid; k < (tile_lines + 31) / 32; k += NT) nb += __popc(S.bad[k]);
            if (nb) atomicAdd(&s_nbad, (int)nb);
        }
        __syncthreads();
        pc.mark(job, 4);  // look-back + wait for the slowest expander
        const unsigned long long pre_out = s_pre_out;
        const bool fits = pre_out + tile_out <= (unsigned long long)job.out_cap;
        if (tid == 0) {
            const int nbad = s_nbad;
            atomicAdd(&job.ctl->total_out, tile_out);
            atomicAdd(&job.ctl->lines, (unsigned long long)(tile_lines - nbad));
            atomicAdd(&job.ctl->in_lines, (unsigned long long)tile_lines);
            if (!fits) atomicOr(&job.ctl->overflow, 1ull);
            unsigned long long esc_bad = 0;
            if (nbad) {
                if (job.lenient) atomicAdd(&job.ctl->skipped, (unsigned long long)nbad);
                // walk the bad records from the pristine input: escapes
                // before the error count too (numba_impl.py:99-101)
                int ord = -1, first_bad = -1;
                for (long long x = T0; x < T0 + tile_len; ++x) {
                    if (!(x == 0 || job.in[x - 1] == '\n')) continue;
                    ++ord;
                    if (!((S.bad[ord >> 5] >> (ord & 31)) & 1u)) continue;
                    long long ge = x;
                    while (ge < job.n && job.in[ge] != '\n') ++ge;
                    long long m = 0, ep = -1;
                    int code = 0;
                    unsigned e2 = 0;
                    const int kind = decode_size(job.in + x, ge - x, S.explen, &m, &ep, &code, &e2);
                    esc_bad += e2;
                    if (first_bad < 0) {
                        first_bad = ord;
                        if (!job.lenient) {
                            TileErr e;
                            e.kind = kind;
                            e.code = code;
                            e.offset = ep;
                            e.ids[0] = e.ids[1] = 0;
                            job.terr[t] = e;
                            __threadfence();
                            atomicMin(&job.ctl->err_key, ((s_pre_lines + (unsigned long long)ord) << 24) |
                                                             (unsigned long long)(t & 0xffffff));
                        }
                    }
                }
            }
            if (s_esc + esc_bad) atomicAdd(&job.ctl->escapes, (unsigned long long)s_esc + esc_bad);
        }
        pc.mark(job, 5);  // stats
        if (!fits) continue;
        if (staged) store_out(job.out + pre_out, S.out, (int)tile_out);
        else if (resident) bp_walk<2, true>(W, S, B, S.bad, dummy, dummy, job.out, pre_out + my_base);
        else bp_walk<2, false>(W, S, B, S.bad, dummy, dummy, job.out, pre_out + my_base);
        pc.mark(job, 6);  // store
    }
}

// ----------------------------------------------------------------------------
// parity-shim kernels: reference kernel layouts, one thread per line, HBM
// ----------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(256) batch_compress(const uint8_t *flat, const long long *starts,
                                                      long long n_lines, uint8_t *out,
                                                      long long *out_lens, uint8_t *dec,
                                                      unsigned long long *escapes, Tables tb) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t *dfa = reinterpret_cast<uint16_t *>(smem);
    uint8_t *codes = smem + align16(tb.n_states * NCOL * 2);
    __shared__ uint8_t explen[256];
    if (W) {
        for (int k = threadIdx.x; k < tb.n_states * NCOL; k += blockDim.x) dfa[k] = tb.dfa[k];
        for (int k = threadIdx.x; k < tb.n_states * FAST_W; k += blockDim.x) codes[k] = tb.codes[k];
    }
    for (int k = threadIdx.x; k < 256; k += blockDim.x) explen[k] = tb.exp_len[k];
    __syncthreads();
    long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (li >= n_lines) return;
    const long long s0 = starts[li], n = starts[li + 1] - s0;
    const uint8_t *s = flat + s0;
    uint8_t *d = dec + s0 + li;  // n+1 decision slots per line
    if (n == 0) { out_lens[li] = 0; return; }
    long long cost;
    if constexpr (W > 0) {
        if (n < (1ll << 24)) {
            cost = dp_fast<W>(s, (int)n, d, dfa, codes);
        } else {
            long long ring[128];
            cost = dp_generic(s, n, d, tb, ring);
        }
    } else {
        long long ring[128];
        cost = dp_generic(s, n, d, tb, ring);
    }
    uint8_t *o = out + 2 * s0;
    long long w = 0;
    unsigned esc = 0;
    for (long long i = 0; i < n;) {
        uint8_t c = d[i];
        if (c == D_ESC) {
            o[w++] = 0x20;
            o[w++] = s[i];
            ++esc;
            ++i;
        } else {
            o[w++] = c;
            i += explen[c];
        }
    }
    out_lens[li] = cost;
    if (esc) atomicAdd(escapes, (unsigned long long)esc);
}

__global__ void batch_decode_sizes(const uint8_t *flat, const long long *starts, long long n_lines,
                                   long long *out_lens, int8_t *status, long long *errpos,
                                   unsigned long long *tot, Tables tb) {
    __shared__ uint8_t explen[256];
    for (int k = threadIdx.x; k < 256; k += blockDim.x) explen[k] = tb.exp_len[k];
    __syncthreads();
    long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (li >= n_lines) return;
    const long long s0 = starts[li];
    long long m = 0, ep = -1;
    int code = 0;
    unsigned esc = 0;
    int st = decode_size(flat + s0, starts[li + 1] - s0, explen, &m, &ep, &code, &esc);
    // reference status codes: 1 unknown code, 2 truncated escape
    status[li] = (int8_t)(st == E_NONE ? 0 : (st == E_UNKNOWN ? 1 : 2));
    errpos[li] = st == E_NONE ? -1 : ep;
    out_lens[li] = st == E_NONE ? m : 0;
    if (st == E_NONE && m) atomicAdd(&tot[0], (unsigned long long)m);
    if (esc) atomicAdd(&tot[1], (unsigned long long)esc);
}

__global__ void batch_decode_fill(const uint8_t *flat, const long long *starts, long long n_lines,
                                  const int8_t *status, uint8_t *out, const long long *out_starts,
                                  Tables tb) {
    __shared__ uint8_t explen[256];
    __shared__ uint16_t expoff[257];
    for (int k = threadIdx.x; k < 256; k += blockDim.x) explen[k] = tb.exp_len[k];
    for (int k = threadIdx.x; k < 257; k += blockDim.x) expoff[k] = tb.exp_off[k];
    __syncthreads();
    long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (li >= n_lines || status[li] != 0) return;
    const long long s0 = starts[li];
    decode_fill(flat + s0, starts[li + 1] - s0, explen, expoff, tb.exp_flat, out + out_starts[li]);
}

__global__ void batch_preprocess(const uint8_t *flat, const long long *starts, long long n_lines,
                                 uint8_t *out, long long *out_lens, int8_t *status,
                                 long long *err_off, unsigned long long *err_ids, uint8_t *marks) {
    long long li = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (li >= n_lines) return;
    const long long s0 = starts[li], n = starts[li + 1] - s0;
    uint8_t *o = out + 3 * s0 + 3 * li;
    int nl2 = 0, eoff = -1;
    unsigned long long ids[2] = {0, 0};
    int k = preprocess_line(flat + s0, (int)n, marks + s0 + li, o, &nl2, &eoff, ids, false);
    status[li] = (int8_t)k;
    out_lens[li] = k == E_NONE ? nl2 : 0;
    err_off[li] = eoff;
    err_ids[2 * li] = ids[0];
    err_ids[2 * li + 1] = ids[1];
}

}  // namespace zs
