// zs_fx.cuh -- streaming decompress (the decode hot path).
//
// Decode is byte-local: every compressed byte maps to its expansion
// (numba_impl.py:115-139), '\n' to itself, a 0x20 mark to nothing and the
// byte after a mark to itself.  Records only matter for errors, so the
// streaming path ignores them.  A buffer is cut into 8 KB tiles; each thread
// of a 256-thread CTA owns 32 consecutive compressed bytes.  Three launches:
//
//   fx_count  one table lookup per byte sums the output bytes of each
//             thread's slice; a block scan gives every thread its u16 offset
//             inside the tile; tile totals, record and escape counts, and a
//             per-tile "has escapes" flag go to HBM.  Unknown codes and
//             dangling escapes (numba_impl.py:94-109) set Ctl.overflow bit 2:
//             the host then re-runs the buffer through the record-aware
//             kernel (decompress_tiles_bp), which owns the error semantics.
//   fx_scan   one CTA: exclusive scan of the tile totals -> tile offsets.
//   fx_emit   each thread appends its expansions to a 64-bit accumulator and
//             stores whole 8-byte words into a zeroed smem staging tile (the
//             two words it shares with its neighbours via atomic OR); the
//             tile then leaves with aligned 16-byte stores.
//
// Tables (built on the host from the reference decode tables,
// dictionary.py:112-129), replicated per bank so lookups never conflict:
//   count: u32 [code][32 lanes] = len | invalid << 10 | mark << 16 | nl << 22
//   emit : u64 [code][16 lanes] = expansion bytes 0-6 | (8 * len) << 56
//          (WIDE, longest expansion 8..15: a second table, bytes 0-7 in the
//          first and bytes 8-14 | (8 * len) << 56 in the second)
// Serves dictionaries whose longest expansion is <= 15 bytes (default: 6).
#pragma once
#include "zs_device.cuh"

namespace zs {

constexpr int FX_NT = 256;               // threads per CTA
constexpr int FX_B = 32;                 // compressed bytes per thread per tile
constexpr int FX_TILE = FX_NT * FX_B;    // 8 KB of compressed input per tile
constexpr int FX_STAGE = 24576;          // emit staging bytes (tile output + 16 alignment)
constexpr int FX_CNT_SMEM = 0;   // static shared only
constexpr int FX_ETAB = 256 * 16 * 8;  // one replicated emit table
__host__ __device__ constexpr int fx_emit_smem(bool wide) { return (wide ? 2 : 1) * FX_ETAB + FX_STAGE; }
constexpr unsigned long long FX_BYTES = (1ull << 56) - 1;

// per-slot scratch layout (device): tile totals, tile offsets, tile flags,
// per-thread offsets inside the tile
struct FxScratch {
    unsigned *tsum;            // [n_tiles] output bytes of the tile
    unsigned long long *toff;  // [n_tiles] exclusive prefix
    uint8_t *tflag;            // [n_tiles] bit 0: escapes in the tile
    unsigned *off32;           // [n_tiles * FX_NT]
};

inline size_t fx_scratch_bytes(long long nt) {
    return (size_t)nt * (4 + 8 + 1 + 4 * FX_NT) + 64;
}

inline FxScratch fx_carve(void *p, long long nt) {
    FxScratch s;
    uint8_t *q = reinterpret_cast<uint8_t *>(p);
    s.toff = reinterpret_cast<unsigned long long *>(q); q += 8 * nt;
    s.tsum = reinterpret_cast<unsigned *>(q); q += 4 * nt;
    s.off32 = reinterpret_cast<unsigned *>(q); q += 4 * nt * FX_NT;
    s.tflag = q;
    return s;
}

// host: table entries per code (a '\n' is a 1-byte code of itself)
inline unsigned fx_count_entry(int b, const uint8_t *exp_len) {
    if (b == '\n') return 1u | (1u << 22);
    if (b == 0x20) return 1u << 16;
    return exp_len[b] ? (unsigned)exp_len[b] : (1u << 10);
}
// narrow entry (longest expansion <= 7), or the two WIDE entries (<= 15)
inline unsigned long long fx_emit_entry(int b, const uint8_t *exp_len, const uint16_t *exp_off,
                                        const uint8_t *exp_flat, bool wide = false, int part = 0) {
    const int L = b == '\n' ? 1 : exp_len[b];
    if (b == 0x20 || L == 0) return 0;
    auto byte = [&](int k) -> unsigned long long { return b == '\n' ? '\n' : exp_flat[exp_off[b] + k]; };
    unsigned long long e = 0;
    if (!wide) {
        e = (unsigned long long)(8 * L) << 56;
        for (int k = 0; k < L && k < 7; ++k) e |= byte(k) << (8 * k);
    } else if (part == 0) {
        for (int k = 0; k < L && k < 8; ++k) e |= byte(k) << (8 * k);
    } else {
        e = (unsigned long long)(8 * L) << 56;
        for (int k = 8; k < L && k < 15; ++k) e |= byte(k) << (8 * (k - 8));
    }
    return e;
}

__device__ __forceinline__ unsigned fx_word(const uint4 &a, const uint4 &b, int k) {
    return k == 0 ? a.x : k == 1 ? a.y : k == 2 ? a.z : k == 3 ? a.w
         : k == 4 ? b.x : k == 5 ? b.y : k == 6 ? b.z : b.w;
}

__device__ __forceinline__ unsigned long long lds64(unsigned a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds32(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(unsigned a, unsigned long long v) {
    asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void red_or64(unsigned a, unsigned long long v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"((unsigned)v) : "memory");
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a + 4), "r"((unsigned)(v >> 32)) : "memory");
}

// parity of the 0x20 run ending just before position p: 1 = p is a literal
__device__ __forceinline__ unsigned fx_escaped(const uint8_t *in, long long p) {
    long long r = 0;
    while (p - 1 - r >= 0 && in[p - 1 - r] == 0x20) ++r;
    return (unsigned)(r & 1);
}

// load the 32-byte slice at c0 (cnt valid bytes; the rest read as 0)
template <bool ALIGNED, bool KEEP = false>
__device__ __forceinline__ void fx_load(const uint8_t *in, long long c0, int cnt, uint4 &va, uint4 &vb) {
    if (ALIGNED && cnt == FX_B) {
        const uint4 *src = reinterpret_cast<const uint4 *>(in + c0);
        va = KEEP ? __ldg(src) : __ldcs(src);
        vb = KEEP ? __ldg(src + 1) : __ldcs(src + 1);
    } else {
        unsigned w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < FX_B; ++k)
            if (k < cnt) w[k >> 2] |= (unsigned)in[c0 + k] << (8 * (k & 3));
        va = make_uint4(w[0], w[1], w[2], w[3]);
        vb = make_uint4(w[4], w[5], w[6], w[7]);
    }
}

// exact walk of one slice with escapes: output bytes, records, literals, bad
__device__ __forceinline__ void fx_walk_esc(const uint4 &va, const uint4 &vb, int cnt, unsigned esc,
                                            const uint8_t *explen, unsigned &sum, unsigned &nl,
                                            unsigned &nesc, unsigned &bad, unsigned &esc_out) {
    sum = nl = nesc = bad = 0;
    for (int k = 0; k < cnt; ++k) {
        const unsigned b = (fx_word(va, vb, k >> 2) >> (8 * (k & 3))) & 0xffu;
        const unsigned lit = esc;
        const unsigned L = explen[b];
        if (lit) {
            bad |= b == '\n';
            sum += 1;
            nesc += 1;
            esc = 0;
        } else if (b == 0x20) {
            esc = 1;
        } else if (b == '\n') {
            sum += 1;
            nl += 1;
        } else {
            bad |= L == 0;
            sum += L;
        }
    }
    esc_out = esc;
}

// ---------------------------------------------------------------------------
// fx_count: per-thread output bytes -> u16 tile offsets; tile totals/flags
// ---------------------------------------------------------------------------

// sum of the count-table entries of the slice's bytes (FULL: all 32 valid)
template <bool FULL>
__device__ __forceinline__ unsigned fx_count_slice(const unsigned (*tab)[32], int lane, const uint4 &va,
                                                   const uint4 &vb, int cnt) {
    unsigned acc = 0;
#pragma unroll
    for (int k = 0; k < FX_B; ++k) {
        if (FULL || k < cnt) {
            const unsigned b = (fx_word(va, vb, k >> 2) >> (8 * (k & 3))) & 0xffu;
            acc += tab[b][lane];
        }
    }
    return acc;
}

template <bool ALIGNED>
__global__ void __launch_bounds__(FX_NT) fx_count(Job job, const unsigned *ctab, FxScratch sc) {
    __shared__ unsigned s_tab[256][32];  // replicated per lane: conflict-free
    __shared__ unsigned long long s_tmp64[FX_NT / 32];
    __shared__ uint8_t s_explen[256];
    __shared__ unsigned s_flag;
    for (int k = threadIdx.x; k < 256 * 32; k += FX_NT) s_tab[k >> 5][k & 31] = ctab[k >> 5];
    for (int k = threadIdx.x; k < 256; k += FX_NT) s_explen[k] = (uint8_t)(ctab[k] & 0xffu);
    const int tid = threadIdx.x, lane = tid & 31;
    const bool ends_nl = job.n > 0 && job.in[job.n - 1] == '\n';
    unsigned long long my_nl = 0, my_esc = 0;
    unsigned any_bad = 0;
    for (long long t = blockIdx.x; t < job.n_tiles; t += gridDim.x) {
        __syncthreads();  // s_flag / s_tmp64 reuse
        if (tid == 0) s_flag = 0;
        const long long c0 = t * (long long)FX_TILE + (long long)tid * FX_B;
        const int cnt = (int)max(0ll, min((long long)FX_B, job.n - c0));
        uint4 va, vb;
        fx_load<ALIGNED, true>(job.in, c0, cnt, va, vb);  // cached: fx_emit reads it again
        const unsigned acc = cnt == FX_B ? fx_count_slice<true>(s_tab, lane, va, vb, cnt)
                                         : fx_count_slice<false>(s_tab, lane, va, vb, cnt);
        unsigned sum = acc & 0x3ffu, bad = (acc >> 10) & 0x3fu, marks = (acc >> 16) & 0x3fu;
        unsigned nl = (acc >> 22) & 0x3fu, nesc = 0;
        // escapes: the byte before the slice, or marks inside it -> exact walk
        const unsigned prev = __shfl_up_sync(0xffffffffu, vb.w >> 24, 1);
        unsigned esc0 = 0;
        if (cnt > 0 && c0 > 0) {
            const unsigned pb = lane ? prev : job.in[c0 - 1];
            if (pb == 0x20) esc0 = fx_escaped(job.in, c0);
        }
        __syncthreads();
        if (marks | esc0) {
            unsigned esc_out;
            fx_walk_esc(va, vb, cnt, esc0, s_explen, sum, nl, nesc, bad, esc_out);
            if (cnt > 0 && c0 + cnt == job.n && esc_out) bad = 1;  // dangling escape at EOF
            s_flag = 1;
        }
        if (cnt > 0 && c0 + cnt == job.n && !ends_nl) {  // virtual '\n' closing the last record
            sum += 1;
            nl += 1;
        }
        any_bad |= bad;
        my_nl += nl;
        my_esc += nesc;
        unsigned long long tot;
        const unsigned long long off = block_exscan_n<unsigned long long, FX_NT>(sum, s_tmp64, tot);
        sc.off32[t * FX_NT + tid] = (unsigned)off;
        if (tid == 0) {
            sc.tsum[t] = (unsigned)tot;
            sc.tflag[t] = (uint8_t)(s_flag | (tot + 16 > (unsigned long long)FX_STAGE ? 2u : 0u));
        }
    }
    // per-CTA totals
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        my_nl += __shfl_xor_sync(0xffffffffu, my_nl, o);
        my_esc += __shfl_xor_sync(0xffffffffu, my_esc, o);
    }
    any_bad = __any_sync(0xffffffffu, any_bad != 0);
    if (lane == 0) {
        if (my_nl) {
            atomicAdd(&job.ctl->lines, my_nl);
            atomicAdd(&job.ctl->in_lines, my_nl);
        }
        if (my_esc) atomicAdd(&job.ctl->escapes, my_esc);
        if (any_bad) atomicOr(&job.ctl->overflow, 4ull);
    }
}

// ---------------------------------------------------------------------------
// fx_scan: one CTA of 1024 threads, exclusive scan of the tile totals
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) fx_scan(Job job, FxScratch sc) {
    // each thread owns a contiguous run of tiles: one pass of loads, one block scan
    __shared__ unsigned long long s_w[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long nt = job.n_tiles;
    const long long per = (nt + 1023) / 1024;
    const long long t0 = min(nt, tid * per), t1 = min(nt, t0 + per);
    unsigned long long sum = 0;
    for (long long t = t0; t < t1; ++t) sum += sc.tsum[t];
    unsigned long long x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    if (wid == 0) {
        unsigned long long w = s_w[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_w[lane] = w;
    }
    __syncthreads();
    unsigned long long run = (wid ? s_w[wid - 1] : 0ull) + x - sum;
    for (long long t = t0; t < t1; ++t) {
        sc.toff[t] = run;
        run += sc.tsum[t];
    }
    if (tid == 0) {
        const unsigned long long total = s_w[31];
        job.ctl->total_out = total;
        if (total > (unsigned long long)job.out_cap) atomicOr(&job.ctl->overflow, 1ull);
    }
}

// ---------------------------------------------------------------------------
// fx_emit: expansions -> staging -> aligned 16-byte stores
// ---------------------------------------------------------------------------

// Append one expansion x (len8 = 8 * its length, <= 56) to the accumulator:
// lo holds sh/8 pending bytes destined for the smem word at `a`; a whole word
// leaves with one 8-byte store.  FIRST: the slice's first word is shared
// with the previous slice (atomic OR into the zeroed staging).
struct FxAcc {
    unsigned long long lo;
    unsigned sh;
    unsigned a;
    bool first;
    template <bool FIRST>
    __device__ __forceinline__ void put(unsigned long long x, unsigned len8) {
        const unsigned long long spill = x >> ((64u - sh) & 63u);  // used only on a flush (sh > 0)
        lo |= x << sh;
        sh += len8;
        const bool f = sh >= 64u;
        if (FIRST) {
            if (f) {
                if (first) red_or64(a, lo);
                else sts64(a, lo);
            }
            first = first && !f;
        } else {
            if (f) sts64(a, lo);
        }
        a += f ? 8u : 0u;
        lo = f ? spill : lo;
        sh -= f ? 64u : 0u;
    }
    // up to 8 bytes (len8 <= 64); a full 8-byte word is legal, so the spill
    // must be 0 when nothing was pending
    __device__ __forceinline__ void put8(unsigned long long x, unsigned len8) {
        const unsigned long long spill = sh ? x >> (64u - sh) : 0ull;
        lo |= x << sh;
        sh += len8;
        const bool f = sh >= 64u;
        if (f) {
            if (first) red_or64(a, lo);
            else sts64(a, lo);
        }
        first = first && !f;
        a += f ? 8u : 0u;
        lo = f ? spill : lo;
        sh -= f ? 64u : 0u;
    }
    __device__ __forceinline__ void finish() {
        if (sh) red_or64(a, lo);
    }
};

__device__ __forceinline__ unsigned long long fx_etab(const unsigned long long (*tab)[16], int lane, unsigned b) {
    return tab[b][lane & 15];
}

// clean slice (no escapes), FULL = all 32 bytes valid.  Every code emits >= 1
// byte, so the first (shared) word is complete within the first 8 codes.
template <bool FULL>
__device__ __forceinline__ void fx_emit_clean(FxAcc &acc, const unsigned long long (*tab)[16], int lane,
                                              const uint4 &va, const uint4 &vb, int cnt) {
#pragma unroll
    for (int k = 0; k < FX_B; ++k) {
        if (FULL || k < cnt) {
            const unsigned b = (fx_word(va, vb, k >> 2) >> (8 * (k & 3))) & 0xffu;
            const unsigned long long e = fx_etab(tab, lane, b);
            const unsigned long long x = e & FX_BYTES;
            const unsigned len8 = (unsigned)(e >> 56);
            if (k < 8 || !FULL) acc.put<true>(x, len8);
            else acc.put<false>(x, len8);
        }
    }
}

template <bool ALIGNED, bool WIDE>
__global__ void __launch_bounds__(FX_NT) fx_emit(Job job, const unsigned long long *etab, FxScratch sc) {
    extern __shared__ __align__(16) uint8_t fsm[];  // emit table(s), then the staging tile
    auto s_tab = reinterpret_cast<unsigned long long (*)[16]>(fsm);        // replicated per half-warp lane
    auto s_tabh = reinterpret_cast<unsigned long long (*)[16]>(fsm + FX_ETAB);  // WIDE: bytes 8-14 | len
    uint8_t *stage = fsm + (WIDE ? 2 : 1) * FX_ETAB;
    for (int k = threadIdx.x; k < 256 * 16; k += FX_NT) s_tab[k >> 4][k & 15] = etab[k >> 4];
    if (WIDE)
        for (int k = threadIdx.x; k < 256 * 16; k += FX_NT) s_tabh[k >> 4][k & 15] = etab[256 + (k >> 4)];
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned a_stage = sa(stage);
    const bool ends_nl = job.n > 0 && job.in[job.n - 1] == '\n';

    // tiles from the end: the input fx_count read last is the one still in L2
    long long t = job.n_tiles - 1 - blockIdx.x;
    uint4 na = make_uint4(0, 0, 0, 0), nb4 = na;
    if (t >= 0) {
        const long long c0 = t * (long long)FX_TILE + (long long)tid * FX_B;
        fx_load<ALIGNED>(job.in, c0, (int)max(0ll, min((long long)FX_B, job.n - c0)), na, nb4);
    }
    for (; t >= 0; t -= gridDim.x) {
        const long long c0 = t * (long long)FX_TILE + (long long)tid * FX_B;
        const int cnt = (int)max(0ll, min((long long)FX_B, job.n - c0));
        const uint4 va = na, vb = nb4;
        // prefetch the next tile's slice
        const long long tn = t - gridDim.x;
        if (tn >= 0) {
            const long long cn = tn * (long long)FX_TILE + (long long)tid * FX_B;
            fx_load<ALIGNED>(job.in, cn, (int)max(0ll, min((long long)FX_B, job.n - cn)), na, nb4);
        }
        const unsigned long long tbase = sc.toff[t];
        const unsigned tsum = sc.tsum[t];
        const unsigned flag = sc.tflag[t];
        const unsigned my_off = sc.off32[t * FX_NT + tid];
        const bool eof_nl = cnt > 0 && c0 + cnt == job.n && !ends_nl;
        if (tsum == 0) continue;
        if (tbase + tsum > (unsigned long long)job.out_cap) continue;  // fx_scan set overflow bit 0
        const bool staged = !(flag & 2u);
        const int shift = (int)(tbase & 15);  // stage[shift + j] <-> out[tbase + j]
        if (staged) {
            __syncthreads();  // previous tile's copy-out is done
            const int words = (shift + (int)tsum + 15) >> 4;
            for (int k = tid; k < words; k += FX_NT)
                asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a_stage + 16u * k), "r"(0u)
                             : "memory");
            __syncthreads();
        }
        if (cnt > 0) {
            unsigned esc = 0;
            if (flag & 1u) {
                const unsigned prev = c0 > 0 ? job.in[c0 - 1] : 0u;
                if (prev == 0x20) esc = fx_escaped(job.in, c0);
            }
            if (staged) {
                const unsigned o = (unsigned)shift + my_off;
                FxAcc acc{0ull, 8u * (o & 7u), a_stage + (o & ~7u), true};
                if (WIDE) {
                    for (int k = 0; k < cnt; ++k) {
                        const unsigned b = (fx_word(va, vb, k >> 2) >> (8 * (k & 3))) & 0xffu;
                        if (esc) {
                            acc.put8(b, 8u);
                            esc = 0;
                        } else if ((flag & 1u) && b == 0x20) {
                            esc = 1;
                        } else {
                            const unsigned long long e0 = s_tab[b][lane & 15], e1 = s_tabh[b][lane & 15];
                            const unsigned len8 = (unsigned)(e1 >> 56);
                            acc.put8(e0, min(len8, 64u));
                            if (len8 > 64u) acc.put8(e1 & FX_BYTES, len8 - 64u);
                        }
                    }
                } else if (!(flag & 1u)) {
                    if (cnt == FX_B) fx_emit_clean<true>(acc, s_tab, lane, va, vb, cnt);
                    else fx_emit_clean<false>(acc, s_tab, lane, va, vb, cnt);
                } else {
                    for (int k = 0; k < cnt; ++k) {
                        const unsigned b = (fx_word(va, vb, k >> 2) >> (8 * (k & 3))) & 0xffu;
                        const unsigned long long e = fx_etab(s_tab, lane, b);
                        if (esc) {
                            acc.put<true>(b, 8u);
                            esc = 0;
                        } else if (b == 0x20) {
                            esc = 1;
                        } else {
                            acc.put<true>(e & FX_BYTES, (unsigned)(e >> 56));
                        }
                    }
                }
                if (eof_nl) acc.put<true>('\n', 8u);
                acc.finish();
            } else {
                // tile output larger than the staging buffer: bytes straight to HBM
                uint8_t *o = job.out + tbase + my_off;
                for (int k = 0; k < cnt; ++k) {
                    const unsigned b = (fx_word(va, vb, k >> 2) >> (8 * (k & 3))) & 0xffu;
                    const unsigned long long e = fx_etab(s_tab, lane, b);
                    if (esc) {
                        *o++ = (uint8_t)b;
                        esc = 0;
                    } else if (b == 0x20) {
                        esc = 1;
                    } else if (WIDE) {
                        const unsigned long long e1 = s_tabh[b][lane & 15];
                        const unsigned L = (unsigned)(e1 >> 56) >> 3;
                        for (unsigned j = 0; j < L; ++j) o[j] = (uint8_t)((j < 8 ? e : e1) >> (8 * (j & 7)));
                        o += L;
                    } else {
                        const unsigned L = (unsigned)(e >> 56) >> 3;
                        for (unsigned j = 0; j < L; ++j) o[j] = (uint8_t)(e >> (8 * j));
                        o += L;
                    }
                }
                if (eof_nl) *o++ = '\n';
            }
        }
        if (staged) {
            __syncthreads();
            // aligned 16-byte chunks [g0, g1) of the output; partial ends bytewise
            const unsigned long long lo = tbase, hi = tbase + tsum;
            const unsigned long long g0 = (lo + 15) & ~15ull, g1 = hi & ~15ull;
            const uint4 *s4 = reinterpret_cast<const uint4 *>(stage);
            if (g0 < g1) {
                const int n16 = (int)((g1 - g0) >> 4);
                const int s0 = (int)((g0 - (lo & ~15ull)) >> 4);
                uint4 *d4 = reinterpret_cast<uint4 *>(job.out + g0);
                for (int k = tid; k < n16; k += FX_NT) __stcs(d4 + k, s4[s0 + k]);
                if (tid < 32) {
                    for (unsigned long long g = lo + tid; g < g0; g += 32) job.out[g] = stage[shift + (g - lo)];
                } else if (tid < 64) {
                    for (unsigned long long g = g1 + (tid - 32); g < hi; g += 32)
                        job.out[g] = stage[shift + (g - lo)];
                }
            } else if (tid < 32) {
                for (unsigned long long g = lo + tid; g < hi; g += 32) job.out[g] = stage[shift + (g - lo)];
            }
        }
    }
}

}  // namespace zs
