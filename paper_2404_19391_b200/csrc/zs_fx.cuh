// zs_fx.cuh -- streaming decompress kernel (the decode hot path).
//
// Decode is byte-local: every compressed byte maps to its expansion
// (numba_impl.py:115-139), '\n' to itself, a 0x20 mark to nothing and the
// byte after a mark to itself.  Records only matter for errors, so this
// kernel ignores them: each thread owns 32 consecutive compressed bytes,
//   pass 1  sums the output bytes of its bytes (one table lookup each),
//   scan    block exclusive scan + decoupled look-back over tiles,
//   pass 2  appends the expansions to a 64-bit accumulator and writes
//           aligned 8-byte words straight to HBM (head/tail bytes singly).
// Any unknown code or dangling escape (numba_impl.py:94-109) sets
// Ctl.overflow bit 2 and the host re-runs the buffer through the
// record-aware kernel (decompress_tiles_bp), which owns error semantics.
//
// Expansion table: u64 per code, bytes 0-6 = expansion, bits 56-59 = length,
// bit 60 = invalid code, bit 61 = escape mark, bit 62 = record end.  It is
// replicated 16x ([code][lane & 15]) so a warp's 64-bit lookups (two
// half-warp wavefronts) never conflict on a bank.  Serves dictionaries whose
// longest expansion is <= 7 bytes (the default one: 6).
#pragma once
#include "zs_device.cuh"

namespace zs {

constexpr int FX_NT = 256;               // threads per CTA
constexpr int FX_B = 32;                 // compressed bytes per thread per tile
constexpr int FX_TILE = FX_NT * FX_B;    // 8 KB of compressed input per tile
constexpr int FX_REP = 16;               // table replicas
constexpr unsigned long long FX_LEN_SHIFT = 56;
constexpr unsigned long long FX_INVALID = 1ull << 60;
constexpr unsigned long long FX_MARK = 1ull << 61;
constexpr unsigned long long FX_NL = 1ull << 62;
constexpr unsigned long long FX_BYTES = (1ull << 56) - 1;
constexpr int FX_SMEM = 256 * FX_REP * 8;

// host: one table entry per code from the decode tables (dictionary.py:112-129)
inline unsigned long long fx_entry(int b, const uint8_t *exp_len, const uint16_t *exp_off,
                                   const uint8_t *exp_flat) {
    if (b == '\n') return (unsigned long long)'\n' | (1ull << FX_LEN_SHIFT) | FX_NL;
    if (b == 0x20) return FX_MARK;
    const int L = exp_len[b];
    if (L == 0) return FX_INVALID;
    unsigned long long e = (unsigned long long)L << FX_LEN_SHIFT;
    for (int k = 0; k < L && k < 7; ++k) e |= (unsigned long long)exp_flat[exp_off[b] + k] << (8 * k);
    return e;
}

__device__ __forceinline__ unsigned fx_byte(const uint4 &a, const uint4 &b, int k) {
    const unsigned w = k < 4 ? a.x : k < 8 ? a.y : k < 12 ? a.z : k < 16 ? a.w
                     : k < 20 ? b.x : k < 24 ? b.y : k < 28 ? b.z : b.w;
    return (w >> (8 * (k & 3))) & 0xffu;
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

// length of the 0x20 run ending just before position p (within [0, p))
__device__ __forceinline__ bool fx_escaped(const uint8_t *in, long long p) {
    long long r = 0;
    while (p - 1 - r >= 0 && in[p - 1 - r] == 0x20) ++r;
    return r & 1;
}

// Writes `len` (<= 7) bytes of x at global byte address o, byte by byte.
__device__ __forceinline__ void fx_put_bytes(uint8_t *o, unsigned long long x, int from, int to) {
    for (int k = from; k < to; ++k) o[k] = (uint8_t)(x >> (8 * k));
}

template <bool ALIGNED>
__global__ void __launch_bounds__(FX_NT) decompress_fx(Job job, const unsigned long long *tab) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ unsigned long long s_tmp64[FX_NT / 32];
    __shared__ unsigned s_red[3][FX_NT / 32];
    __shared__ long long s_tile;
    __shared__ unsigned long long s_pre_out;

    unsigned long long *stab = reinterpret_cast<unsigned long long *>(smem);
    for (int k = threadIdx.x; k < 256 * FX_REP; k += FX_NT) stab[k] = tab[k >> 4];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned a_tab = sa(stab) + 8u * (lane & (FX_REP - 1));
    const bool ends_nl = job.n > 0 && job.in[job.n - 1] == '\n';

    for (;;) {
        if (tid == 0) s_tile = (long long)atomicAdd(&job.ctl->ticket, 1ull);
        __syncthreads();
        const long long t = s_tile;
        if (t >= job.n_tiles) break;
        const long long c0 = t * (long long)FX_TILE + (long long)tid * FX_B;
        const int cnt = (int)max(0ll, min((long long)FX_B, job.n - c0));
        uint4 va = make_uint4(0, 0, 0, 0), vb = va;
        if (cnt == FX_B && ALIGNED) {
            const uint4 *src = reinterpret_cast<const uint4 *>(job.in + c0);
            va = __ldcs(src);
            vb = __ldcs(src + 1);
        } else if (cnt > 0) {
            unsigned w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int k = 0; k < cnt; ++k) w[k >> 2] |= (unsigned)job.in[c0 + k] << (8 * (k & 3));
            va = make_uint4(w[0], w[1], w[2], w[3]);
            vb = make_uint4(w[4], w[5], w[6], w[7]);
        }
        // escape state at the chunk start: parity of the 0x20 run before it
        const unsigned prev = __shfl_up_sync(0xffffffffu, vb.w >> 24, 1);
        bool esc0 = false;
        if (cnt > 0 && c0 > 0) {
            const unsigned pb = lane ? prev : job.in[c0 - 1];
            if (pb == 0x20) esc0 = fx_escaped(job.in, c0);
        }
        // the virtual '\n' closing a final record without one
        const bool eof_nl = cnt > 0 && c0 + cnt == job.n && !ends_nl;

        // ---- pass 1: output bytes, records, escapes, errors ----
        unsigned sum = 0, nl = 0, nesc = 0, bad = 0;
        bool esc = esc0;
#pragma unroll
        for (int k = 0; k < FX_B; ++k) {
            if (k < cnt) {
                const unsigned b = fx_byte(va, vb, k);
                const unsigned hi = lds32(a_tab + 8u * FX_REP * b + 4u);
                const bool lit = esc;
                const unsigned len = lit ? 1u : (hi >> 24) & 15u;
                bad |= lit ? (b == '\n') : ((hi >> 28) & 1u);  // literal '\n' / unknown code
                esc = !lit && ((hi >> 29) & 1u);
                nl += !lit && ((hi >> 30) & 1u);
                nesc += lit;
                sum += len;
            }
        }
        if (cnt > 0 && c0 + cnt == job.n && esc) bad = 1;  // dangling escape at EOF
        if (eof_nl) {
            sum += 1;
            nl += 1;
        }
        if (bad) atomicOr(&job.ctl->overflow, 4ull);
        // ---- block scan of output bytes; record and escape totals ----
        unsigned long long tile_out;
        const unsigned long long my_off = block_exscan_n<unsigned long long, FX_NT>(sum, s_tmp64, tile_out);
        unsigned r_nl = nl, r_esc = nesc;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            r_nl += __shfl_xor_sync(0xffffffffu, r_nl, o);
            r_esc += __shfl_xor_sync(0xffffffffu, r_esc, o);
        }
        if (lane == 0) {
            s_red[0][wid] = r_nl;
            s_red[1][wid] = r_esc;
        }
        __syncthreads();
        if (wid == 0) {
            unsigned a = lane < FX_NT / 32 ? s_red[0][lane] : 0u, e = lane < FX_NT / 32 ? s_red[1][lane] : 0u;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                e += __shfl_xor_sync(0xffffffffu, e, o);
            }
            if (lane == 0) lookback_publish(job.ts, t, tile_out, a);
            unsigned long long po, pl;
            lookback_resolve(job.ts, t, tile_out, a, po, pl);
            if (lane == 0) {
                s_pre_out = po;
                atomicAdd(&job.ctl->total_out, tile_out);
                atomicAdd(&job.ctl->lines, (unsigned long long)a);
                atomicAdd(&job.ctl->in_lines, (unsigned long long)a);
                if (e) atomicAdd(&job.ctl->escapes, (unsigned long long)e);
                if (po + tile_out > (unsigned long long)job.out_cap) atomicOr(&job.ctl->overflow, 1ull);
            }
        }
        __syncthreads();
        const unsigned long long pre_out = s_pre_out;
        if (pre_out + tile_out > (unsigned long long)job.out_cap) continue;

        // ---- pass 2: expand into aligned 8-byte words ----
        if (sum) {
            const unsigned long long o = pre_out + my_off;
            uint8_t *w = job.out + (o & ~7ull);
            const int head = (int)(o & 7);
            unsigned long long lo = 0;
            int nb = head;
            bool first = true;
            esc = esc0;
#pragma unroll
            for (int k = 0; k <= FX_B; ++k) {
                unsigned long long x;
                unsigned len;
                if (k < FX_B) {
                    if (k >= cnt) continue;
                    const unsigned b = fx_byte(va, vb, k);
                    const unsigned long long e = lds64(a_tab + 8u * FX_REP * b);
                    const bool lit = esc;
                    len = lit ? 1u : (unsigned)(e >> FX_LEN_SHIFT) & 15u;
                    x = lit ? (unsigned long long)b : (e & FX_BYTES);
                    esc = !lit && (e & FX_MARK);
                } else {
                    if (!eof_nl) continue;
                    x = '\n';
                    len = 1;
                }
                const int sh = 8 * nb;
                lo |= x << sh;
                const unsigned long long spill = (x >> 1) >> (63 - sh);
                nb += (int)len;
                if (nb >= 8) {
                    if (first) {
                        fx_put_bytes(w, lo, head, 8);
                        first = false;
                    } else {
                        *reinterpret_cast<unsigned long long *>(w) = lo;
                    }
                    w += 8;
                    lo = spill;
                    nb -= 8;
                }
            }
            if (nb > (first ? head : 0)) fx_put_bytes(w, lo, first ? head : 0, nb);
        }
    }
}

}  // namespace zs
