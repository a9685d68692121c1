// zs_ix.cuh -- random access into a compressed library resident in HBM.
//
// ZSMILES keeps one record per line so a line can be fetched and decoded on
// its own (pkg/README.md:106-110): "grab line i, decode line
// i".  Two steps, both on the device:
//
//   index   ix_count (newlines per 8 KB tile, SWAR) -> ix_scan (one CTA)
//           -> ix_write: offsets[r] = first byte of record r (records are
//           framed by '\n' exactly as pipeline.py:49-74 splits them)
//   decode  ix_sizes (thread per selected record: output bytes / status,
//           numba_impl.py:74-112) -> ix_scan of the sizes -> ix_fill
//           (thread per record, numba_impl.py:115-139)
#pragma once
#include "zs_kernels.cuh"

namespace zs {

constexpr int IX_NT = 256;
constexpr int IX_TILE = IX_NT * 32;  // 32 bytes per thread

__device__ __forceinline__ unsigned ix_nl_mask4(unsigned w) {
    const unsigned x = w ^ 0x0a0a0a0au;
    return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu);  // bit 7 of a byte: == '\n'
}

// newlines in the thread's 32 bytes [c0, c0 + cnt)
__device__ __forceinline__ unsigned ix_slice_count(const uint8_t *in, long long c0, int cnt) {
    unsigned k = 0;
    if (cnt == 32 && ((reinterpret_cast<uintptr_t>(in + c0) & 15) == 0)) {
        const uint4 *p = reinterpret_cast<const uint4 *>(in + c0);
        const uint4 a = __ldg(p), b = __ldg(p + 1);
        k = __popc(ix_nl_mask4(a.x)) + __popc(ix_nl_mask4(a.y)) + __popc(ix_nl_mask4(a.z)) +
            __popc(ix_nl_mask4(a.w)) + __popc(ix_nl_mask4(b.x)) + __popc(ix_nl_mask4(b.y)) +
            __popc(ix_nl_mask4(b.z)) + __popc(ix_nl_mask4(b.w));
    } else {
        for (int j = 0; j < cnt; ++j) k += in[c0 + j] == '\n';
    }
    return k;
}

__global__ void __launch_bounds__(IX_NT) ix_count(const uint8_t *in, long long n, long long nt, unsigned *tcount) {
    __shared__ unsigned s_w[IX_NT / 32];
    for (long long t = blockIdx.x; t < nt; t += gridDim.x) {
        const long long c0 = t * IX_TILE + 32ll * threadIdx.x;
        const int cnt = (int)max(0ll, min(32ll, n - c0));
        unsigned k = ix_slice_count(in, c0, cnt);
#pragma unroll
        for (int o = 16; o; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
        if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = k;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned s = 0;
            for (int w = 0; w < IX_NT / 32; ++w) s += s_w[w];
            tcount[t] = s;
        }
        __syncthreads();
    }
}

// one CTA: exclusive scan of v[0..m) into out (u64), total into *total
template <typename T>
__global__ void __launch_bounds__(1024) ix_scan(const T *v, long long m, unsigned long long *out,
                                                unsigned long long *total) {
    __shared__ unsigned long long s_w[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long per = (m + 1023) / 1024;
    const long long a = min(m, tid * per), b = min(m, a + per);
    unsigned long long sum = 0;
    for (long long i = a; i < b; ++i) sum += (unsigned long long)v[i];
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
    for (long long i = a; i < b; ++i) {
        out[i] = run;
        run += (unsigned long long)v[i];
    }
    if (tid == 0) *total = s_w[31];
}

// offsets[1 + ordinal of a '\n'] = its position + 1; offsets[0] = 0
__global__ void __launch_bounds__(IX_NT) ix_write(const uint8_t *in, long long n, long long nt,
                                                  const unsigned long long *tbase, unsigned long long *offsets) {
    __shared__ unsigned s_w[IX_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (blockIdx.x == 0 && tid == 0) offsets[0] = 0;
    for (long long t = blockIdx.x; t < nt; t += gridDim.x) {
        const long long c0 = t * IX_TILE + 32ll * tid;
        const int cnt = (int)max(0ll, min(32ll, n - c0));
        const unsigned k = ix_slice_count(in, c0, cnt);
        unsigned x = k;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[wid] = x;
        __syncthreads();
        unsigned pre = 0;
        for (int w = 0; w < wid; ++w) pre += s_w[w];
        unsigned long long r = tbase[t] + pre + x - k;  // newlines before this slice
        for (int j = 0; j < cnt; ++j)
            if (in[c0 + j] == '\n') offsets[1 + r++] = (unsigned long long)(c0 + j + 1);
        __syncthreads();
    }
}

// selected records: output bytes and status (0 ok, 1 unknown code, 2 dangling escape)
__global__ void ix_sizes(const uint8_t *in, const unsigned long long *offsets, long long n_rec,
                         const long long *idx, long long k, const uint8_t *explen, long long *len,
                         int8_t *status, long long *errpos) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k; j += (long long)gridDim.x * blockDim.x) {
        const long long r = idx[j];
        long long m = 0, ep = -1;
        int code = 0, st = 0;
        unsigned esc = 0;
        if (r < 0 || r >= n_rec) {
            st = 3;  // no such record
        } else {
            const long long s = (long long)offsets[r], e = (long long)offsets[r + 1] - 1;
            const int kind = decode_size(in + s, e - s, explen, &m, &ep, &code, &esc);
            st = kind == E_UNKNOWN ? 1 : kind == E_TRUNC ? 2 : 0;
            if (st == 1) ep = ((long long)code << 40) | ep;  // code in the high bits
        }
        len[j] = st ? 0 : m;
        status[j] = (int8_t)st;
        errpos[j] = ep;
    }
}

__global__ void ix_fill(const uint8_t *in, const unsigned long long *offsets, const long long *idx, long long k,
                        const int8_t *status, const unsigned long long *out_off, const uint8_t *explen,
                        const uint16_t *expoff, const uint8_t *expflat, uint8_t *out) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < k; j += (long long)gridDim.x * blockDim.x) {
        if (status[j]) continue;
        const long long r = idx[j];
        const long long s = (long long)offsets[r], e = (long long)offsets[r + 1] - 1;
        decode_fill(in + s, e - s, explen, expoff, expflat, out + out_off[j]);
    }
}

}  // namespace zs
