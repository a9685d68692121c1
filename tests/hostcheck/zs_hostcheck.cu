// Host build of the per-line device routines (csrc/zs_device.cuh), for CPU
// unit tests against the oracle.  TEST INFRASTRUCTURE ONLY: the product runs
// these routines on sm_100a inside the tile kernels.
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../paper_2404_19391_b200/csrc/zs_device.cuh"

using namespace zs;

extern "C" {

// Renumber one line exactly as compress_tiles does: fast path, fallback to
// preprocess_line on pristine bytes.  Returns the error kind (0 ok, -1 =
// line grows, needs the out-of-smem path) and the renumbered bytes.
int hc_renumber(const uint8_t *in, int n, uint8_t *out, int *out_len, int *err_off,
                uint64_t *ids, int *used_fallback) {
    uint8_t lut[8 * 256];
    for (int k = 0; k < 8 * 256; ++k) lut[k] = tk_entry(k >> 8, k & 255);
    std::vector<uint8_t> s(in, in + n), marks(n + 1, 0xaa);
    int nl = n, eoff = -1;
    unsigned long long id2[2] = {0, 0};
    int k = renumber_fast(s.data(), n, lut, marks.data(), &nl, &eoff, id2);
    *used_fallback = 0;
    if (k == RN_FALLBACK) {
        *used_fallback = 1;
        s.assign(in, in + n);
        int nl2 = n;
        k = preprocess_line(s.data(), n, marks.data(), s.data(), &nl2, &eoff, id2);
        nl = nl2;
    }
    *err_off = eoff;
    ids[0] = id2[0];
    ids[1] = id2[1];
    if (k == 0) {
        memcpy(out, s.data(), nl);
        *out_len = nl;
    }
    return k;
}

// renumber_bm (bitmap variant used by the in-place kernel) + fallback
int hc_renumber_bm(const uint8_t *in, int n, uint8_t *out, int *out_len, int *err_off,
                   uint64_t *ids, int *used_fallback, int bit0) {
    uint8_t lut[8 * 256];
    for (int k = 0; k < 8 * 256; ++k) lut[k] = tk_entry(k >> 8, k & 255);
    std::vector<uint8_t> s(in, in + n);
    std::vector<unsigned> bm((bit0 + n) / 32 + 2, 0);
    int nl = n, eoff = -1;
    unsigned long long id2[2] = {0, 0};
    int k = renumber_bm(s.data(), n, lut, bm.data(), bit0, &nl, &eoff, id2);
    *used_fallback = 0;
    if (k == RN_FALLBACK) {
        *used_fallback = 1;
        s.assign(in, in + n);
        std::vector<uint8_t> marks(n + 1);
        int nl2 = n;
        k = preprocess_line(s.data(), n, marks.data(), s.data(), &nl2, &eoff, id2);
        nl = nl2;
    }
    *err_off = eoff;
    ids[0] = id2[0];
    ids[1] = id2[1];
    if (k == 0) {
        memcpy(out, s.data(), nl);
        *out_len = nl;
    }
    return k;
}

// preprocess_line alone (the general routine), out of place
int hc_preprocess(const uint8_t *in, int n, uint8_t *out, int *out_len, int *err_off,
                  uint64_t *ids, int cr_is_error) {
    std::vector<uint8_t> marks(n + 1);
    unsigned long long id2[2] = {0, 0};
    int k = preprocess_line(in, n, marks.data(), out, out_len, err_off, id2, cr_is_error != 0);
    ids[0] = id2[0];
    ids[1] = id2[1];
    return k;
}

// dp_t2 (cost-window transducer) + emit for one line
long long hc_compress_t2(const uint16_t *dfa2, const uint32_t *t2, const uint8_t *codes,
                         const int32_t *exp_len, const uint8_t *line, int n, uint8_t *out) {
    std::vector<uint8_t> dec(n + 1);
    int cost = dp_t2(line, n, dec.data(), dfa2, t2, codes);
    long long w = 0;
    for (int i = 0; i < n;) {
        uint8_t c = dec[i];
        if (c == D_ESC) {
            out[w++] = 0x20;
            out[w++] = line[i++];
        } else {
            out[w++] = c;
            i += exp_len[c];
        }
    }
    return w == cost ? w : -1;
}

// The in-place kernel's per-line pipeline on a whole newline-framed buffer:
// renumber_bm (optional) -> dp_t2_inplace over the buffer bytes -> emit from
// the in-band encoding.  Returns the output length (out must hold 2n+2).
long long hc_inplace_stream(const uint16_t *dfa2, const uint32_t *t2, const uint8_t *codes,
                            const int32_t *exp_len, const uint8_t *in, int n, int preprocess,
                            uint8_t *out) {
    uint8_t lut[8 * 256];
    for (int k = 0; k < 8 * 256; ++k) lut[k] = tk_entry(k >> 8, k & 255);
    std::vector<uint8_t> win(in, in + n);
    win.push_back('\n');
    std::vector<unsigned> rb(n / 32 + 4, 0), eb(n / 32 + 4, 0);
    std::vector<int> starts;
    for (int p = 0; p < n; ++p)
        if (p == 0 || in[p - 1] == '\n') starts.push_back(p);
    for (int p : starts) {
        int e = p;
        while (e < n && in[e] != '\n') ++e;
        int n_l = e - p;
        uint8_t *s = win.data() + p;
        if (preprocess) {
            int nl = n_l, off = -1;
            unsigned long long ids[2] = {0, 0};
            int k = renumber_bm(s, n_l, lut, rb.data(), p, &nl, &off, ids);
            if (k != E_NONE) return -1000 - k;
            if (nl < n_l) s[nl] = '\n';
            n_l = nl;
        }
        dp_t2_inplace(s, n_l, dfa2, t2, codes, eb.data(), p);
    }
    long long w = 0;
    for (int p : starts) {
        for (int i = p;;) {
            const uint8_t c = win[i];
            if (c == '\n') break;
            if ((eb[i >> 5] >> (i & 31)) & 1) {
                out[w++] = 0x20;
                out[w++] = c;
                ++i;
            } else {
                out[w++] = c;
                i += exp_len[c];
            }
        }
        out[w++] = '\n';
    }
    return w;
}

// dp_fast<W> + emit for one line
long long hc_compress_fast(const uint16_t *dfa, const uint8_t *codes, int W, const int32_t *exp_len,
                           const uint8_t *line, int n, uint8_t *out) {
    std::vector<uint8_t> dec(n + 1);
    int cost;
    switch (W) {
    case 2: cost = dp_fast<2>(line, n, dec.data(), dfa, codes); break;
    case 4: cost = dp_fast<4>(line, n, dec.data(), dfa, codes); break;
    case 6: cost = dp_fast<6>(line, n, dec.data(), dfa, codes); break;
    default: cost = dp_fast<8>(line, n, dec.data(), dfa, codes); break;
    }
    long long w = 0;
    for (int i = 0; i < n;) {
        uint8_t c = dec[i];
        if (c == D_ESC) {
            out[w++] = 0x20;
            out[w++] = line[i++];
        } else {
            out[w++] = c;
            i += exp_len[c];
        }
    }
    return w == cost ? w : -1;
}
}
