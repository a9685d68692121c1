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
    uint8_t lut[256];
    for (int b = 0; b < 256; ++b) lut[b] = tok_bits(b);
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
