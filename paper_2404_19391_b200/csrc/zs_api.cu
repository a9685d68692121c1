// zs_api.cu -- C ABI (include/zs.h) over the sm_100a kernels.
//
// Host side: dictionary tables in the reference layouts -> device tables
// (dense trie for the generic walk, reversed-pattern Aho-Corasick DFA for the
// fast path, compact decode tables); per-context stream, events and grow-only
// device buffers; the whole-buffer calls (one persistent-kernel launch per
// buffer or chunk) and the parity-shim calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <set>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "../../include/zs_debug.h"
#include "zs_kernels.cuh"
#include "zs_fx.cuh"
#include "zs_cx.cuh"
#include "zs_ll.cuh"
#include "zs_ix.cuh"
#include "zs_train.cuh"

using namespace zs;

namespace {

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { release(); }  // (zs_ctx_destroy sets the device first)
    cudaError_t reserve(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t c = std::max<size_t>(n, 256);
        cudaError_t e = cudaMalloc(&p, c);
        if (e == cudaSuccess) cap = c;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T> T *as() const { return reinterpret_cast<T *>(p); }
    // grow to >= n bytes keeping the first `keep` bytes (stream-ordered copy)
    cudaError_t grow_keep(size_t n, size_t keep, cudaStream_t st) {
        if (n <= cap) return cudaSuccess;
        void *q = nullptr;
        const size_t c = std::max<size_t>(n, 2 * cap);
        cudaError_t e = cudaMalloc(&q, c);
        if (e != cudaSuccess) return e;
        if (keep) e = cudaMemcpyAsync(q, p, keep, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (p) cudaFree(p);
        p = q;
        cap = c;
        return e;
    }
};

struct HostTables {
    int n_nodes = 0, max_len = 0;
    std::vector<int32_t> children;
    std::vector<int16_t> term_code;
    bool fast = false;
    int n_states = 0;
    std::vector<uint16_t> dfa;
    std::vector<uint8_t> codes;
    // cost-window transducer (see build_t2): dfa2 = dfa with a mask *index*
    bool t2_ok = false;
    int n_windows = 0, n_masks = 0;
    std::vector<uint16_t> dfa2;
    std::vector<uint32_t> t2;
    // lane-chunk compress kernel tables (zs_cx.cuh): '\n' column + transducer slot
    bool cx_ok = false;
    // lane-chunk kernel, key-window parse for patterns of up to 16 bytes (build_kw)
    bool kw_ok = false;
    int kw_states = 0, kw_cols = 0;
    std::vector<uint8_t> kw_cmap, kw_codes;
    std::vector<uint32_t> kw_dfa;
    int cx_states = 0, cx_cols = 0;  // minimised DFA: states x byte-class columns
    std::vector<uint8_t> cx_cmap;     // byte -> column
    std::vector<uint16_t> cx_dfa;
    std::vector<uint16_t> cx_t2;
    std::vector<uint8_t> cx_codes;
    // product automaton of the minimised DFA and the cost-window transducer
    // (build_pa): one table lookup per byte in compress_cx<true>'s parse
    bool pa_ok = false;
    int pa_states = 0, pa_cols = 0;
    std::vector<uint8_t> pa_cmap4;  // byte -> column * 4
    std::vector<uint32_t> pa;       // [state][column] entries (PaEntry layout, zs_cx.cuh)
    uint8_t exp_len[256];
    uint16_t exp_off[257];
    std::vector<uint8_t> exp_flat;
};

}  // namespace

struct zs_ctx {
    int dev = 0;
    int n_sm = 0;
    static constexpr int NSLOT = 3;  // host pipeline depth (chunk k+3 reuses chunk k's buffers)
    cudaStream_t stream[NSLOT] = {};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    const char *last_kernel = "";
    cudaEvent_t ev_ctl[NSLOT] = {}, ev_out[NSLOT] = {};
    std::string err;
    bool have_dict = false;
    HostTables ht;
    Tables tb{};
    int fast_w = 0;
    DevBuf d_pa, d_pacmap, d_dfa, d_codes, d_children, d_term, d_explen, d_expoff, d_expflat, d_dfa2, d_t2, d_fxc, d_fxe, d_cxdfa, d_cxt2, d_cxcodes, d_cxcmap;
    int no_pa = 0;  // debug: DFA + transducer parse instead of the product automaton
    int slices = 0;  // compress_cx<true, true>: every phase on byte-exact slices
    int nk[NSLOT] = {};  // kernels the last launch_stream on a slot issued (zs_result.gpu_launches)
    int p4_lane = 0;  // debug: parse per line-lane range instead of byte-exact slices
    bool fx_ok = false;  // streaming decode kernel serves this dictionary (max expansion <= 7)
    int fx_blocks[2] = {0, 0};  // resident fx_count / fx_emit CTAs per SM
    int fx_wide = -1;           // fx_blocks were sized for this emit variant
    int no_t2 = 0;  // debug: force the key-window DP
    int no_ip = 0;  // debug: force the decision-array kernel
    // per-slot work buffers (NSLOT-deep host pipeline)
    DevBuf ctl[NSLOT], ts[NSLOT], terr[NSLOT], in[NSLOT], out[NSLOT], arena[NSLOT];  // arena: per slot
    DevBuf fxs[NSLOT];  // streaming-decode scratch per slot
    // long lines (zs_ll.cuh) per slot: the recorded lines, the tiles' last
    // newlines, per-block arrays, events, renumbered lines, decisions, output
    DevBuf ll[NSLOT], tl[NSLOT], llb[NSLOT], lle[NSLOT], llc[NSLOT], llr[NSLOT], lld[NSLOT], llo[NSLOT];
    DevBuf d_lltok;  // long-line tokenizer tables
    int no_ll = 0;  // debug: long lines on the general routine (one thread each)
    DevBuf ixs;     // record-index scratch
    // dictionary training (zs_train.cuh): corpus, census scratch, rank table, selection state
    struct {
        DevBuf buf, run, pos[2], key[2], lcp, runs, v, ex, bstart, cand, cub, nsel;
        DevBuf rpos, rocc, rlen;  // rank table rows
        DevBuf rank[2], idx[2], dead, child, term, ctl, blk, sel;
        long long n = 0, rows = 0;
        int lmax = 0;
    } tr;
    // shim scratch
    DevBuf s_flat, s_starts, s_out, s_lens, s_dec, s_stat, s_errpos, s_tot, s_ids, s_outst;
    Ctl *h_ctl = nullptr;  // pinned, NSLOT slots
    uint8_t *h_last = nullptr;  // pinned: the device input's last byte (run_device)
    float last_ms = 0.f;
    int timing = 0;
    cudaStream_t user_stream = nullptr;  // zs_set_stream: device-pointer calls order after it
    cudaEvent_t ev_user = nullptr;
};

namespace {

int fail(zs_ctx *ctx, cudaError_t e, const char *what) {
    if (ctx) ctx->err = std::string(what) + ": " + cudaGetErrorString(e);
    return ZS_E_CUDA;
}

#define CK(call)                                         \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return fail(ctx, e_, #call); \
    } while (0)

// device-pointer calls: wait for the work queued on the caller's stream
// (zs_set_stream) before reading its buffers
int after_user_stream(zs_ctx *ctx) {
    CK(cudaEventRecord(ctx->ev_user, ctx->user_stream));
    CK(cudaStreamWaitEvent(ctx->stream[0], ctx->ev_user, 0));
    return ZS_OK;
}

// ---------------------------------------------------------------------------
// dictionary -> device tables
// ---------------------------------------------------------------------------

// Walk the reference trie (trie.py:22-50 layout) to recover (pattern, code).
void trie_patterns(const int32_t *children, const int16_t *term_code, int n_nodes,
                   std::vector<std::pair<std::string, int>> &out) {
    std::vector<std::pair<int, std::string>> stack{{0, std::string()}};
    while (!stack.empty()) {
        auto [node, s] = stack.back();
        stack.pop_back();
        if (node < 0 || node >= n_nodes) continue;
        if (term_code[node] >= 0) out.emplace_back(s, term_code[node]);
        for (int b = 255; b >= 0; --b) {
            int c = children[(size_t)node * 256 + b];
            if (c >= 0) stack.emplace_back(c, s + (char)b);
        }
    }
}

// Reversed-pattern Aho-Corasick DFA.  Reading a line right to left, the state
// after consuming byte i has as outputs exactly the patterns that START at i
// (a reversed pattern is a suffix of the reversed text read so far).
bool build_dfa(const std::vector<std::pair<std::string, int>> &pats, int max_len, HostTables &ht) {
    if (max_len > FAST_W) return false;
    for (auto &pc : pats)
        for (unsigned char c : pc.first)
            if (c < 0x21 || c > 0x7e) return false;
    std::vector<std::array<int, 256>> go(1);
    go[0].fill(-1);
    std::vector<uint32_t> own(1, 0);
    std::vector<std::array<int, FAST_W>> own_code(1);
    own_code[0].fill(-1);
    for (auto &pc : pats) {
        int node = 0;
        for (auto it = pc.first.rbegin(); it != pc.first.rend(); ++it) {
            unsigned char c = (unsigned char)*it;
            if (go[node][c] < 0) {
                go[node][c] = (int)go.size();
                go.emplace_back();
                go.back().fill(-1);
                own.push_back(0);
                own_code.emplace_back();
                own_code.back().fill(-1);
            }
            node = go[node][c];
        }
        int L = (int)pc.first.size();
        own[node] |= 1u << (L - 1);
        own_code[node][L - 1] = pc.second;
    }
    const int ns = (int)go.size();
    if (ns > FAST_STATES) return false;
    std::vector<int> failv(ns, 0), order;
    std::vector<uint32_t> outm(own);
    std::vector<std::array<int, FAST_W>> code(own_code);
    order.push_back(0);
    for (size_t qi = 0; qi < order.size(); ++qi) {
        int s = order[qi];
        for (int c = 0; c < 256; ++c) {
            int ch = go[s][c];
            if (ch >= 0) {
                failv[ch] = s == 0 ? 0 : go[failv[s]][c];
                outm[ch] = own[ch] | outm[failv[ch]];
                for (int L = 0; L < FAST_W; ++L)
                    code[ch][L] = own_code[ch][L] >= 0 ? own_code[ch][L] : code[failv[ch]][L];
                order.push_back(ch);
            } else {
                go[s][c] = s == 0 ? 0 : go[failv[s]][c];
            }
        }
    }
    ht.n_states = ns;
    ht.dfa.assign((size_t)align16(ns * NCOL * 2) / 2, 0);
    ht.codes.assign((size_t)align16(ns * FAST_W), 0);
    for (int s = 0; s < ns; ++s) {
        for (int col = 0; col < NCOL; ++col) {
            int b = col < 96 ? 0x20 + col : 0x00;  // col 96: every byte outside 0x20..0x7f
            int nx = go[s][b];
            ht.dfa[(size_t)s * NCOL + col] = (uint16_t)(nx | (outm[nx] << 8));
        }
        for (int L = 0; L < FAST_W; ++L)
            ht.codes[(size_t)s * FAST_W + L] = (uint8_t)(code[s][L] < 0 ? 0 : code[s][L]);
    }
    return true;
}

// Cost-window transducer for the parse.  The parse decision at byte i is a
// function of the AC match mask M(i) and of the window of suffix costs of
// positions i+1..i+W relative to cost[i+1] (plus INF past the line end).
// Those windows come from a small closed set, so the DP step becomes
//   (window, mask) -> (next window, chosen length L (0 = escape), cost delta)
// precomputed here by BFS over the joint (AC state, window) states reachable
// from the line-end state under every byte.  Built only if it fits smem.
bool build_t2(HostTables &ht, int W) {
    constexpr int8_t INF = 127;
    const int ns = ht.n_states;
    // distinct masks -> indices (stored in the DFA entry's high byte)
    std::vector<int> mask_id(256, -1);
    std::vector<unsigned> masks;
    for (int s = 0; s < ns; ++s)
        for (int col = 0; col < NCOL; ++col) {
            unsigned m = ht.dfa[(size_t)s * NCOL + col] >> 8;
            if (mask_id[m] < 0) {
                mask_id[m] = (int)masks.size();
                masks.push_back(m);
            }
        }
    if (masks.size() > (size_t)T2_MASKS) return false;
    typedef std::array<int8_t, FAST_W> Win;  // w[L-1] = cost[i+L] - cost[i+1]
    std::map<Win, int> win_id;
    std::vector<Win> wins;
    auto wid = [&](const Win &w) {
        auto it = win_id.find(w);
        if (it != win_id.end()) return it->second;
        int id = (int)wins.size();
        win_id.emplace(w, id);
        wins.push_back(w);
        return id;
    };
    Win w0;
    w0.fill(INF);
    w0[0] = 0;
    wid(w0);
    std::map<std::pair<int, int>, uint32_t> step;  // (window, mask index) -> entry
    auto transition = [&](int wi, int mi) -> uint32_t {
        auto key = std::make_pair(wi, mi);
        auto it = step.find(key);
        if (it != step.end()) return it->second;
        const Win w = wins[wi];
        const unsigned M = masks[mi];
        int bc = 2, bl = 1, L_sel = 0;  // escape: 0x20 + literal, cost 2
        for (int L = 1; L <= W; ++L) {
            if (!((M >> (L - 1)) & 1) || w[L - 1] == INF) continue;
            int c = w[L - 1] + 1;
            if (c < bc || (c == bc && L > bl)) {  // numba_impl.py:50
                bc = c;
                bl = L;
                L_sel = L;
            }
        }
        Win nw;
        nw.fill(INF);
        nw[0] = 0;
        for (int L = 1; L < W; ++L) nw[L] = w[L - 1] == INF ? INF : (int8_t)(w[L - 1] - bc);
        int nwi = wid(nw);
        uint32_t e = (uint32_t)nwi | ((uint32_t)L_sel << 12) | ((uint32_t)(bc + 16) << 16);
        step.emplace(key, e);
        return e;
    };
    // BFS over joint states
    std::set<std::pair<int, int>> seen;
    std::vector<std::pair<int, int>> q{{0, 0}};
    seen.insert({0, 0});
    for (size_t qi = 0; qi < q.size(); ++qi) {
        const int st = q[qi].first, wi = q[qi].second;
        for (int col = 0; col < NCOL; ++col) {
            const uint16_t e = ht.dfa[(size_t)st * NCOL + col];
            const int s2 = e & 0xff, mi = mask_id[e >> 8];
            const uint32_t x = transition(wi, mi);
            std::pair<int, int> nxt{s2, (int)(x & 0xfff)};
            if (seen.insert(nxt).second) q.push_back(nxt);
            if (wins.size() > (size_t)T2_WINDOWS || q.size() > 400000) return false;
        }
    }
    ht.n_windows = (int)wins.size();
    ht.n_masks = (int)masks.size();
    ht.t2.assign((size_t)ht.n_windows * T2_MASKS, 0xffffffffu);
    for (auto &kv : step) ht.t2[(size_t)kv.first.first * T2_MASKS + kv.first.second] = kv.second;
    ht.dfa2 = ht.dfa;
    for (size_t k = 0; k < (size_t)ns * NCOL; ++k)
        ht.dfa2[k] = (uint16_t)((ht.dfa[k] & 0xff) | (mask_id[ht.dfa[k] >> 8] << 8));
    ht.t2_ok = true;
    return true;
}

// Tables of the lane-chunk kernel: the DFA gets a '\n' column (column
// c = min(b - 10, 118): 0 = '\n', 22..117 = 0x20..0x7f, the rest = other)
// whose entry returns to the root with the reserved mask slot CX_NLMASK; the
// transducer's CX_NLMASK entry of every window resets to the line-end window
// with code slot 9 (the record separator, cost +1).  Code slot 0 (an escape)
// is 0x20, so the parse writes every decision without a branch.
// Key-window parse tables for patterns of up to 16 bytes (the lane-chunk
// kernel's P4 when the cost-window transducer does not apply): the reversed
// Aho-Corasick DFA with 16-bit match masks, Moore-minimised, over byte-class
// columns; entry = next state << 16 | match mask of the target state (bit
// L-1: a pattern of length L starts at the byte just read).  Codes per state
// for L = 2..16 (a length-1 match is the identity code: the byte itself).
bool build_kw(const std::vector<std::pair<std::string, int>> &pats, int max_len, HostTables &ht) {
    constexpr int KW = 16;
    if (max_len < 1 || max_len > KW) return false;
    for (auto &pc : pats)
        for (unsigned char c : pc.first)
            if (c < 0x21 || c > 0x7e) return false;
    std::vector<std::array<int, 256>> go(1);
    go[0].fill(-1);
    std::vector<uint32_t> own(1, 0);
    std::vector<std::array<int, KW>> own_code(1);
    own_code[0].fill(-1);
    for (auto &pc : pats) {
        int node = 0;
        for (auto it = pc.first.rbegin(); it != pc.first.rend(); ++it) {
            const unsigned char c = (unsigned char)*it;
            if (go[node][c] < 0) {
                go[node][c] = (int)go.size();
                go.emplace_back();
                go.back().fill(-1);
                own.push_back(0);
                own_code.emplace_back();
                own_code.back().fill(-1);
            }
            node = go[node][c];
        }
        const int L = (int)pc.first.size();
        own[node] |= 1u << (L - 1);
        own_code[node][L - 1] = pc.second;
    }
    const int ns = (int)go.size();
    if (ns > 65535) return false;
    std::vector<int> failv(ns, 0), order{0};
    std::vector<uint32_t> outm(own);
    std::vector<std::array<int, KW>> code(own_code);
    for (size_t qi = 0; qi < order.size(); ++qi) {
        const int st = order[qi];
        for (int c = 0; c < 256; ++c) {
            const int ch = go[st][c];
            if (ch >= 0) {
                failv[ch] = st == 0 ? 0 : go[failv[st]][c];
                outm[ch] = own[ch] | outm[failv[ch]];
                for (int L = 0; L < KW; ++L)
                    code[ch][L] = own_code[ch][L] >= 0 ? own_code[ch][L] : code[failv[ch]][L];
                order.push_back(ch);
            } else {
                go[st][c] = st == 0 ? 0 : go[failv[st]][c];
            }
        }
    }
    // Moore minimisation (outputs: match mask, codes for L >= 2)
    std::vector<int> cls(ns), tmp(ns);
    {
        std::map<std::vector<int>, int> ids;
        for (int st = 0; st < ns; ++st) {
            std::vector<int> key{(int)outm[st]};
            for (int L = 2; L <= KW; ++L) key.push_back(code[st][L - 1]);
            cls[st] = ids.emplace(key, (int)ids.size()).first->second;
        }
    }
    for (int nc = -1;;) {
        std::map<std::vector<int>, int> ids;
        for (int st = 0; st < ns; ++st) {
            std::vector<int> key{cls[st]};
            for (int b = 0; b < 256; ++b)
                if (b != '\n') key.push_back(cls[go[st][b]]);
            tmp[st] = ids.emplace(key, (int)ids.size()).first->second;
        }
        cls = tmp;
        if ((int)ids.size() == nc) break;
        nc = (int)ids.size();
    }
    std::vector<int> ren(ns, -1);
    int S = 0;
    ren[cls[0]] = S++;
    for (int st = 0; st < ns; ++st)
        if (ren[cls[st]] < 0) ren[cls[st]] = S++;
    std::vector<int> rep(S, -1);
    for (int st = 0; st < ns; ++st)
        if (rep[ren[cls[st]]] < 0) rep[ren[cls[st]]] = st;
    std::map<std::vector<int>, int> cols;
    std::vector<int> cmap(256);
    for (int b = 0; b < 256; ++b) {
        std::vector<int> key;
        for (int q = 0; q < S; ++q) key.push_back(ren[cls[go[rep[q]][b]]]);
        cmap[b] = cols.emplace(key, (int)cols.size()).first->second;
    }
    const int nc = (int)cols.size();
    if (nc > 255) return false;
    ht.kw_states = S;
    ht.kw_cols = nc;
    ht.kw_cmap.assign(cmap.begin(), cmap.end());
    ht.kw_dfa.assign((size_t)S * nc, 0);
    ht.kw_codes.assign((size_t)S * CX_CODES, 0);
    for (int q = 0; q < S; ++q) {
        for (int b = 0; b < 256; ++b) {
            const int t = go[rep[q]][b];
            ht.kw_dfa[(size_t)q * nc + cmap[b]] = ((uint32_t)ren[cls[t]] << 16) | outm[t];
        }
        for (int L = 2; L <= KW; ++L) {
            const int c = code[rep[q]][L - 1];
            ht.kw_codes[(size_t)q * CX_CODES + L - 1] = (uint8_t)(c < 0 ? 0 : c);
        }
    }
    return true;
}

// dynamic shared memory compress_cx can opt into on this device (the
// opt-in maximum minus the kernel's static shared memory)
int cx_dyn_smem_limit() {
    static int lim = -1;
    if (lim < 0) {
        int dev = 0, optin = 0;
        cudaFuncAttributes fa{};
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess &&
            cudaFuncGetAttributes(&fa, compress_cx<false, false>) == cudaSuccess)
            lim = optin - (int)fa.sharedSizeBytes;
        else
            lim = 227 * 1024 - 16 * 1024;  // no device: a conservative bound
    }
    return lim;
}

bool build_cx(HostTables &ht, int max_len) {
    if (!ht.t2_ok || ht.n_masks > CX_NLMASK || max_len > 8) return false;
    const int ns = ht.n_states, nw = ht.n_windows;
    // byte-level machine: next state and (target) mask index per byte; '\n'
    // gets its own column (back to the root with the reserved mask slot)
    auto col_of = [](int b) { return (b >= 0x20 && b <= 0x7f) ? b - 0x20 : 96; };
    std::vector<int> nxt((size_t)ns * 256), mk(ns, 0);
    for (int st = 0; st < ns; ++st)
        for (int b = 0; b < 256; ++b) {
            const uint16_t e = ht.dfa2[(size_t)st * NCOL + col_of(b)];
            nxt[(size_t)st * 256 + b] = e & 0xff;
            mk[e & 0xff] = e >> 8;  // the mask index belongs to the target state
        }
    // Moore minimisation.  A state's output is its match-mask index and its
    // codes for lengths 2..8; the length-1 code is the byte itself (identity
    // codes map a byte to itself), so the states reached by identity-only
    // bytes merge.
    std::vector<int> cls(ns), tmp(ns);
    {
        std::map<std::vector<int>, int> ids;
        for (int st = 0; st < ns; ++st) {
            std::vector<int> key{mk[st]};
            for (int L = 2; L <= FAST_W; ++L) key.push_back(ht.codes[(size_t)st * FAST_W + L - 1]);
            cls[st] = ids.emplace(key, (int)ids.size()).first->second;
        }
    }
    for (int nc = -1;;) {
        std::map<std::vector<int>, int> ids;
        for (int st = 0; st < ns; ++st) {
            std::vector<int> key{cls[st]};
            for (int b = 0; b < 256; ++b)
                if (b != '\n') key.push_back(cls[nxt[(size_t)st * 256 + b]]);
            tmp[st] = ids.emplace(key, (int)ids.size()).first->second;
        }
        cls = tmp;
        if ((int)ids.size() == nc) break;
        nc = (int)ids.size();
    }
    // renumber so the root is state 0
    std::vector<int> ren(ns, -1);
    int S = 0;
    ren[cls[0]] = S++;
    for (int st = 0; st < ns; ++st)
        if (ren[cls[st]] < 0) ren[cls[st]] = S++;
    std::vector<int> rep(S, -1);  // a representative original state per class
    for (int st = 0; st < ns; ++st)
        if (rep[ren[cls[st]]] < 0) rep[ren[cls[st]]] = st;
    // byte columns: bytes with identical transitions from every state
    std::map<std::vector<int>, int> cols;
    std::vector<int> cmap(256);
    cols[std::vector<int>{-1}] = 0;  // column 0: '\n'
    for (int b = 0; b < 256; ++b) {
        if (b == '\n') {
            cmap[b] = 0;
            continue;
        }
        std::vector<int> key;
        for (int q = 0; q < S; ++q) key.push_back(ren[cls[nxt[(size_t)rep[q] * 256 + b]]]);
        cmap[b] = cols.emplace(key, (int)cols.size()).first->second;
    }
    const int nc = (int)cols.size();
    if (S > 256 || nc > 255 || cx_smem_bytes(S, nw, nc) > cx_dyn_smem_limit()) return false;
    ht.cx_states = S;
    ht.cx_cols = nc;
    ht.cx_cmap.assign(cmap.begin(), cmap.end());
    ht.cx_dfa.assign((size_t)cx_align16(S * nc * 2) / 2, 0);
    for (int q = 0; q < S; ++q)
        for (int b = 0; b < 256; ++b) {
            uint16_t e;
            if (b == '\n') {
                e = (uint16_t)(0 | (CX_NLMASK << 8));
            } else {
                const int t = nxt[(size_t)rep[q] * 256 + b];
                e = (uint16_t)(ren[cls[t]] | (mk[t] << 8));
            }
            ht.cx_dfa[(size_t)q * nc + cmap[b]] = e;
        }
    // transducer entries as u16: next window (9 bits) | L << 9 | (delta + 4) << 13
    if (nw > 512) return false;
    ht.cx_t2.assign((size_t)nw * CX_T2S, 0);
    for (int w = 0; w < nw; ++w)
        for (int m = 0; m < T2_MASKS; ++m) {
            const uint32_t x = ht.t2[(size_t)w * T2_MASKS + m];
            uint32_t e;
            if (m == CX_NLMASK) {
                e = 0u | (9u << 9) | ((1u + 4u) << 13);
            } else if (x == 0xffffffffu) {
                e = 0;  // unreachable (mask index unused)
            } else {
                const int delta = (int)(x >> 16) - 16;
                if (delta < -4 || delta > 3 || (x & 0xfffu) > 511u) return false;
                e = (x & 0x1ffu) | (((x >> 12) & 15u) << 9) | ((uint32_t)(delta + 4) << 13);
            }
            ht.cx_t2[(size_t)w * CX_T2S + m] = (uint16_t)e;
        }
    // code slot L: 0 = escape (0x20, never a code), 2..8 = the match of length L,
    // 9 = '\n'; length 1 is the byte itself
    ht.cx_codes.assign((size_t)cx_align16(S * CX_CODES), 0);
    for (int q = 0; q < S; ++q) {
        ht.cx_codes[(size_t)q * CX_CODES] = 0x20;
        for (int L = 2; L <= FAST_W; ++L)
            ht.cx_codes[(size_t)q * CX_CODES + L] = ht.codes[(size_t)rep[q] * FAST_W + L - 1];
        ht.cx_codes[(size_t)q * CX_CODES + 9] = '\n';
    }
    ht.cx_ok = true;
    if (getenv("ZS_VERBOSE"))
        fprintf(stderr, "zs: cx tables: %d -> %d states, %d byte columns, %d windows, %d masks, smem %d B\n", ns, S,
                nc, nw, ht.n_masks, cx_smem_bytes(S, nw, nc));
    return true;
}

// Product automaton for the parse (compress_cx<true>).  The parse state of
// compress_cx is the pair (minimised DFA state q, cost window w); reading one
// byte of column c moves it to (dfa(q, c), t2(w, mask(dfa(q, c)))) and emits
// a decision (code, identity byte, escape or '\n') and a cost delta.  The
// joint states reachable from the line-end state (0, 0) are enumerated and
// Moore-minimised over those outputs, and the byte columns are recomputed for
// the minimised machine: for the default dictionary 164 states x 27 columns,
// one u32 lookup per byte instead of a DFA, a transducer and a code lookup.
// Entry: next state's row offset in bytes (bits 0-15) | code << 16 |
// (cost delta + 4) << 24 | identity << 31 (the decision is the byte itself).
bool build_pa(HostTables &ht) {
    ht.pa_ok = false;
    if (!ht.cx_ok) return false;
    const int S = ht.cx_states, nc = ht.cx_cols;
    std::map<std::pair<int, int>, int> id;
    std::vector<std::pair<int, int>> js{{0, 0}};
    id[{0, 0}] = 0;
    std::vector<int> nxt, out;  // [joint][col]: next joint, output (code | d4 << 8 | identity << 11)
    for (size_t k = 0; k < js.size(); ++k) {
        const int q = js[k].first, w = js[k].second;
        for (int c = 0; c < nc; ++c) {
            const uint16_t e = ht.cx_dfa[(size_t)q * nc + c];
            const int q2 = e & 0xff, m = e >> 8;
            const uint16_t x = ht.cx_t2[(size_t)w * CX_T2S + m];
            const int w2 = x & 0x1ff, L = (x >> 9) & 15, d4 = x >> 13;
            const int o = L == 1 ? (1 << 11) | (d4 << 8) : (ht.cx_codes[(size_t)q2 * CX_CODES + L] | (d4 << 8));
            auto it = id.find({q2, w2});
            int j;
            if (it == id.end()) {
                j = (int)js.size();
                id[{q2, w2}] = j;
                js.push_back({q2, w2});
                if (js.size() > 200000) return false;
            } else {
                j = it->second;
            }
            nxt.push_back(j);
            out.push_back(o);
        }
    }
    const int N = (int)js.size();
    // Moore minimisation (partition refinement on (class, outputs, next classes))
    std::vector<int> cls(N, 0), tmp(N);
    int ncls = 0;
    for (int round = 0;; ++round) {
        std::map<std::vector<int>, int> ids;
        for (int s = 0; s < N; ++s) {
            std::vector<int> key;
            key.reserve(2 * nc + 1);
            key.push_back(cls[s]);
            for (int c = 0; c < nc; ++c) {
                key.push_back(out[(size_t)s * nc + c]);
                key.push_back(round ? cls[nxt[(size_t)s * nc + c]] : 0);
            }
            tmp[s] = ids.emplace(key, (int)ids.size()).first->second;
        }
        cls = tmp;
        if ((int)ids.size() == ncls) break;
        ncls = (int)ids.size();
    }
    // renumber: the line-end state (0, 0) is state 0
    std::vector<int> ren(ncls, -1), rep;
    int P = 0;
    for (int s = 0; s < N; ++s)
        if (ren[cls[s]] < 0) {
            ren[cls[s]] = P++;
            rep.push_back(s);
        }
    // byte columns of the minimised machine
    std::map<std::vector<int>, int> cols;
    std::vector<int> cmap(256);
    for (int b = 0; b < 256; ++b) {
        const int c = ht.cx_cmap[b];
        std::vector<int> key;
        for (int p = 0; p < P; ++p) {
            key.push_back(out[(size_t)rep[p] * nc + c]);
            key.push_back(ren[cls[nxt[(size_t)rep[p] * nc + c]]]);
        }
        cmap[b] = cols.emplace(key, (int)cols.size()).first->second;
    }
    const int npc = (int)cols.size();
    if (npc * 4 > 255 || (long long)P * npc * 4 > 65536) return false;
    if (cx_pa_smem_bytes(P, npc, true) > cx_dyn_smem_limit()) return false;
    std::vector<int> col_rep(npc, -1);
    for (int b = 0; b < 256; ++b)
        if (col_rep[cmap[b]] < 0) col_rep[cmap[b]] = ht.cx_cmap[b];
    ht.pa.assign((size_t)P * npc, 0);
    for (int p = 0; p < P; ++p)
        for (int k = 0; k < npc; ++k) {
            const int c = col_rep[k];
            const int o = out[(size_t)rep[p] * nc + c];
            const int to = ren[cls[nxt[(size_t)rep[p] * nc + c]]];
            uint32_t e = (uint32_t)(to * npc * 4);
            if (o & (1 << 11)) e |= 1u << 31;
            else e |= (uint32_t)(o & 0xff) << 16;
            e |= (uint32_t)((o >> 8) & 7) << 24;
            ht.pa[(size_t)p * npc + k] = e;
        }
    ht.pa_states = P;
    ht.pa_cols = npc;
    ht.pa_cmap4.resize(256);
    for (int b = 0; b < 256; ++b) ht.pa_cmap4[b] = (uint8_t)(cmap[b] * 4);
    ht.pa_ok = true;
    if (getenv("ZS_VERBOSE"))
        fprintf(stderr, "zs: parse automaton: %d joint states -> %d states x %d columns (%d B)\n", N, P, npc,
                P * npc * 4);
    return true;
}

// The dynamic shared-memory limit of a kernel is one value per device: raise
// it when a launch needs more than the value set so far, and skip the call
// otherwise (it is not free on the per-launch path)
template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
    static std::map<std::pair<const void *, int>, int> limit;  // (kernel, device) -> bytes set
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_pair(reinterpret_cast<const void *>(kernel), dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = limit.find(key);
    if (it != limit.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) limit[key] = bytes;
    return e;
}

typedef void (*TileKernel)(Job, Tables);

TileKernel compress_kernel(int w, bool t2) {
    if (t2) return compress_tiles<8, true>;  // W only sizes the (unused) key window
    switch (w) {
    case 2: return compress_tiles<2, false>;
    case 4: return compress_tiles<4, false>;
    case 6: return compress_tiles<6, false>;
    case 8: return compress_tiles<8, false>;
    default: return compress_tiles<0, false>;
    }
}

typedef void (*BatchKernel)(const uint8_t *, const long long *, long long, uint8_t *, long long *,
                            uint8_t *, unsigned long long *, Tables);
BatchKernel batch_kernel(int w) {
    switch (w) {
    case 2: return batch_compress<2>;
    case 4: return batch_compress<4>;
    case 6: return batch_compress<6>;
    case 8: return batch_compress<8>;
    default: return batch_compress<0>;
    }
}

// one whole-buffer launch (device pointers) on `slot`'s buffers and stream
int run_ll(zs_ctx *ctx, int slot, const uint8_t *d_in, long long n_in, long long nt, int flags, int *n_ll_out,
           int *launches);

int launch_stream(zs_ctx *ctx, int slot, bool compress, const uint8_t *d_in, long long n,
                  uint8_t *d_out, long long out_cap, int flags, bool timed, bool general = false,
                  bool ll = false) {
    const bool cx = compress && (ctx->ht.cx_ok || ctx->ht.kw_ok) && !general && !ctx->no_t2 && !ctx->no_ip;
    const bool fx = !compress && ctx->fx_ok && !general;
    const long long tile = cx ? CX_TILE : fx ? FX_TILE : TILE;
    const long long nt = (n + tile - 1) / tile;
    cudaStream_t st = ctx->stream[slot];
    if (ctx->ctl[slot].reserve(sizeof(Ctl)) || ctx->ts[slot].reserve(sizeof(TileState) * (nt + 1)) ||
        ctx->terr[slot].reserve(sizeof(TileErr) * (nt + 1)))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(tile state)");
    if (!ctx->arena[slot].p && ctx->arena[slot].reserve(64ull << 20))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(arena)");
    CK(cudaMemsetAsync(ctx->ctl[slot].p, 0, sizeof(Ctl), st));
    // err_key starts at ~0
    CK(cudaMemsetAsync((char *)ctx->ctl[slot].p + offsetof(Ctl, err_key), 0xff, 8, st));
    CK(cudaMemsetAsync(ctx->ts[slot].p, 0, sizeof(TileState) * (nt + 1), st));
    Job job;
    job.in = d_in;
    job.n = n;
    job.out = d_out;
    job.out_cap = out_cap;
    job.preprocess = (flags & ZS_F_PREPROCESS) ? 1 : 0;
    job.lenient = (flags & ZS_F_LENIENT) ? 1 : 0;
    job.n_tiles = nt;
    job.ctl = ctx->ctl[slot].as<Ctl>();
    job.ts = ctx->ts[slot].as<TileState>();
    job.terr = ctx->terr[slot].as<TileErr>();
    job.arena = ctx->arena[slot].as<uint8_t>();
    job.arena_cap = (long long)ctx->arena[slot].cap;
    job.timing = ctx->timing;
    ctx->nk[slot] = nt > 0 ? 1 : 0;
    // long lines: mode 0 records them (a re-run codes them first, mode 1)
    const bool ll_ok = cx && ctx->ht.pa_ok && ctx->ht.cx_ok && !ctx->no_pa && !ctx->no_ll && nt > 0;
    int ll_n = 0, ll_launches = 0;
    if (ll_ok) {
        if (ctx->ll[slot].reserve(sizeof(LLine) * LL_CAP) || ctx->tl[slot].reserve(sizeof(long long) * nt))
            return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(long lines)");
        if (ll) {
            if (int rc = run_ll(ctx, slot, d_in, n, nt, flags, &ll_n, &ll_launches)) return rc;
        }
        job.ll = ctx->ll[slot].as<LLine>();
        job.tl = ctx->tl[slot].as<long long>();
        job.ll_cap = LL_CAP;
        job.ll_mode = ll ? 1 : 0;
        job.ll_n = ll_n;
    }
    if (nt > 0) {
        const int grid = (int)std::min<long long>(nt, ctx->n_sm);
        if (timed) CK(cudaEventRecord(ctx->ev0, st));
        if (cx) {
            const bool kw = !ctx->ht.cx_ok;
            const bool pa = ctx->ht.pa_ok && !kw && !ctx->no_pa;
            const int ctas = pa && !ctx->slices ? cx_ctas<true, false>() : cx_ctas<true, true>();
            const int g2 = (int)std::min<long long>(nt, (long long)ctx->n_sm * ctas);
            if (pa) {
                const int smem = cx_pa_smem_bytes(ctx->ht.pa_states, ctx->ht.pa_cols, ctx->slices != 0);
                auto k = ctx->slices ? compress_cx<true, true> : compress_cx<true, false>;
                CK(set_smem(k, smem));
                CxTables ct{nullptr, nullptr, nullptr, ctx->d_pacmap.as<uint8_t>(), ctx->ht.pa_states, 0,
                            ctx->ht.pa_cols, 0, 0, ctx->p4_lane ? 0 : 1, 0, smem, ctx->d_pa.as<uint32_t>()};
                k<<<g2, CX_NT, smem, st>>>(job, ctx->tb, ct);
                ctx->last_kernel = ctx->slices ? "compress_cx<slices>" : "compress_cx";
                if (ll && ll_n > 0) {  // the coded long lines to the offsets compress_cx reserved
                    ll_place<<<dim3(ll_n, std::max(1, std::min(512, 4096 / ll_n))), LL_NT, 0, st>>>(job.ll, ll_n, ctx->llo[slot].as<uint8_t>(),
                                                              d_out, out_cap);
                    ++ll_launches;
                    static const bool trace = getenv("ZS_LL_TRACE") != nullptr;
                    if (trace) {  // measurement / debug aid: the coded lines after placement
                        std::vector<LLine> L(ll_n);
                        CK(cudaStreamSynchronize(st));
                        CK(cudaMemcpy(L.data(), job.ll, sizeof(LLine) * ll_n, cudaMemcpyDeviceToHost));
                        for (const auto &l : L)
                            fprintf(stderr, "zs_ll ge %lld gs %lld nblk %d ev %d+%d status %d cost %lld esc %lld "
                                    "obase %lld dst %lld\n", l.ge, l.gs, l.nblk, l.ev0, l.nev, l.status, l.cost,
                                    l.esc, l.obase, l.dst);
                    }
                }
                ctx->nk[slot] += ll_launches;
            } else {
                const CxLayout L = kw ? cx_layout(ctx->ht.kw_states, 0, 2 * ctx->ht.kw_cols)
                                      : cx_layout(ctx->ht.cx_states, ctx->ht.n_windows, ctx->ht.cx_cols);
                const int smem = L.bytes + (kw ? cx_kw_ring_bytes() : 0);
                CK(set_smem(compress_cx<false, false>, smem));
                CxTables ct{ctx->d_cxdfa.as<uint16_t>(), kw ? nullptr : ctx->d_cxt2.as<uint16_t>(),
                            ctx->d_cxcodes.as<uint8_t>(), ctx->d_cxcmap.as<uint8_t>(),
                            kw ? ctx->ht.kw_states : ctx->ht.cx_states, kw ? 0 : ctx->ht.n_windows,
                            kw ? 2 * ctx->ht.kw_cols : ctx->ht.cx_cols, L.o_t2, L.o_codes, ctx->p4_lane ? 0 : 1,
                            kw ? 1 : 0, L.bytes, nullptr};
                compress_cx<false, false><<<g2, CX_NT, smem, st>>>(job, ctx->tb, ct);
                ctx->last_kernel = kw ? "compress_cx<kw16>" : "compress_cx<t2>";
            }
        } else if (compress) {
            const bool t2 = ctx->fast_w && ctx->ht.t2_ok && !ctx->no_t2;
            TileKernel k = compress_kernel(ctx->fast_w, t2);
            const int smem = compress_smem_bytes(ctx->fast_w ? ctx->tb.n_states : 0,
                                                 t2 ? ctx->ht.n_windows : 0);
            CK(set_smem(k, smem));
            k<<<grid, NT, smem, st>>>(job, ctx->tb);
            ctx->last_kernel = ctx->fast_w ? (t2 ? "compress_tiles<W,t2>" : "compress_tiles<W>")
                                           : "compress_tiles<0>";
        } else if (fx) {
            const bool al = (reinterpret_cast<uintptr_t>(d_in) & 15) == 0;
            const bool wide = ctx->tb.max_exp > 7;
            if (ctx->fxs[slot].reserve(fx_scratch_bytes(nt)))
                return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(fx scratch)");
            const FxScratch sc = fx_carve(ctx->fxs[slot].p, nt);
            auto kc = al ? fx_count<true> : fx_count<false>;
            auto ke = wide ? (al ? fx_emit<true, true> : fx_emit<false, true>)
                           : (al ? fx_emit<true, false> : fx_emit<false, false>);
            const int esm = fx_emit_smem(wide);
            CK(set_smem(kc, FX_CNT_SMEM));
            CK(set_smem(ke, esm));
            if (!ctx->fx_blocks[0] || ctx->fx_wide != (int)wide) {
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->fx_blocks[0], kc, FX_NT, FX_CNT_SMEM));
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->fx_blocks[1], ke, FX_NT, esm));
                ctx->fx_wide = (int)wide;
            }
            auto grid_of = [&](int b) { return (int)std::min<long long>(nt, (long long)ctx->n_sm * std::max(1, b)); };
            kc<<<grid_of(ctx->fx_blocks[0]), FX_NT, FX_CNT_SMEM, st>>>(job, ctx->d_fxc.as<unsigned>(), sc);
            fx_scan<<<1, 1024, 0, st>>>(job, sc);
            ke<<<grid_of(ctx->fx_blocks[1]), FX_NT, esm, st>>>(job, ctx->d_fxe.as<unsigned long long>(), sc);
            ctx->last_kernel = "fx_count+fx_scan+fx_emit";
            ctx->nk[slot] = 3;
        } else {
            const int smem = bp_smem_bytes(ctx->tb.n_flat);
            CK(set_smem(decompress_tiles_bp, smem));
            decompress_tiles_bp<<<grid, NT, smem, st>>>(job, ctx->tb);
            ctx->last_kernel = "decompress_tiles_bp";
        }
        CK(cudaGetLastError());
        if (timed) CK(cudaEventRecord(ctx->ev1, st));
    }
    CK(cudaMemcpyAsync(&ctx->h_ctl[slot], ctx->ctl[slot].p, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(ctx->ev_ctl[slot], st));
    return ZS_OK;
}

// Long lines (zs_ll.cuh): code the lines compress_cx recorded on `slot` in
// its last run (mode 0) with the block-parallel kernels, on the slot's
// stream; the host reads back the few sizes it allocates by.  On return the
// slot's line list holds, sorted by ge, every recorded line with its output
// size (or LL_FALLBACK) for compress_cx's mode 1.
int run_ll(zs_ctx *ctx, int slot, const uint8_t *d_in, long long n_in, long long nt, int flags, int *n_ll_out,
           int *launches) {
    cudaStream_t st = ctx->stream[slot];
    const int n_ll = (int)std::min<unsigned long long>(ctx->h_ctl[slot].ll_n, (unsigned long long)LL_CAP);
    *n_ll_out = n_ll;
    if (n_ll == 0) return ZS_OK;
    LLine *d_ln = ctx->ll[slot].as<LLine>();
    std::vector<LLine> L(n_ll);
    // ZS_LL_TRACE: host time at each round trip (a measurement aid)
    static const bool trace = getenv("ZS_LL_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    int trips = 0;
    auto d2h = [&](void *dst, const void *src, size_t bytes) -> int {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (trace)
            fprintf(stderr, "zs_ll trip %d at %.1f us\n", ++trips,
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
        return ZS_OK;
    };
    if (int rc = d2h(L.data(), d_ln, sizeof(LLine) * n_ll)) return rc;
    std::sort(L.begin(), L.end(), [](const LLine &a, const LLine &b) { return a.ge < b.ge; });
    CK(cudaMemcpyAsync(d_ln, L.data(), sizeof(LLine) * n_ll, cudaMemcpyHostToDevice, st));
    ll_setup<<<(n_ll * 32 + 255) / 256, 256, 0, st>>>(d_ln, n_ll, ctx->tl[slot].as<long long>(), nt, CX_TILE);
    int nk = 1;
    if (int rc = d2h(L.data(), d_ln, sizeof(LLine) * n_ll)) return rc;
    // blocks of 256 bytes per line, within the per-launch byte budget
    long long bytes = 0;
    int nb = 0;
    for (auto &l : L) {
        const long long len = l.ge - l.gs;
        l.blk0 = nb;
        l.nblk = 0;
        l.ev0 = l.nev = 0;
        if (len <= 0 || len >= (1ll << 30) || bytes + len > LL_MAXBYTES) {
            l.status = LL_FALLBACK;
            continue;
        }
        l.nblk = (int)((len + LL_B - 1) / LL_B);
        nb += l.nblk;
        bytes += len;
    }
    CK(cudaMemcpyAsync(d_ln, L.data(), sizeof(LLine) * n_ll, cudaMemcpyHostToDevice, st));
    if (nb == 0) {
        CK(cudaStreamSynchronize(st));
        *launches += nk;
        return ZS_OK;
    }
    // Buffers at their worst case for `bytes` line bytes (a byte starts at
    // most one ring token; a 1-byte token grows to 3; an escape doubles), so
    // the passes below queue without host round trips.  Per block: map, cnt,
    // rlen, pin, pout, g, x, ocnt, oesc, ooff (4 B) and par (16 B), nb + 1 each.
    const size_t nb1 = (size_t)nb + 1, a4 = (nb1 * 4 + 15) & ~(size_t)15;
    const size_t ne = (size_t)bytes + 1, e4 = (ne * 4 + 15) & ~(size_t)15, e2 = (ne * 2 + 15) & ~(size_t)15;
    const size_t nseg = (ne + LL_SEG - 1) / LL_SEG;
    const size_t rcap = 3 * (size_t)bytes + 64, ocap = 2 * rcap + (size_t)n_ll + 64;
    const bool pre = (flags & ZS_F_PREPROCESS) != 0;
    if (ctx->llb[slot].reserve(a4 * 10 + nb1 * 16 + 64) ||
        (pre && (ctx->lle[slot].reserve(2 * e4 + e2 + ne + 64) ||
                 ctx->llc[slot].reserve(nseg * LL_CS * 8))) ||
        ctx->llr[slot].reserve(rcap) || ctx->lld[slot].reserve(rcap) || ctx->llo[slot].reserve(ocap))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(long lines)");
    uint8_t *pb = ctx->llb[slot].as<uint8_t>();
    LLWork W{};
    W.in = d_in;
    W.n = n_in;
    W.ln = d_ln;
    W.n_ll = n_ll;
    W.nb = nb;
    W.preprocess = pre ? 1 : 0;
    W.map = reinterpret_cast<unsigned *>(pb);
    W.cnt = reinterpret_cast<int *>(pb + a4);
    W.rlen = reinterpret_cast<int *>(pb + 2 * a4);
    W.pin = reinterpret_cast<unsigned *>(pb + 3 * a4);
    W.pout = reinterpret_cast<unsigned *>(pb + 4 * a4);
    W.g = reinterpret_cast<int *>(pb + 5 * a4);
    W.x = reinterpret_cast<int *>(pb + 6 * a4);
    W.ocnt = reinterpret_cast<int *>(pb + 7 * a4);
    W.oesc = reinterpret_cast<int *>(pb + 8 * a4);
    W.ooff = reinterpret_cast<int *>(pb + 9 * a4);
    W.par = reinterpret_cast<uint4 *>(pb + 10 * a4);
    int *flag = reinterpret_cast<int *>(pb + 10 * a4 + nb1 * 16);  // fix-loop flags: colour, parse, emit
    if (pre) {
        uint8_t *pe = ctx->lle[slot].as<uint8_t>();
        W.epos = reinterpret_cast<int *>(pe);
        W.epart = reinterpret_cast<int *>(pe + e4);
        W.eflag = reinterpret_cast<uint16_t *>(pe + 2 * e4);
        W.ecol = pe + 2 * e4 + e2;
    }
    int *exits = pre ? ctx->llc[slot].as<int>() : nullptr;
    int *assumed = pre ? exits + nseg * LL_CS : nullptr;
    W.R = ctx->llr[slot].as<uint8_t>();
    W.D = ctx->lld[slot].as<uint8_t>();
    W.O = ctx->llo[slot].as<uint8_t>();
    W.pa = ctx->d_pa.as<uint32_t>();
    W.cmap = ctx->d_pacmap.as<uint8_t>();
    W.pa_words = ctx->ht.pa_states * ctx->ht.pa_cols;
    W.explen = ctx->tb.exp_len;
    if (!ctx->d_lltok.p) {
        LLTok T;
        ll_tok_build(T);
        if (ctx->d_lltok.reserve(sizeof T)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(tokenizer)");
        CK(cudaMemcpy(ctx->d_lltok.p, &T, sizeof T, cudaMemcpyHostToDevice));
    }
    W.tok = ctx->d_lltok.as<LLTok>();
    W.ecap = pre ? (long long)ne : 0;
    W.rcap = (long long)rcap;
    W.ocap = (long long)ocap;
    const int gb = (nb + LL_NT - 1) / LL_NT;
    const int gseg = (int)((nseg + LL_NT - 1) / LL_NT);
    const int pa_smem = W.pa_words * 4;
    CK(set_smem(ll_parse, pa_smem));
    CK(set_smem(ll_parse_fix, pa_smem));
    // a fix pass per stage: the flag tells whether the pass changed an exit
    auto colour_pass = [&](int pass) -> int {
        W.changed = flag;
        CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
        ll_colour<<<gseg, LL_NT, 0, st>>>(W, (int)(ne - 1), pass, exits, assumed);
        ++nk;
        return ZS_OK;
    };
    auto parse_pass = [&]() -> int {
        W.changed = flag + 1;
        CK(cudaMemsetAsync(flag + 1, 0, sizeof(int), st));
        ll_parse_fix<<<gb, LL_NT, pa_smem, st>>>(W);
        ++nk;
        return ZS_OK;
    };
    auto emit_pass = [&]() -> int {
        W.changed = flag + 2;
        CK(cudaMemsetAsync(flag + 2, 0, sizeof(int), st));
        ll_emit_fix<<<gb, LL_NT, 0, st>>>(W);
        ++nk;
        return ZS_OK;
    };
    auto settle = [&](int which, const std::function<int()> &pass) -> int {
        for (int changed = 1; changed;) {
            if (int rc = pass()) return rc;
            if (int rc = d2h(&changed, flag + which, sizeof(int))) return rc;
        }
        return ZS_OK;
    };
    // stage 0: tokens, events, colours
    if (pre) {
        ll_tok_map<true><<<gb, LL_NT, 0, st>>>(W);
        ll_scan<LLMap><<<1, LL_SNT, 0, st>>>(W.map, W.map, nb);
        ll_tok_count<<<gb, LL_NT, 0, st>>>(W);
        ll_scan<LLAdd><<<1, LL_SNT, 0, st>>>(W.cnt, W.cnt, nb);
        ll_scan<LLXor><<<1, LL_SNT, 0, st>>>(W.par, W.par, nb);
        ll_tok_events<<<gb, LL_NT, 0, st>>>(W);
        // ne - 1 = the events bound; ll_pair / ll_colour stop at the real count
        ll_pair<<<(int)((ne - 1 + LL_NT - 1) / LL_NT), LL_NT, 0, st>>>(W, (int)(ne - 1));
        nk += 7;
        if (int rc = colour_pass(0)) return rc;
        ll_umin<<<1, LL_SNT, 0, st>>>(W, (int)(ne - 1), assumed);
        ++nk;
        for (int pass = 0; pass < 3; ++pass)
            if (int rc = colour_pass(1)) return rc;
    } else {
        ll_tok_map<false><<<gb, LL_NT, 0, st>>>(W);
        ++nk;
    }
    // stages 1-3 queue with two fix passes each; one round trip checks that
    // the last pass of each changed nothing (else that stage settles and
    // everything after it runs again)
    for (int from = 1;;) {
        if (from <= 1) {
            ll_rlen<<<gb, LL_NT, 0, st>>>(W);
            ll_scan<LLAdd><<<1, LL_SNT, 0, st>>>(W.rlen, W.rlen, nb);
            ll_rewrite<<<gb, LL_NT, 0, st>>>(W);
            ll_parse<<<gb, LL_NT, pa_smem, st>>>(W);
            nk += 4;
            for (int k = 0; k < 2; ++k)
                if (int rc = parse_pass()) return rc;
        }
        if (from <= 2) {
            ll_emit_count<<<gb, LL_NT, 0, st>>>(W);
            ++nk;
            for (int k = 0; k < 2; ++k)
                if (int rc = emit_pass()) return rc;
        }
        ll_scan<LLAdd><<<1, LL_SNT, 0, st>>>(W.ocnt, W.ooff, nb);
        ll_emit_write<<<gb, LL_NT, 0, st>>>(W);
        nk += 2;
        int f[3] = {0, 0, 0};
        if (int rc = d2h(f, flag, sizeof f)) return rc;
        if (pre && f[0]) {  // colours still moving: settle them, then redo everything after
            if (int rc = settle(0, [&] { return colour_pass(1); })) return rc;
            from = 1;
            CK(cudaMemsetAsync(flag, 0, sizeof(int), st));
            continue;
        }
        if (f[1]) {
            if (int rc = settle(1, parse_pass)) return rc;
            from = 2;
            continue;
        }
        if (f[2]) {
            if (int rc = settle(2, emit_pass)) return rc;
            from = 3;
            continue;
        }
        break;
    }
    CK(cudaGetLastError());
    *launches += nk;
    return ZS_OK;
}

// Fill res from a finished slot; returns ZS_OK, or 1 = re-run needed
// (arena exhausted), 2 = output capacity exceeded.
int collect(zs_ctx *ctx, int slot, long long n, const uint8_t *h_last_byte_src, bool trailing,
            long long line_base, zs_result *res, bool accumulate) {
    const Ctl &c = ctx->h_ctl[slot];
    if (c.overflow & 2ull) {
        size_t need = (size_t)c.arena_used * 2 + (64ull << 20);
        ctx->arena[slot].release();
        if (ctx->arena[slot].reserve(need)) return fail(ctx, cudaErrorMemoryAllocation, "arena");
        return 1;
    }
    (void)h_last_byte_src;
    if (c.overflow & 12ull) return 3;  // fast kernel met a case it hands over: re-run the general one
    if (c.overflow & 16ull) return 4;  // long lines recorded: code them, run again (mode 1)
    zs_result r{};
    r.lines = (long long)c.lines;
    r.in_bytes = n;
    r.out_bytes = (long long)c.total_out;
    if (!trailing && r.lines > 0) r.out_bytes -= 1;
    r.escapes = (long long)c.escapes;
    r.skipped = (long long)c.skipped;
    r.flagged = (long long)c.flagged;
    if (c.err_key != ~0ull) {
        const long long line_idx = (long long)(c.err_key >> 24);
        const long long tile = (long long)(c.err_key & 0xffffff);
        TileErr e;
        cudaError_t ce = cudaMemcpy(&e, ctx->terr[slot].as<TileErr>() + tile, sizeof e,
                                    cudaMemcpyDeviceToHost);
        if (ce != cudaSuccess) return fail(ctx, ce, "cudaMemcpy(terr)");
        r.err_line = line_base + line_idx + 1;
        r.err_kind = e.kind;
        r.err_code = e.code;
        r.err_offset = e.offset;
        r.err_ids[0] = e.ids[0];
        r.err_ids[1] = e.ids[1];
    }
    if (accumulate) {
        res->lines += r.lines;
        res->in_bytes += r.in_bytes;
        res->out_bytes += r.out_bytes;
        res->escapes += r.escapes;
        res->skipped += r.skipped;
        res->flagged += r.flagged;
        if (!res->err_line && r.err_line) {
            res->err_line = r.err_line;
            res->err_kind = r.err_kind;
            res->err_code = r.err_code;
            res->err_offset = r.err_offset;
            res->err_ids[0] = r.err_ids[0];
            res->err_ids[1] = r.err_ids[1];
        }
        res->gpu_launches += ctx->nk[slot];
    } else {
        r.gpu_launches = ctx->nk[slot];
        *res = r;
    }
    return (c.overflow & 1ull) ? 2 : ZS_OK;
}

// The long-line buffers are sized for the worst case of the lines' bytes; a
// call that needed more than 1 GB of them gives it back.
void ll_trim(zs_ctx *ctx) {
    for (int s = 0; s < zs_ctx::NSLOT; ++s) {
        size_t tot = 0;
        for (DevBuf *b : {&ctx->llb[s], &ctx->lle[s], &ctx->llc[s], &ctx->llr[s], &ctx->lld[s], &ctx->llo[s]})
            tot += b->cap;
        if (tot > (1ull << 30))
            for (DevBuf *b : {&ctx->llb[s], &ctx->lle[s], &ctx->llc[s], &ctx->llr[s], &ctx->lld[s], &ctx->llo[s]})
                b->release();
    }
}

int run_device_(zs_ctx *ctx, bool compress, const uint8_t *d_in, int64_t n, uint8_t *d_out,
                int64_t out_cap, int flags, zs_result *res) {
    if (!ctx || !res || n < 0 || (n > 0 && !d_in)) return ZS_E_ARG;
    if (!ctx->have_dict) return ZS_E_NODICT;
    CK(cudaSetDevice(ctx->dev));
    memset(res, 0, sizeof *res);
    if (int rc = after_user_stream(ctx)) return rc;
    // the input's last byte (the trailing-newline rule) arrives with the
    // results: an async copy into pinned memory, read after the call's sync
    if (n > 0) CK(cudaMemcpyAsync(ctx->h_last, d_in + n - 1, 1, cudaMemcpyDeviceToHost, ctx->stream[0]));
    bool general = false, ll = false;
    for (int attempt = 0; attempt < 6; ++attempt) {
        int rc = launch_stream(ctx, 0, compress, d_in, n, d_out, out_cap, flags, true, general, ll);
        if (rc) return rc;
        CK(cudaEventSynchronize(ctx->ev_ctl[0]));
        if (n > 0) CK(cudaEventElapsedTime(&ctx->last_ms, ctx->ev0, ctx->ev1));
        const bool trailing = n == 0 || *ctx->h_last == '\n';
        rc = collect(ctx, 0, n, nullptr, trailing, 0, res, false);
        if (rc == 1) continue;  // arena grown, re-run
        if (rc == 3) {          // bad record: the record-aware kernel decides
            general = true;
            continue;
        }
        if (rc == 4) {          // long lines: the block-parallel long-line kernels first
            ll = true;
            continue;
        }
        if (rc == 2) {
            res->out_bytes = (long long)ctx->h_ctl[0].total_out;
            return ZS_E_CAPACITY;
        }
        return rc;
    }
    ctx->err = "arena re-run limit";
    return ZS_E_NOMEM;
}

int run_device(zs_ctx *ctx, bool compress, const uint8_t *d_in, int64_t n, uint8_t *d_out,
               int64_t out_cap, int flags, zs_result *res) {
    const int rc = run_device_(ctx, compress, d_in, n, d_out, out_cap, flags, res);
    if (ctx) ll_trim(ctx);
    return rc;
}

// Host-buffer chunk boundaries, each just past a newline.  Sizes ramp up
// from ch/16 (the first D2H / kernel starts after a short H2D) to ch and back
// down over the last ~ch bytes (a short tail of kernel + D2H after the last
// H2D).  cuts[0] = 0, cuts.back() = n.
std::vector<long long> chunk_cuts(const uint8_t *h_in, long long n, long long ch) {
    const long long lo = std::max<long long>(ch >> 4, 1 << 18);
    long long up = lo;
    std::vector<long long> cuts{0};
    while (cuts.back() < n) {
        const long long s = cuts.back(), rem = n - s;
        long long size = std::min(up, ch);
        up = std::min(2 * up, ch);  // (unclamped doubling overflowed after ~41 chunks)
        if (rem < 2 * size) size = std::max(lo, rem / 2);
        long long e = std::min<long long>(n, s + size);
        if (e < n) {
            const void *nl = memchr(h_in + e, '\n', (size_t)(n - e));
            e = nl ? (long long)((const uint8_t *)nl - h_in) + 1 : n;
        }
        cuts.push_back(e);
    }
    return cuts;
}

// Host-buffer pipeline: newline-aligned chunks, NSLOT slots on NSLOT streams so
// chunk k+1's H2D and kernel overlap chunk k's D2H.
int run_host_(zs_ctx *ctx, bool compress, const uint8_t *h_in, int64_t n, uint8_t *h_out,
              int64_t out_cap, int flags, zs_result *res);

int run_host(zs_ctx *ctx, bool compress, const uint8_t *h_in, int64_t n, uint8_t *h_out,
             int64_t out_cap, int flags, zs_result *res) {
    const int rc = run_host_(ctx, compress, h_in, n, h_out, out_cap, flags, res);
    if (ctx) {
        for (int s = 0; s < zs_ctx::NSLOT; ++s) cudaStreamSynchronize(ctx->stream[s]);  // (error paths return early)
        ll_trim(ctx);
    }
    return rc;
}

int run_host_(zs_ctx *ctx, bool compress, const uint8_t *h_in, int64_t n, uint8_t *h_out,
              int64_t out_cap, int flags, zs_result *res) {
    if (!ctx || !res || n < 0 || (n > 0 && !h_in)) return ZS_E_ARG;
    if (!ctx->have_dict) return ZS_E_NODICT;
    CK(cudaSetDevice(ctx->dev));
    memset(res, 0, sizeof *res);
    const bool trailing = n == 0 || h_in[n - 1] == '\n';
    // newline-aligned chunks small enough that chunk k's D2H overlaps chunk
    // k+1's H2D and kernel (ZS_CHUNK_MB overrides, for measurements)
    static const long long CH = [] {
        const char *e = getenv("ZS_CHUNK_MB");
        const long long mb = e ? atoll(e) : 64;
        return (mb > 0 ? mb : 64) << 20;
    }();
    const long long ch = compress ? CH : std::max<long long>(CH * 3 / 8, 1 << 20);
    const std::vector<long long> cuts = chunk_cuts(h_in, n, ch);
    const int nch = (int)cuts.size() - 1;
    // ZS_TRACE=1: per-chunk event timeline on stderr (H2D end, kernel end,
    // D2H end, ms from the call's start) -- a measurement aid
    static const bool trace = getenv("ZS_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    if (trace) {
        tev.resize(1 + 3 * (size_t)nch);
        for (auto &e : tev) cudaEventCreate(&e);
        cudaEventRecord(tev[0], ctx->stream[0]);
    }
    auto mark = [&](int k, int what, int slot) {
        if (trace) cudaEventRecord(tev[1 + 3 * k + what], ctx->stream[slot]);
    };
    std::vector<int> chunk_of_slot(zs_ctx::NSLOT, -1);
    long long written = 0, line_base = 0;
    bool general = false;  // a chunk hit a bad record: its re-runs (and later re-runs) use the record-aware kernel
    bool capacity_hit = false;
    int pending = -1;  // slot whose output is waiting for D2H
    long long pend_len = 0, pend_n = 0;
    auto out_bound = [&](long long m) {
        return compress ? 2 * m + 64 : std::max<long long>(4 * m, 1 << 20);
    };
    auto finish = [&](int slot, long long cn, long long clen) -> int {
        // wait for ctl, then D2H this chunk's output
        CK(cudaEventSynchronize(ctx->ev_ctl[slot]));
        zs_result r{};
        int rc = collect(ctx, slot, cn, nullptr, true, line_base, &r, false);
        if (rc < 0) return rc;
        (void)clen;
        if (rc >= 1 && rc <= 4) return 10 + rc;  // caller re-runs this chunk synchronously
        long long ob = (long long)ctx->h_ctl[slot].total_out;
        if (!capacity_hit && written + ob <= out_cap && ob > 0 && !r.err_line)
            CK(cudaMemcpyAsync(h_out + written, ctx->out[slot].p, ob, cudaMemcpyDeviceToHost,
                               ctx->stream[slot]));
        mark(chunk_of_slot[slot], 2, slot);
        if (written + ob > out_cap) capacity_hit = true;
        CK(cudaEventRecord(ctx->ev_out[slot], ctx->stream[slot]));
        written += ob;
        res->lines += r.lines;
        res->escapes += r.escapes;
        res->skipped += r.skipped;
        res->flagged += r.flagged;
        res->gpu_launches += ctx->nk[slot];
        if (!res->err_line && r.err_line) {
            res->err_line = r.err_line;
            res->err_kind = r.err_kind;
            res->err_code = r.err_code;
            res->err_offset = r.err_offset;
            res->err_ids[0] = r.err_ids[0];
            res->err_ids[1] = r.err_ids[1];
        }
        line_base += (long long)ctx->h_ctl[slot].in_lines;
        return ZS_OK;
    };
    for (int k = 0; k < nch && !res->err_line; ++k) {
        const int slot = k % zs_ctx::NSLOT;
        const long long cs = cuts[k], cn = cuts[k + 1] - cs;
        // slot reuse: its previous output copy must be done
        CK(cudaEventSynchronize(ctx->ev_out[slot]));
        if (ctx->in[slot].reserve(cn + 16) || ctx->out[slot].reserve(out_bound(cn)))
            return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(chunk)");
        CK(cudaMemcpyAsync(ctx->in[slot].p, h_in + cs, cn, cudaMemcpyHostToDevice, ctx->stream[slot]));
        chunk_of_slot[slot] = k;
        mark(k, 0, slot);
        int rc = launch_stream(ctx, slot, compress, ctx->in[slot].as<uint8_t>(), cn,
                               ctx->out[slot].as<uint8_t>(), (long long)ctx->out[slot].cap, flags,
                               false);
        if (rc) return rc;
        mark(k, 1, slot);
        if (pending >= 0) {
            rc = finish(pending, pend_n, pend_len);
            bool ll_chunk = false;
            while (rc >= 10) {  // re-run the previous chunk synchronously with bigger buffers
                const int ps = pending;
                CK(cudaStreamSynchronize(ctx->stream[ps]));
                if (rc == 12 && ctx->out[ps].reserve((size_t)ctx->h_ctl[ps].total_out + 64))
                    return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(out)");
                CK(cudaMemcpyAsync(ctx->in[ps].p, h_in + cuts[k - 1], pend_n, cudaMemcpyHostToDevice,
                                   ctx->stream[ps]));
                general |= rc == 13;
                ll_chunk |= rc == 14;
                rc = launch_stream(ctx, ps, compress, ctx->in[ps].as<uint8_t>(), pend_n,
                                   ctx->out[ps].as<uint8_t>(), (long long)ctx->out[ps].cap, flags, false,
                                   general, ll_chunk && !general);
                if (rc) return rc;
                rc = finish(ps, pend_n, pend_len);
            }
            if (rc) return rc;
        }
        pending = slot;
        pend_n = cn;
    }
    if (pending >= 0 && !res->err_line) {
        int rc = finish(pending, pend_n, pend_len);
        bool ll_chunk = false;
        while (rc >= 10) {
            const int ps = pending;
            CK(cudaStreamSynchronize(ctx->stream[ps]));
            if (rc == 12 && ctx->out[ps].reserve((size_t)ctx->h_ctl[ps].total_out + 64))
                return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(out)");
            CK(cudaMemcpyAsync(ctx->in[ps].p, h_in + cuts[nch - 1], pend_n, cudaMemcpyHostToDevice,
                               ctx->stream[ps]));
            general |= rc == 13;
            ll_chunk |= rc == 14;
            rc = launch_stream(ctx, ps, compress, ctx->in[ps].as<uint8_t>(), pend_n,
                               ctx->out[ps].as<uint8_t>(), (long long)ctx->out[ps].cap, flags, false,
                               general, ll_chunk && !general);
            if (rc) return rc;
            rc = finish(ps, pend_n, pend_len);
        }
        if (rc) return rc;
    }
    for (int s = 0; s < zs_ctx::NSLOT; ++s) CK(cudaStreamSynchronize(ctx->stream[s]));
    if (trace) {
        for (int k = 0; k < nch; ++k) {
            float t[3] = {0, 0, 0};
            for (int w = 0; w < 3; ++w) cudaEventElapsedTime(&t[w], tev[0], tev[1 + 3 * k + w]);
            fprintf(stderr, "zs_trace %s chunk %d %lld B: h2d %.3f kernel %.3f d2h %.3f ms\n",
                    compress ? "c" : "d", k, cuts[k + 1] - cuts[k], t[0], t[1], t[2]);
        }
        for (auto &e : tev) cudaEventDestroy(e);
    }
    res->in_bytes = n;
    res->out_bytes = written;
    if (!trailing && res->lines > 0) res->out_bytes -= 1;
    if (capacity_hit) return ZS_E_CAPACITY;
    return ZS_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int zs_device_count(int *n) {
    if (!n) return ZS_E_ARG;
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        *n = 0;
        return ZS_E_CUDA;
    }
    return ZS_OK;
}

int zs_ctx_create(int device, zs_ctx **out) {
    if (!out) return ZS_E_ARG;
    *out = nullptr;
    zs_ctx *ctx = new zs_ctx();
    ctx->dev = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, device);
    for (int s = 0; s < zs_ctx::NSLOT && e == cudaSuccess; ++s) {
        e = cudaStreamCreateWithFlags(&ctx->stream[s], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_ctl[s], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_out[s], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_out[s], ctx->stream[s]);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_user, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&ctx->ev1);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_ctl, zs_ctx::NSLOT * sizeof(Ctl));
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_last, 16);
    if (e != cudaSuccess) {
        delete ctx;
        return ZS_E_CUDA;
    }
    *out = ctx;
    return ZS_OK;
}

int zs_ctx_destroy(zs_ctx *ctx) {
    if (!ctx) return ZS_OK;
    cudaSetDevice(ctx->dev);
    for (DevBuf *b : {&ctx->d_dfa2, &ctx->d_t2, &ctx->d_dfa, &ctx->d_codes, &ctx->d_children, &ctx->d_term, &ctx->d_explen,
                      &ctx->d_expoff, &ctx->d_expflat, &ctx->d_fxc, &ctx->d_fxe, &ctx->d_cxdfa, &ctx->d_cxt2, &ctx->d_cxcodes, &ctx->d_cxcmap, &ctx->ixs, &ctx->s_flat, &ctx->s_starts,
                      &ctx->s_out, &ctx->s_lens, &ctx->s_dec, &ctx->s_stat, &ctx->s_errpos,
                      &ctx->s_tot, &ctx->s_ids, &ctx->s_outst, &ctx->tr.buf, &ctx->tr.run, &ctx->tr.pos[0],
                      &ctx->tr.pos[1], &ctx->tr.key[0], &ctx->tr.key[1], &ctx->tr.lcp, &ctx->tr.runs, &ctx->tr.v,
                      &ctx->tr.ex, &ctx->tr.bstart, &ctx->tr.cand, &ctx->tr.cub, &ctx->tr.nsel, &ctx->tr.rpos,
                      &ctx->tr.rocc, &ctx->tr.rlen, &ctx->tr.rank[0], &ctx->tr.rank[1], &ctx->tr.idx[0],
                      &ctx->tr.idx[1], &ctx->tr.dead, &ctx->tr.child, &ctx->tr.term, &ctx->tr.ctl, &ctx->tr.blk,
                      &ctx->tr.sel})
        b->release();
    for (int s = 0; s < zs_ctx::NSLOT; ++s) {
        for (DevBuf *b : {&ctx->fxs[s], &ctx->ctl[s], &ctx->ts[s], &ctx->terr[s], &ctx->in[s], &ctx->out[s],
                          &ctx->arena[s]})
            b->release();
        if (ctx->stream[s]) cudaStreamDestroy(ctx->stream[s]);
        if (ctx->ev_ctl[s]) cudaEventDestroy(ctx->ev_ctl[s]);
        if (ctx->ev_out[s]) cudaEventDestroy(ctx->ev_out[s]);
    }
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev_user) cudaEventDestroy(ctx->ev_user);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->h_ctl) cudaFreeHost(ctx->h_ctl);
    if (ctx->h_last) cudaFreeHost(ctx->h_last);
    delete ctx;
    return ZS_OK;
}

const char *zs_last_error(zs_ctx *ctx) { return ctx ? ctx->err.c_str() : "no context"; }

float zs_last_kernel_ms(zs_ctx *ctx) { return ctx ? ctx->last_ms : 0.f; }
const char *zs_last_kernel(zs_ctx *ctx) { return ctx ? ctx->last_kernel : ""; }
void *zs_stream(zs_ctx *ctx) { return ctx ? (void *)ctx->stream[0] : nullptr; }

int zs_set_phase_timing(zs_ctx *ctx, int on) {
    if (!ctx) return ZS_E_ARG;
    ctx->timing = on;  // 1: per-phase clocks; 2: lane-range statistics (compress_cx)
    return ZS_OK;
}

int zs_last_phase_cycles(zs_ctx *ctx, uint64_t *cycles8) {
    if (!ctx || !cycles8) return ZS_E_ARG;
    for (int k = 0; k < 8; ++k) cycles8[k] = ctx->h_ctl[0].phase[k];
    return ZS_OK;
}

int zs_set_dictionary(zs_ctx *ctx, const int32_t *children, const int16_t *term_code,
                      int32_t n_nodes, const int32_t *exp_len, const uint8_t *valid,
                      const int64_t *exp_off, const uint8_t *exp_flat) {
    if (!ctx || !children || !term_code || n_nodes < 1 || !exp_len || !valid || !exp_off)
        return ZS_E_ARG;
    CK(cudaSetDevice(ctx->dev));
    HostTables &ht = ctx->ht;
    ht = HostTables();
    ht.n_nodes = n_nodes;
    ht.children.assign(children, children + (size_t)n_nodes * 256);
    ht.term_code.assign(term_code, term_code + n_nodes);
    std::vector<std::pair<std::string, int>> pats;
    trie_patterns(children, term_code, n_nodes, pats);
    ht.max_len = 0;
    for (auto &p : pats) ht.max_len = std::max<int>(ht.max_len, (int)p.first.size());
    ht.fast = build_dfa(pats, ht.max_len, ht);
    ht.cx_ok = ht.kw_ok = false;
    if (ht.fast && build_t2(ht, std::max(1, ht.max_len)) && build_cx(ht, ht.max_len)) build_pa(ht);
    if (!ht.cx_ok && build_kw(pats, ht.max_len, ht)) {
        const CxLayout L = cx_layout(ht.kw_states, 0, 2 * ht.kw_cols);
        ht.kw_ok = L.bytes + cx_kw_ring_bytes() <= cx_dyn_smem_limit();
    }
    // decode tables (dictionary.py:112-129): valid codes have exp_len > 0
    if (exp_off[256] > 65535) {
        ctx->err = "expansion table too large";
        return ZS_E_ARG;
    }
    for (int b = 0; b < 256; ++b) {
        if (valid[b] && (exp_len[b] < 1 || exp_len[b] > 255)) {
            ctx->err = "bad expansion length";
            return ZS_E_ARG;
        }
        ht.exp_len[b] = valid[b] ? (uint8_t)exp_len[b] : 0;
    }
    for (int b = 0; b <= 256; ++b) ht.exp_off[b] = (uint16_t)exp_off[b];
    ht.exp_flat.assign(exp_flat, exp_flat + exp_off[256]);
    ht.exp_flat.resize(ht.exp_flat.size() + 16, 0);
    // upload
    auto up = [&](DevBuf &b, const void *src, size_t bytes) -> cudaError_t {
        cudaError_t e = b.reserve(bytes + 16);
        if (e == cudaSuccess) e = cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice);
        return e;
    };
    CK(up(ctx->d_children, ht.children.data(), ht.children.size() * 4));
    CK(up(ctx->d_term, ht.term_code.data(), ht.term_code.size() * 2));
    CK(up(ctx->d_explen, ht.exp_len, 256));
    CK(up(ctx->d_expoff, ht.exp_off, 257 * 2));
    CK(up(ctx->d_expflat, ht.exp_flat.data(), ht.exp_flat.size()));
    if (ht.fast) {
        CK(up(ctx->d_dfa, ht.dfa.data(), ht.dfa.size() * 2));
        CK(up(ctx->d_codes, ht.codes.data(), ht.codes.size()));
    }
    if (ht.t2_ok) {
        CK(up(ctx->d_dfa2, ht.dfa2.data(), ht.dfa2.size() * 2));
        CK(up(ctx->d_t2, ht.t2.data(), ht.t2.size() * 4));
    }
    if (ht.kw_ok) {
        CK(up(ctx->d_cxcmap, ht.kw_cmap.data(), 256));
        CK(up(ctx->d_cxdfa, ht.kw_dfa.data(), ht.kw_dfa.size() * 4));
        CK(up(ctx->d_cxcodes, ht.kw_codes.data(), ht.kw_codes.size()));
    }
    if (ht.cx_ok) {
        CK(up(ctx->d_cxcmap, ht.cx_cmap.data(), 256));
        CK(up(ctx->d_cxdfa, ht.cx_dfa.data(), ht.cx_dfa.size() * 2));
        CK(up(ctx->d_cxt2, ht.cx_t2.data(), ht.cx_t2.size() * 2));
        CK(up(ctx->d_cxcodes, ht.cx_codes.data(), ht.cx_codes.size()));
    }
    if (ht.pa_ok) {
        CK(up(ctx->d_pa, ht.pa.data(), ht.pa.size() * 4));
        CK(up(ctx->d_pacmap, ht.pa_cmap4.data(), 256));
    }
    {
        unsigned fxc[256];
        unsigned long long fxe[512];
        int mx = 0;
        for (int b = 0; b < 256; ++b) mx = std::max<int>(mx, ht.exp_len[b]);
        const bool wide = mx > 7;
        for (int b = 0; b < 256; ++b) {
            fxc[b] = fx_count_entry(b, ht.exp_len);
            fxe[b] = fx_emit_entry(b, ht.exp_len, ht.exp_off, ht.exp_flat.data(), wide, 0);
            fxe[256 + b] = fx_emit_entry(b, ht.exp_len, ht.exp_off, ht.exp_flat.data(), wide, 1);
        }
        CK(up(ctx->d_fxc, fxc, sizeof fxc));
        CK(up(ctx->d_fxe, fxe, sizeof fxe));
    }
    Tables &tb = ctx->tb;
    tb.dfa = ht.fast ? ctx->d_dfa.as<uint16_t>() : nullptr;
    tb.codes = ht.fast ? ctx->d_codes.as<uint8_t>() : nullptr;
    tb.n_states = ht.fast ? ht.n_states : 0;
    tb.fast = ht.fast ? 1 : 0;
    tb.dfa2 = ht.t2_ok ? ctx->d_dfa2.as<uint16_t>() : nullptr;
    tb.t2 = ht.t2_ok ? ctx->d_t2.as<uint32_t>() : nullptr;
    tb.n_windows = ht.t2_ok ? ht.n_windows : 0;
    tb.children = ctx->d_children.as<int32_t>();
    tb.term_code = ctx->d_term.as<int16_t>();
    tb.n_nodes = n_nodes;
    tb.max_len = ht.max_len;
    tb.exp_len = ctx->d_explen.as<uint8_t>();
    tb.exp_off = ctx->d_expoff.as<uint16_t>();
    tb.exp_flat = ctx->d_expflat.as<uint8_t>();
    tb.n_flat = (int)exp_off[256];
    tb.max_exp = 0;
    for (int b = 0; b < 256; ++b) tb.max_exp = std::max<int>(tb.max_exp, ht.exp_len[b]);
    ctx->fx_ok = tb.max_exp <= 15;
    ctx->fast_w = 0;
    if (ht.fast) {
        const int L = std::max(1, ht.max_len);
        ctx->fast_w = L <= 2 ? 2 : L <= 4 ? 4 : L <= 6 ? 6 : 8;
    }
    ctx->have_dict = true;
    return ZS_OK;
}

int zs_dictionary_fast(zs_ctx *ctx) { return ctx && ctx->have_dict ? ctx->fast_w : -1; }

int zs_build_t2_host(const int32_t *children, const int16_t *term_code, int32_t n_nodes,
                     uint16_t *dfa2, uint32_t *t2, int32_t *n_windows, int32_t *n_masks) {
    if (!children || !term_code || n_nodes < 1 || !dfa2 || !t2 || !n_windows || !n_masks)
        return ZS_E_ARG;
    std::vector<std::pair<std::string, int>> pats;
    trie_patterns(children, term_code, n_nodes, pats);
    HostTables ht;
    for (auto &p : pats) ht.max_len = std::max<int>(ht.max_len, (int)p.first.size());
    *n_windows = *n_masks = 0;
    if (!build_dfa(pats, ht.max_len, ht) || !build_t2(ht, std::max(1, ht.max_len))) return 0;
    *n_windows = ht.n_windows;
    *n_masks = ht.n_masks;
    memcpy(dfa2, ht.dfa2.data(), (size_t)ht.n_states * NCOL * 2);
    memcpy(t2, ht.t2.data(), ht.t2.size() * 4);
    return 1;
}

int zs_set_stream(zs_ctx *ctx, void *stream) {
    if (!ctx) return ZS_E_ARG;
    ctx->user_stream = static_cast<cudaStream_t>(stream);
    return ZS_OK;
}

int64_t zs_debug_chunk_cuts(const uint8_t *h_in, int64_t n, int64_t chunk, int64_t *cuts, int64_t cap) {
    if (n < 0 || (n > 0 && !h_in) || chunk <= 0 || (cap > 0 && !cuts)) return ZS_E_ARG;
    const std::vector<long long> c = chunk_cuts(h_in, n, chunk);
    for (size_t k = 0; k < c.size() && (int64_t)k < cap; ++k) cuts[k] = c[k];
    return (int64_t)c.size();
}

int zs_set_transducer(zs_ctx *ctx, int on) {
    if (!ctx) return ZS_E_ARG;
    // measurement / parity switches over the compress kernels (default 3):
    ctx->no_t2 = (on & 1) ? 0 : 1;   // bit 0 clear: generic key-window / trie-walk kernel (compress_tiles)
    ctx->no_ip = (on & 2) ? 0 : 1;   // bit 1 clear: likewise (kept for the old mode numbers)
    ctx->p4_lane = (on & 16) ? 1 : 0;  // bit 4: compress_cx parse over line-lane ranges, not byte slices
    ctx->no_pa = (on & 64) ? 1 : 0;    // bit 6: DFA + transducer parse instead of the product automaton
    ctx->slices = (on & 128) ? 1 : 0;  // bit 7: compress_cx on byte-exact slices in every phase
    ctx->no_ll = (on & 256) ? 1 : 0;   // bit 8: long lines on the general routine, not zs_ll.cuh
    return ZS_OK;
}

int zs_build_tables_host(const int32_t *children, const int16_t *term_code, int32_t n_nodes,
                         uint16_t *dfa, uint8_t *codes, int32_t *n_states, int32_t *max_len) {
    if (!children || !term_code || n_nodes < 1 || !dfa || !codes || !n_states || !max_len)
        return ZS_E_ARG;
    std::vector<std::pair<std::string, int>> pats;
    trie_patterns(children, term_code, n_nodes, pats);
    HostTables ht;
    ht.max_len = 0;
    for (auto &p : pats) ht.max_len = std::max<int>(ht.max_len, (int)p.first.size());
    *max_len = ht.max_len;
    *n_states = 0;
    if (!build_dfa(pats, ht.max_len, ht)) return 0;
    *n_states = ht.n_states;
    memcpy(dfa, ht.dfa.data(), (size_t)ht.n_states * NCOL * 2);
    memcpy(codes, ht.codes.data(), (size_t)ht.n_states * FAST_W);
    return 1;
}

int zs_index_build(zs_ctx *ctx, const uint8_t *d_comp, int64_t n, uint64_t *d_offsets, int64_t cap,
                   int64_t *n_records) {
    if (!ctx || n < 0 || (n > 0 && !d_comp) || !d_offsets || !n_records) return ZS_E_ARG;
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t st = ctx->stream[0];
    if (int rc = after_user_stream(ctx)) return rc;
    *n_records = 0;
    if (n == 0) {
        if (cap < 1) return ZS_E_CAPACITY;
        CK(cudaMemsetAsync(d_offsets, 0, 8, st));
        CK(cudaStreamSynchronize(st));
        return ZS_OK;
    }
    const long long nt = (n + IX_TILE - 1) / IX_TILE;
    if (ctx->ixs.reserve((size_t)nt * 12 + 64)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(index)");
    unsigned *tcount = ctx->ixs.as<unsigned>();
    unsigned long long *tbase = reinterpret_cast<unsigned long long *>(ctx->ixs.as<uint8_t>() + ((nt * 4 + 15) & ~15ll));
    unsigned long long *tot = tbase + nt;
    const int grid = (int)std::min<long long>(nt, (long long)ctx->n_sm * 8);
    ix_count<<<grid, IX_NT, 0, st>>>(d_comp, n, nt, tcount);
    ix_scan<unsigned><<<1, 1024, 0, st>>>(tcount, nt, tbase, tot);
    CK(cudaGetLastError());
    unsigned long long h_nl = 0;
    uint8_t last = 0;
    CK(cudaMemcpyAsync(&h_nl, tot, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&last, d_comp + n - 1, 1, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const long long recs = (long long)h_nl + (last != '\n' ? 1 : 0);
    *n_records = recs;
    if (cap < recs + 1) return ZS_E_CAPACITY;
    ix_write<<<grid, IX_NT, 0, st>>>(d_comp, n, nt, tbase, reinterpret_cast<unsigned long long *>(d_offsets));
    CK(cudaGetLastError());
    if (last != '\n') {
        const unsigned long long end = (unsigned long long)n + 1;
        CK(cudaMemcpyAsync(d_offsets + recs, &end, 8, cudaMemcpyHostToDevice, st));
    }
    CK(cudaStreamSynchronize(st));
    return ZS_OK;
}

int zs_decode_records(zs_ctx *ctx, const uint8_t *d_comp, const uint64_t *d_offsets, int64_t n_records,
                      const int64_t *d_idx, int64_t k, uint8_t *d_out, int64_t out_cap, int64_t *d_out_off,
                      int8_t *d_status, int64_t *d_errpos, int64_t *total_out) {
    if (!ctx || !d_comp || !d_offsets || n_records < 0 || k < 0 || (k > 0 && (!d_idx || !d_out_off || !d_status ||
        !d_errpos)) || !total_out)
        return ZS_E_ARG;
    if (!ctx->have_dict) return ZS_E_NODICT;
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t st = ctx->stream[0];
    if (int rc = after_user_stream(ctx)) return rc;
    *total_out = 0;
    if (k == 0) return ZS_OK;
    if (ctx->ixs.reserve((size_t)k * 8 + 64)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(index)");
    long long *len = ctx->ixs.as<long long>();
    const int grid = (int)std::min<long long>((k + 255) / 256, (long long)ctx->n_sm * 8);
    ix_sizes<<<grid, 256, 0, st>>>(d_comp, reinterpret_cast<const unsigned long long *>(d_offsets), n_records,
                                   reinterpret_cast<const long long *>(d_idx), k, ctx->tb.exp_len, len, d_status,
                                   reinterpret_cast<long long *>(d_errpos));
    unsigned long long *off = reinterpret_cast<unsigned long long *>(d_out_off);
    ix_scan<long long><<<1, 1024, 0, st>>>(len, k, off, off + k);
    CK(cudaGetLastError());
    unsigned long long h_tot = 0;
    CK(cudaMemcpyAsync(&h_tot, off + k, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *total_out = (int64_t)h_tot;
    if ((long long)h_tot > out_cap) return ZS_E_CAPACITY;
    if (h_tot)
        ix_fill<<<grid, 256, 0, st>>>(d_comp, reinterpret_cast<const unsigned long long *>(d_offsets),
                                      reinterpret_cast<const long long *>(d_idx), k, d_status, off, ctx->tb.exp_len,
                                      ctx->tb.exp_off, ctx->tb.exp_flat, d_out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return ZS_OK;
}

int zs_host_alloc(zs_ctx *ctx, int64_t bytes, void **p) {
    if (!ctx || bytes < 0 || !p) return ZS_E_ARG;
    *p = nullptr;
    CK(cudaSetDevice(ctx->dev));
    CK(cudaHostAlloc(p, (size_t)std::max<int64_t>(bytes, 1), cudaHostAllocDefault));
    return ZS_OK;
}

int zs_host_free(zs_ctx *ctx, void *p) {
    if (!ctx) return ZS_E_ARG;
    if (p) CK(cudaFreeHost(p));
    return ZS_OK;
}

int64_t zs_compress_bound(int64_t n) { return 2 * n + 64; }

int64_t zs_decompress_bound(zs_ctx *ctx, int64_t n) {
    int m = 1;
    if (ctx && ctx->have_dict)
        for (int b = 0; b < 256; ++b) m = std::max<int>(m, ctx->ht.exp_len[b]);
    return (int64_t)m * n + 64;
}

int zs_compress_device(zs_ctx *ctx, const uint8_t *d_in, int64_t n, uint8_t *d_out,
                       int64_t out_cap, int flags, zs_result *res) {
    return run_device(ctx, true, d_in, n, d_out, out_cap, flags, res);
}

int zs_decompress_device(zs_ctx *ctx, const uint8_t *d_in, int64_t n, uint8_t *d_out,
                         int64_t out_cap, int flags, zs_result *res) {
    return run_device(ctx, false, d_in, n, d_out, out_cap, flags, res);
}

int zs_compress_host(zs_ctx *ctx, const uint8_t *h_in, int64_t n, uint8_t *h_out,
                     int64_t out_cap, int flags, zs_result *res) {
    return run_host(ctx, true, h_in, n, h_out, out_cap, flags, res);
}

int zs_decompress_host(zs_ctx *ctx, const uint8_t *h_in, int64_t n, uint8_t *h_out,
                       int64_t out_cap, int flags, zs_result *res) {
    return run_host(ctx, false, h_in, n, h_out, out_cap, flags, res);
}

// ---------------------------------------------------------------------------
// parity shim
// ---------------------------------------------------------------------------
static int upload_batch(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts, int64_t n_lines) {
    const long long n = starts[n_lines];
    if (ctx->s_flat.reserve(n + 16) || ctx->s_starts.reserve(8 * (n_lines + 1)))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(batch)");
    cudaStream_t st = ctx->stream[0];
    if (n) CK(cudaMemcpyAsync(ctx->s_flat.p, flat, n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->s_starts.p, starts, 8 * (n_lines + 1), cudaMemcpyHostToDevice, st));
    return ZS_OK;
}

int zs_compress_batch(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts, int64_t n_lines,
                      uint8_t *out, int64_t *out_lens, int64_t *escapes) {
    if (!ctx || !starts || n_lines < 0 || !out_lens) return ZS_E_ARG;
    if (!ctx->have_dict) return ZS_E_NODICT;
    if (escapes) *escapes = 0;
    if (n_lines == 0) return ZS_OK;
    CK(cudaSetDevice(ctx->dev));
    int rc = upload_batch(ctx, flat, starts, n_lines);
    if (rc) return rc;
    const long long n = starts[n_lines];
    cudaStream_t st = ctx->stream[0];
    if (ctx->s_out.reserve(2 * n + 16) || ctx->s_lens.reserve(8 * n_lines) ||
        ctx->s_dec.reserve(n + n_lines + 16) || ctx->s_tot.reserve(16))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(batch)");
    CK(cudaMemsetAsync(ctx->s_tot.p, 0, 16, st));
    BatchKernel k = batch_kernel(ctx->fast_w);
    const int smem = ctx->fast_w ? align16(ctx->tb.n_states * NCOL * 2) + align16(ctx->tb.n_states * FAST_W) : 0;
    CK(set_smem(k, smem));
    const int blocks = (int)((n_lines + 255) / 256);
    k<<<blocks, 256, smem, st>>>(ctx->s_flat.as<uint8_t>(), ctx->s_starts.as<long long>(), n_lines,
                                 ctx->s_out.as<uint8_t>(), ctx->s_lens.as<long long>(),
                                 ctx->s_dec.as<uint8_t>(), ctx->s_tot.as<unsigned long long>(), ctx->tb);
    CK(cudaGetLastError());
    if (n && out) CK(cudaMemcpyAsync(out, ctx->s_out.p, 2 * n, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_lens, ctx->s_lens.p, 8 * n_lines, cudaMemcpyDeviceToHost, st));
    unsigned long long esc = 0;
    CK(cudaMemcpyAsync(&esc, ctx->s_tot.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (escapes) *escapes = (int64_t)esc;
    return ZS_OK;
}

int zs_decompress_sizes(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts,
                        int64_t n_lines, int64_t *out_lens, int8_t *status, int64_t *errpos,
                        int64_t *total, int64_t *escapes) {
    if (!ctx || !starts || n_lines < 0 || !out_lens || !status || !errpos) return ZS_E_ARG;
    if (!ctx->have_dict) return ZS_E_NODICT;
    if (total) *total = 0;
    if (escapes) *escapes = 0;
    if (n_lines == 0) return ZS_OK;
    CK(cudaSetDevice(ctx->dev));
    int rc = upload_batch(ctx, flat, starts, n_lines);
    if (rc) return rc;
    cudaStream_t st = ctx->stream[0];
    if (ctx->s_lens.reserve(8 * n_lines) || ctx->s_stat.reserve(n_lines) ||
        ctx->s_errpos.reserve(8 * n_lines) || ctx->s_tot.reserve(16))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(batch)");
    CK(cudaMemsetAsync(ctx->s_tot.p, 0, 16, st));
    batch_decode_sizes<<<(int)((n_lines + 255) / 256), 256, 0, st>>>(
        ctx->s_flat.as<uint8_t>(), ctx->s_starts.as<long long>(), n_lines, ctx->s_lens.as<long long>(),
        ctx->s_stat.as<int8_t>(), ctx->s_errpos.as<long long>(), ctx->s_tot.as<unsigned long long>(),
        ctx->tb);
    CK(cudaGetLastError());
    unsigned long long tot[2];
    CK(cudaMemcpyAsync(out_lens, ctx->s_lens.p, 8 * n_lines, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(status, ctx->s_stat.p, n_lines, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(errpos, ctx->s_errpos.p, 8 * n_lines, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(tot, ctx->s_tot.p, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (total) *total = (int64_t)tot[0];
    if (escapes) *escapes = (int64_t)tot[1];
    return ZS_OK;
}

int zs_decompress_fill(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts, int64_t n_lines,
                       const int8_t *status, uint8_t *out, const int64_t *out_starts) {
    if (!ctx || !starts || n_lines < 0 || !status || !out_starts) return ZS_E_ARG;
    if (!ctx->have_dict) return ZS_E_NODICT;
    if (n_lines == 0) return ZS_OK;
    CK(cudaSetDevice(ctx->dev));
    int rc = upload_batch(ctx, flat, starts, n_lines);
    if (rc) return rc;
    cudaStream_t st = ctx->stream[0];
    const long long total = out_starts[n_lines];
    if (ctx->s_stat.reserve(n_lines) || ctx->s_outst.reserve(8 * (n_lines + 1)) ||
        ctx->s_out.reserve(total + 16))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(batch)");
    CK(cudaMemcpyAsync(ctx->s_stat.p, status, n_lines, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ctx->s_outst.p, out_starts, 8 * (n_lines + 1), cudaMemcpyHostToDevice, st));
    batch_decode_fill<<<(int)((n_lines + 255) / 256), 256, 0, st>>>(
        ctx->s_flat.as<uint8_t>(), ctx->s_starts.as<long long>(), n_lines, ctx->s_stat.as<int8_t>(),
        ctx->s_out.as<uint8_t>(), ctx->s_outst.as<long long>(), ctx->tb);
    CK(cudaGetLastError());
    if (total && out) CK(cudaMemcpyAsync(out, ctx->s_out.p, total, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return ZS_OK;
}

int zs_preprocess_batch(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts,
                        int64_t n_lines, uint8_t *out, int64_t *out_lens, int8_t *status,
                        int64_t *err_off, uint64_t *err_ids) {
    if (!ctx || !starts || n_lines < 0 || !out || !out_lens || !status || !err_off || !err_ids)
        return ZS_E_ARG;
    if (n_lines == 0) return ZS_OK;
    CK(cudaSetDevice(ctx->dev));
    int rc = upload_batch(ctx, flat, starts, n_lines);
    if (rc) return rc;
    cudaStream_t st = ctx->stream[0];
    const long long n = starts[n_lines];
    const long long ocap = 3 * n + 3 * n_lines;
    if (ctx->s_out.reserve(ocap + 16) || ctx->s_lens.reserve(8 * n_lines) ||
        ctx->s_stat.reserve(n_lines) || ctx->s_errpos.reserve(8 * n_lines) ||
        ctx->s_ids.reserve(16 * n_lines) || ctx->s_dec.reserve(n + n_lines + 16))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(batch)");
    batch_preprocess<<<(int)((n_lines + 255) / 256), 256, 0, st>>>(
        ctx->s_flat.as<uint8_t>(), ctx->s_starts.as<long long>(), n_lines, ctx->s_out.as<uint8_t>(),
        ctx->s_lens.as<long long>(), ctx->s_stat.as<int8_t>(), ctx->s_errpos.as<long long>(),
        ctx->s_ids.as<unsigned long long>(), ctx->s_dec.as<uint8_t>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, ctx->s_out.p, ocap, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_lens, ctx->s_lens.p, 8 * n_lines, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(status, ctx->s_stat.p, n_lines, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(err_off, ctx->s_errpos.p, 8 * n_lines, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(err_ids, ctx->s_ids.p, 16 * n_lines, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return ZS_OK;
}


// ---------------------------------------------------------------------------
// dictionary training (zs_train.cuh; dictionary.py:169-320)
// ---------------------------------------------------------------------------

int zs_train_count(zs_ctx *ctx, const uint8_t *h_buf, int64_t n, int32_t l_min, int32_t l_max, int64_t *n_rows) {
    if (!ctx || n < 0 || (n > 0 && !h_buf) || !n_rows || l_min < 2 || l_min > l_max || l_max > 64 ||
        n >= (int64_t)0xffffff00ll)
        return ZS_E_ARG;
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t st = ctx->stream[0];
    auto &T = ctx->tr;
    *n_rows = 0;
    T.rows = 0;
    T.n = n;
    T.lmax = l_max;
    if (n == 0) return ZS_OK;
    auto grid = [&](long long m) { return (int)std::max(1ll, std::min<long long>((m + 255) / 256, (long long)ctx->n_sm * 16)); };
    if (T.buf.reserve((size_t)n + 16) || T.run.reserve((size_t)n) || T.pos[0].reserve((size_t)n * 4) ||
        T.pos[1].reserve((size_t)n * 4) || T.nsel.reserve(64))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(train)");
    CK(cudaMemcpyAsync(T.buf.p, h_buf, (size_t)n, cudaMemcpyHostToDevice, st));
    tr_runs<<<grid((n + TR_SPAN - 1) / TR_SPAN), TR_NT, 0, st>>>(T.buf.as<uint8_t>(), n, l_max, T.run.as<uint8_t>());
    CK(cudaGetLastError());
    // candidate starts: alphabet run >= l_min
    size_t tb = 0;
    thrust::counting_iterator<uint32_t> it(0);
    const TrAtLeast sel_op{T.run.as<uint8_t>(), l_min};
    CK(cub::DeviceSelect::If(nullptr, tb, it, T.pos[0].as<uint32_t>(), T.nsel.as<long long>(), n, sel_op, st));
    if (T.cub.reserve(tb)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(cub)");
    CK(cub::DeviceSelect::If(T.cub.p, tb, it, T.pos[0].as<uint32_t>(), T.nsel.as<long long>(), n, sel_op, st));
    long long m = 0;
    CK(cudaMemcpyAsync(&m, T.nsel.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (m == 0) return ZS_OK;
    if (T.key[0].reserve((size_t)m * 8) || T.key[1].reserve((size_t)m * 8) || T.lcp.reserve((size_t)m) ||
        T.runs.reserve((size_t)m) || T.v.reserve((size_t)m * 8) || T.ex.reserve((size_t)m * 8) ||
        T.bstart.reserve((size_t)m * 4 + 8) || T.cand.reserve((size_t)m * 4))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(train)");
    // LSD sort of the starts by their first l_max bytes
    cub::DoubleBuffer<unsigned long long> keys(T.key[0].as<unsigned long long>(), T.key[1].as<unsigned long long>());
    cub::DoubleBuffer<uint32_t> vals(T.pos[0].as<uint32_t>(), T.pos[1].as<uint32_t>());
    const int W = (l_max + 7) / 8;
    for (int w = W - 1; w >= 0; --w) {
        const int nb = std::min(8, l_max - 8 * w);
        tr_key<<<grid(m), 256, 0, st>>>(T.buf.as<uint8_t>(), n, vals.Current(), m, w, nb, keys.Current());
        CK(cudaGetLastError());
        tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, vals, (int)m, 64 - 8 * nb, 64, st));
        if (T.cub.reserve(tb)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(cub)");
        CK(cub::DeviceRadixSort::SortPairs(T.cub.p, tb, keys, vals, (int)m, 64 - 8 * nb, 64, st));
    }
    const uint32_t *pos = vals.Current();
    tr_lcp<<<grid(m), 256, 0, st>>>(T.buf.as<uint8_t>(), pos, m, T.run.as<uint8_t>(), T.lcp.as<uint8_t>(),
                                    T.runs.as<uint8_t>());
    CK(cudaGetLastError());
    tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, T.v.as<unsigned long long>(), T.ex.as<unsigned long long>(), (int)m, st));
    if (T.cub.reserve(tb)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(cub)");
    long long rows = 0;
    for (int L = l_min; L <= l_max; ++L) {
        if (n < L) break;  // dictionary.py:187-188
        tr_flags<<<grid(m), 256, 0, st>>>(T.lcp.as<uint8_t>(), T.runs.as<uint8_t>(), m, L, T.v.as<unsigned long long>());
        CK(cub::DeviceScan::ExclusiveSum(T.cub.p, tb, T.v.as<unsigned long long>(), T.ex.as<unsigned long long>(),
                                         (int)m, st));
        unsigned long long tail[2];
        CK(cudaMemcpyAsync(&tail[0], T.v.as<unsigned long long>() + m - 1, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&tail[1], T.ex.as<unsigned long long>() + m - 1, 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const long long c = (long long)((tail[0] & 0xffffffffull) + (tail[1] & 0xffffffffull));
        if (c == 0) continue;
        tr_scatter<<<grid(m), 256, 0, st>>>(T.v.as<unsigned long long>(), T.ex.as<unsigned long long>(), m,
                                            T.bstart.as<uint32_t>(), T.cand.as<uint32_t>());
        if (T.rpos.grow_keep((size_t)(rows + c) * 4, (size_t)rows * 4, st) ||
            T.rocc.grow_keep((size_t)(rows + c) * 4, (size_t)rows * 4, st) ||
            T.rlen.grow_keep((size_t)(rows + c), (size_t)rows, st))
            return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(rank table)");
        tr_rows<<<grid(c), 256, 0, st>>>(T.cand.as<uint32_t>(), c, pos, T.ex.as<unsigned long long>(),
                                         T.bstart.as<uint32_t>(), L, T.rpos.as<uint32_t>() + rows,
                                         T.rocc.as<uint32_t>() + rows, T.rlen.as<uint8_t>() + rows);
        CK(cudaGetLastError());
        rows += c;
    }
    CK(cudaStreamSynchronize(st));
    if (rows >= (long long)0xffffffffll) return fail(ctx, cudaErrorInvalidValue, "rank table over 2^32 rows");
    T.rows = rows;
    *n_rows = rows;
    return ZS_OK;
}

int zs_train_rows(zs_ctx *ctx, int64_t *pos, int32_t *len, int64_t *occ) {
    if (!ctx || (ctx->tr.rows && (!pos || !len || !occ))) return ZS_E_ARG;
    CK(cudaSetDevice(ctx->dev));
    const long long m = ctx->tr.rows;
    if (!m) return ZS_OK;
    std::vector<uint32_t> p((size_t)m), o((size_t)m);
    std::vector<uint8_t> l((size_t)m);
    cudaStream_t st = ctx->stream[0];
    CK(cudaMemcpyAsync(p.data(), ctx->tr.rpos.p, (size_t)m * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(o.data(), ctx->tr.rocc.p, (size_t)m * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(l.data(), ctx->tr.rlen.p, (size_t)m, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (long long i = 0; i < m; ++i) {
        pos[i] = p[i];
        len[i] = l[i];
        occ[i] = o[i];
    }
    return ZS_OK;
}

int zs_train_load(zs_ctx *ctx, const uint8_t *patterns, int32_t width, const int64_t *lengths, const int64_t *occ,
                  int64_t m) {
    if (!ctx || m < 0 || width < 1 || width > 64 || (m > 0 && (!patterns || !lengths || !occ)) ||
        m * (int64_t)width >= (int64_t)0xffffff00ll)
        return ZS_E_ARG;
    CK(cudaSetDevice(ctx->dev));
    auto &T = ctx->tr;
    T.rows = 0;
    T.n = m * width;
    T.lmax = width;
    if (!m) return ZS_OK;
    std::vector<uint32_t> p((size_t)m), o((size_t)m);
    std::vector<uint8_t> l((size_t)m);
    for (long long i = 0; i < m; ++i) {
        if (lengths[i] < 1 || lengths[i] > width || occ[i] < 0 || occ[i] > 0xffffffffll) return ZS_E_ARG;
        p[i] = (uint32_t)(i * width);
        l[i] = (uint8_t)lengths[i];
        o[i] = (uint32_t)occ[i];
    }
    cudaStream_t st = ctx->stream[0];
    if (T.buf.reserve((size_t)(m * width) + 16) || T.rpos.reserve((size_t)m * 4) || T.rocc.reserve((size_t)m * 4) ||
        T.rlen.reserve((size_t)m))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(train)");
    CK(cudaMemcpyAsync(T.buf.p, patterns, (size_t)(m * width), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(T.rpos.p, p.data(), (size_t)m * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(T.rocc.p, o.data(), (size_t)m * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(T.rlen.p, l.data(), (size_t)m, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    T.rows = m;
    return ZS_OK;
}

int zs_train_select(zs_ctx *ctx, int32_t t, int64_t cap, int64_t *rows_out, int32_t *n_selected) {
    if (!ctx || t < 0 || t > 128 || cap < 1 || !n_selected || (t > 0 && !rows_out)) return ZS_E_ARG;
    CK(cudaSetDevice(ctx->dev));
    auto &T = ctx->tr;
    cudaStream_t st = ctx->stream[0];
    *n_selected = 0;
    const long long M = T.rows;
    if (t == 0 || M == 0) return ZS_OK;
    auto grid = [&](long long m) { return (int)std::max(1ll, std::min<long long>((m + 255) / 256, (long long)ctx->n_sm * 16)); };
    const long long nodes = 1 + (long long)t * T.lmax;
    if (T.rank[0].reserve((size_t)M * 8) || T.rank[1].reserve((size_t)M * 8) || T.idx[0].reserve((size_t)M * 4) ||
        T.idx[1].reserve((size_t)M * 4) || T.dead.reserve((size_t)M) ||
        T.child.reserve((size_t)nodes * TR_TRIE_W * 2) || T.term.reserve((size_t)nodes) ||
        T.ctl.reserve(sizeof(TrCtl)) || T.sel.reserve(128 * 4))
        return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(select)");
    const TrRows R{T.buf.as<uint8_t>(), T.rpos.as<uint32_t>(), T.rlen.as<uint8_t>()};
    for (;;) {  // select_patterns (dictionary.py:300-307)
        tr_init_rank<<<grid(M), 256, 0, st>>>(T.rocc.as<uint32_t>(), T.rlen.as<uint8_t>(), M,
                                              T.rank[0].as<unsigned long long>(), T.idx[0].as<uint32_t>());
        CK(cudaGetLastError());
        const uint32_t *ws = T.idx[0].as<uint32_t>();
        long long nws = M, excluded_max = -1;
        if (cap < M) {  // working set: top-cap by initial rank, stable (dictionary.py:256-264)
            size_t tb = 0;
            CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, T.rank[0].as<unsigned long long>(),
                                                         T.rank[1].as<unsigned long long>(), T.idx[0].as<uint32_t>(),
                                                         T.idx[1].as<uint32_t>(), (int)M, 0, 64, st));
            if (T.cub.reserve(tb)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(cub)");
            CK(cub::DeviceRadixSort::SortPairsDescending(T.cub.p, tb, T.rank[0].as<unsigned long long>(),
                                                         T.rank[1].as<unsigned long long>(), T.idx[0].as<uint32_t>(),
                                                         T.idx[1].as<uint32_t>(), (int)M, 0, 64, st));
            unsigned long long ex = 0;
            CK(cudaMemcpyAsync(&ex, T.rank[1].as<unsigned long long>() + cap, 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            ws = T.idx[1].as<uint32_t>();
            nws = cap;
            excluded_max = (long long)ex;
        }
        const int nblk = grid(nws);
        if (T.blk.reserve((size_t)nblk * sizeof(TrBest))) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(select)");
        const TrCtl c0{0, 0, 0, 1};
        CK(cudaMemsetAsync(T.dead.p, 0, (size_t)nws, st));
        CK(cudaMemsetAsync(T.child.p, 0xff, (size_t)nodes * TR_TRIE_W * 2, st));
        CK(cudaMemsetAsync(T.term.p, 0, (size_t)nodes, st));
        CK(cudaMemcpyAsync(T.ctl.p, &c0, sizeof c0, cudaMemcpyHostToDevice, st));
        for (int k = 0; k < t; ++k) {  // _try_select (dictionary.py:266-297), no host round trip
            tr_rank<<<nblk, TR_NT, 0, st>>>(R, T.rocc.as<uint32_t>(), ws, nws, T.dead.as<uint8_t>(),
                                            T.child.as<int16_t>(), T.term.as<uint8_t>(), T.ctl.as<TrCtl>(),
                                            T.blk.as<TrBest>());
            tr_pick<<<1, 1024, 0, st>>>(R, T.dead.as<uint8_t>(), T.child.as<int16_t>(), T.term.as<uint8_t>(),
                                        T.ctl.as<TrCtl>(), T.blk.as<TrBest>(), nblk, excluded_max, T.sel.as<uint32_t>());
        }
        CK(cudaGetLastError());
        TrCtl c1;
        uint32_t sel[128];
        CK(cudaMemcpyAsync(&c1, T.ctl.p, sizeof c1, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(sel, T.sel.p, 128 * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (c1.fail) {
            cap *= 4;
            continue;
        }
        for (int k = 0; k < c1.nsel; ++k) rows_out[k] = sel[k];
        *n_selected = c1.nsel;
        return ZS_OK;
    }
}

int zs_overlap_batch(zs_ctx *ctx, const int32_t *children, const int16_t *term_len, int32_t n_nodes,
                     const uint8_t *pats, int32_t width, const int64_t *lens, int64_t n, int64_t *out) {
    if (!ctx || n < 0 || n_nodes < 1 || width < 0 || !children || !term_len ||
        (n > 0 && (!lens || !out || (width > 0 && !pats))))
        return ZS_E_ARG;
    for (int64_t r = 0; r < n; ++r)
        if (lens[r] < 0 || lens[r] > width) return ZS_E_ARG;
    if (n == 0) return ZS_OK;
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t st = ctx->stream[0];
    auto &T = ctx->tr;
    const size_t cb = (size_t)n_nodes * 256 * 4, tb = (size_t)n_nodes * 2, pb = (size_t)n * width;
    // scratch: children | term_len | pats | lens | out
    DevBuf &S = T.cub;
    if (S.reserve(cb + tb + pb + (size_t)n * 16 + 64)) return fail(ctx, cudaErrorMemoryAllocation, "cudaMalloc(overlap)");
    uint8_t *b = S.as<uint8_t>();
    int32_t *d_ch = reinterpret_cast<int32_t *>(b);
    int16_t *d_tl = reinterpret_cast<int16_t *>(b + cb);
    uint8_t *d_p = b + cb + tb;
    long long *d_l = reinterpret_cast<long long *>(b + ((cb + tb + pb + 15) & ~(size_t)15));
    long long *d_o = d_l + n;
    CK(cudaMemcpyAsync(d_ch, children, cb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_tl, term_len, tb, cudaMemcpyHostToDevice, st));
    if (pb) CK(cudaMemcpyAsync(d_p, pats, pb, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_l, lens, (size_t)n * 8, cudaMemcpyHostToDevice, st));
    tr_overlap_batch<<<(int)std::min<long long>((n + 255) / 256, (long long)ctx->n_sm * 16), 256, 0, st>>>(
        d_ch, d_tl, d_p, width, d_l, n, d_o);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, d_o, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return ZS_OK;
}

}  // extern "C"
