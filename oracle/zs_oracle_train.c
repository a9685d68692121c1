/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY (see zs_oracle.c).
 *
 * Plain-C restatement of the reference dictionary trainer, the CPU checker
 * for the GPU trainer (paper_2404_19391_b200/csrc/zs_train.cuh).  Pinned
 * against the reference's own outputs in tests/golden/train_cases.json.gz
 * and the .zsd files under tests/golden/dicts (tests/test_oracle_train.py).
 *
 *   zo_count_substrings  dictionary.py:169-221  per-length window census:
 *                        windows wholly inside the alphabet (smiles.py
 *                        ALPHABET), lines joined on '\n' so no window
 *                        crosses a line; rows length-major, bytewise
 *                        ascending within a length (np.unique order)
 *   zo_overlap           numba_impl.py:142-169  greedy longest-match cover
 *   zo_select_patterns   dictionary.py:241-307  _try_select / select_patterns
 *                        with the working-set cap and its retry, permanent
 *                        removal of rank <= 0 candidates, the _pick tie rule
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "zs_oracle.h"

static const char ALPHA[] =
    "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789[]()=#-+@/\\%.:*$~";

static void alpha_mask(uint8_t m[256]) {
    memset(m, 0, 256);
    for (const char *c = ALPHA; *c; ++c) m[(uint8_t)*c] = 1;
}

/* ---- count_substrings ---- */
static const uint8_t *g_buf;
static int g_len;

static int cmp_window(const void *a, const void *b) {
    const int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    const int c = memcmp(g_buf + x, g_buf + y, (size_t)g_len);
    return c ? c : (x < y ? -1 : x > y);
}

typedef struct {
    uint64_t key;
    int64_t pos;
} kp_t;

static int cmp_kp(const void *a, const void *b) {
    const kp_t *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->pos < y->pos ? -1 : x->pos > y->pos;
}

int64_t zo_count_substrings(const uint8_t *buf, int64_t n, int lmin, int lmax, int64_t **pos_out,
                            int32_t **len_out, int64_t **occ_out) {
    uint8_t am[256];
    alpha_mask(am);
    /* run[i] = alphabet bytes starting at i (the nonmember cumsum test, :183-190) */
    int32_t *run = malloc(sizeof(int32_t) * (size_t)(n + 1));
    run[n] = 0;
    for (int64_t i = n - 1; i >= 0; --i) run[i] = am[buf[i]] ? run[i + 1] + 1 : 0;
    int64_t cap = 1024, m = 0;
    int64_t *P = malloc(sizeof(int64_t) * cap), *O = malloc(sizeof(int64_t) * cap);
    int32_t *Ln = malloc(sizeof(int32_t) * cap);
    int64_t *win = malloc(sizeof(int64_t) * (size_t)(n + 1));
    kp_t *kp = malloc(sizeof(kp_t) * (size_t)(n + 1));
    for (int L = lmin; L <= lmax; ++L) {
        if (n < L) break; /* :187-188 */
        int64_t nw = 0;
        for (int64_t i = 0; i + L <= n; ++i)
            if (run[i] >= L) win[nw++] = i;
        if (!nw) continue;
        if (L <= 8) { /* big-endian u64 keys + np.unique (:193-201) */
            for (int64_t k = 0; k < nw; ++k) {
                uint64_t key = 0;
                for (int j = 0; j < L; ++j) key = (key << 8) | buf[win[k] + j];
                kp[k].key = key;
                kp[k].pos = win[k];
            }
            qsort(kp, (size_t)nw, sizeof(kp_t), cmp_kp);
            for (int64_t k = 0; k < nw; ++k) win[k] = kp[k].pos;
        } else { /* void-row np.unique: bytewise order (:202-208) */
            g_buf = buf;
            g_len = L;
            qsort(win, (size_t)nw, sizeof(int64_t), cmp_window);
        }
        for (int64_t a = 0; a < nw;) {
            int64_t b = a + 1;
            while (b < nw && memcmp(buf + win[a], buf + win[b], (size_t)L) == 0) ++b;
            if (m == cap) {
                cap *= 2;
                P = realloc(P, sizeof(int64_t) * cap);
                O = realloc(O, sizeof(int64_t) * cap);
                Ln = realloc(Ln, sizeof(int32_t) * cap);
            }
            P[m] = win[a];
            Ln[m] = L;
            O[m] = b - a;
            ++m;
            a = b;
        }
    }
    free(run);
    free(win);
    free(kp);
    *pos_out = P;
    *len_out = Ln;
    *occ_out = O;
    return m;
}

/* ---- overlap_batch ---- */
typedef struct {
    int32_t *child; /* [nodes][256] */
    uint8_t *term;
    int nodes, cap;
} trie_t;

static void trie_init(trie_t *t, int cap) {
    t->cap = cap;
    t->child = malloc(sizeof(int32_t) * 256 * (size_t)cap);
    t->term = calloc((size_t)cap, 1);
    memset(t->child, 0xff, sizeof(int32_t) * 256);
    t->nodes = 1;
}

static void trie_insert(trie_t *t, const uint8_t *p, int n) { /* trie.py:22-50 */
    int node = 0;
    for (int j = 0; j < n; ++j) {
        int nx = t->child[node * 256 + p[j]];
        if (nx < 0) {
            nx = t->nodes++;
            memset(t->child + (size_t)nx * 256, 0xff, sizeof(int32_t) * 256);
            t->term[nx] = 0;
            t->child[node * 256 + p[j]] = nx;
        }
        node = nx;
    }
    t->term[node] = 1;
}

static int cover(const trie_t *t, const uint8_t *p, int n) { /* numba_impl.py:149-169 */
    int pos = 0, cov = 0;
    while (pos < n) {
        int node = 0, best = 0;
        for (int j = pos; j < n; ++j) {
            node = t->child[node * 256 + p[j]];
            if (node < 0) break;
            if (t->term[node]) best = j + 1 - pos;
        }
        if (best > 0) {
            cov += best;
            pos += best;
        } else {
            pos += 1;
        }
    }
    return cov;
}

int64_t zo_overlap(const uint8_t *p, int n, const uint8_t *sel, const int32_t *sel_len, int nsel) {
    if (!nsel || !n) return 0; /* dictionary.py:227-228 */
    int tot = 1;
    for (int k = 0; k < nsel; ++k) tot += sel_len[k];
    trie_t t;
    trie_init(&t, tot);
    for (int k = 0, off = 0; k < nsel; off += sel_len[k], ++k) trie_insert(&t, sel + off, sel_len[k]);
    const int64_t r = cover(&t, p, n);
    free(t.child);
    free(t.term);
    return r;
}

/* ---- select_patterns ---- */
static const int64_t *g_rank;

static int cmp_rank_desc(const void *a, const void *b) { /* argsort(-rank, kind="stable") */
    const int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    if (g_rank[x] != g_rank[y]) return g_rank[x] > g_rank[y] ? -1 : 1;
    return x < y ? -1 : x > y;
}

static int64_t try_select(const uint8_t *buf, const int64_t *pos, const int32_t *len, const int64_t *occ,
                          int64_t m, int t, int64_t cap, int64_t *out) {
    int64_t *init = malloc(sizeof(int64_t) * (size_t)(m + 1));
    for (int64_t i = 0; i < m; ++i) init[i] = occ[i] * len[i];
    int64_t *ws = malloc(sizeof(int64_t) * (size_t)(m + 1)), nws = m, excluded_max = -1;
    for (int64_t i = 0; i < m; ++i) ws[i] = i;
    if (cap < m) { /* dictionary.py:256-264 */
        g_rank = init;
        qsort(ws, (size_t)m, sizeof(int64_t), cmp_rank_desc);
        excluded_max = init[ws[cap]];
        nws = cap;
    }
    uint8_t *alive = malloc((size_t)nws + 1);
    memset(alive, 1, (size_t)nws);
    int maxl = 1;
    for (int64_t k = 0; k < nws; ++k) maxl = len[ws[k]] > maxl ? len[ws[k]] : maxl;
    trie_t tr;
    trie_init(&tr, 1 + t * maxl);
    int nsel = 0, fail = 0;
    while (nsel < t) {
        int64_t best = -1, rmax = 0;
        for (int64_t k = 0; k < nws; ++k) {
            if (!alive[k]) continue;
            const int64_t i = ws[k];
            const int64_t r = occ[i] * (len[i] - (nsel ? cover(&tr, buf + pos[i], len[i]) : 0));
            if (r <= 0) { /* :279-284: dropped for good */
                alive[k] = 0;
                continue;
            }
            /* _pick (:229-238): highest rank, then longest, then bytewise smallest */
            int better = best < 0 || r > rmax;
            if (!better && r == rmax) {
                if (len[i] != len[best]) better = len[i] > len[best];
                else better = memcmp(buf + pos[i], buf + pos[best], (size_t)len[i]) < 0;
            }
            if (better) {
                best = i;
                rmax = r;
            }
        }
        if (best < 0) break;             /* :285-286 */
        if (rmax <= excluded_max) {      /* :288-289 */
            fail = 1;
            break;
        }
        out[nsel++] = best;
        trie_insert(&tr, buf + pos[best], len[best]);
        for (int64_t k = 0; k < nws; ++k)
            if (ws[k] == best) alive[k] = 0;
    }
    free(init);
    free(ws);
    free(alive);
    free(tr.child);
    free(tr.term);
    return fail ? -1 : nsel;
}

int64_t zo_select_patterns(const uint8_t *buf, const int64_t *pos, const int32_t *len, const int64_t *occ,
                           int64_t m, int t, int64_t cap, int64_t *out) {
    for (;;) { /* dictionary.py:300-307 */
        const int64_t r = try_select(buf, pos, len, occ, m, t, cap, out);
        if (r >= 0) return r;
        cap *= 4;
    }
}
