/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference ZSMILES per-line codec path, used as
 * the CPU checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg.  It is never linked into or called by
 * the product path (paper_2404_19391_b200/), which runs on sm_100a only.
 *
 * Parity pinned against outputs of the reference itself (the unmodified
 * Python/numba package run in the build container): see
 * tests/golden/make_golden.py and tests/test_oracle.py.
 *
 * Functions and the reference code they restate:
 *   zo_compress_batch    kernels/numba_impl.py:16-71   (min-cost DP + emit)
 *   zo_decompress_sizes  kernels/numba_impl.py:74-112  (size + validate)
 *   zo_decompress_fill   kernels/numba_impl.py:115-139 (table expansion)
 *   zo_preprocess_line   smiles.py:83-213 (tokenize, _ring_intervals,
 *                        _color_intervals, re-emit)
 *   zo_run_stream        pipeline.py:49-74,97-167 (newline framing, CR
 *                        policy, strict/lenient, stats) over a whole buffer,
 *                        sharded over pthreads (lines are independent,
 *                        SPEC.md:248), in-order concatenation.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "zs_oracle.h"

/* ------------------------------------------------------------------ */
/* compress: right-to-left DP over trie matches, forward emit          */
/* ------------------------------------------------------------------ */

/* One line.  cost/blen/code are caller scratch of >= n+1 entries.
 * Returns payload length; *esc += escapes emitted. */
static int64_t compress_one(const int32_t *children, const int16_t *term_code,
                            const uint8_t *s, int64_t n, uint8_t *out,
                            int64_t *cost, int32_t *blen, int16_t *code, int64_t *esc) {
    if (n == 0) return 0;
    cost[n] = 0;
    for (int64_t i = n - 1; i >= 0; i--) {
        int64_t best = cost[i + 1] + 2; /* escape edge: 0x20 + literal */
        int32_t bl = 1;
        int16_t bc = -1;
        int32_t node = 0;
        for (int64_t j = i; j < n; j++) {
            node = children[(int64_t)node * 256 + s[j]];
            if (node < 0) break;
            int16_t tc = term_code[node];
            if (tc < 0) continue;
            int64_t cand = cost[j + 1] + 1;
            int32_t len = (int32_t)(j + 1 - i);
            /* strictly cheaper, or equally cheap and longer (numba_impl.py:50) */
            if (cand < best || (cand == best && len > bl)) {
                best = cand;
                bl = len;
                bc = tc;
            }
        }
        cost[i] = best;
        blen[i] = bl;
        code[i] = bc;
    }
    int64_t w = 0;
    for (int64_t i = 0; i < n;) {
        if (code[i] < 0) {
            out[w++] = 0x20;
            out[w++] = s[i];
            (*esc)++;
            i++;
        } else {
            out[w++] = (uint8_t)code[i];
            i += blen[i];
        }
    }
    return w;
}

typedef struct {
    int64_t *cost;
    int32_t *blen;
    int16_t *code;
    int64_t cap;
} dp_scratch;

static int scratch_reserve(dp_scratch *sc, int64_t n) {
    if (n + 1 <= sc->cap) return 0;
    int64_t c = sc->cap ? sc->cap : 256;
    while (c < n + 1) c *= 2;
    free(sc->cost); free(sc->blen); free(sc->code);
    sc->cost = (int64_t *)malloc(sizeof(int64_t) * c);
    sc->blen = (int32_t *)malloc(sizeof(int32_t) * c);
    sc->code = (int16_t *)malloc(sizeof(int16_t) * c);
    sc->cap = c;
    return (sc->cost && sc->blen && sc->code) ? 0 : -1;
}

static void scratch_free(dp_scratch *sc) {
    free(sc->cost); free(sc->blen); free(sc->code);
    memset(sc, 0, sizeof *sc);
}

int64_t zo_compress_batch(const int32_t *children, const int16_t *term_code,
                          const uint8_t *flat, const int64_t *starts, int64_t n_lines,
                          uint8_t *out, int64_t *out_lens) {
    dp_scratch sc = {0};
    int64_t esc = 0;
    for (int64_t li = 0; li < n_lines; li++) {
        int64_t s = starts[li], n = starts[li + 1] - s;
        if (scratch_reserve(&sc, n)) { scratch_free(&sc); return -1; }
        out_lens[li] = compress_one(children, term_code, flat + s, n, out + 2 * s,
                                    sc.cost, sc.blen, sc.code, &esc);
    }
    scratch_free(&sc);
    return esc;
}

/* ------------------------------------------------------------------ */
/* decompress                                                           */
/* ------------------------------------------------------------------ */

/* Size + validate one record.  Returns status 0/1/2; *len, *errpos, *esc. */
static int decode_size_one(const int32_t *exp_len, const uint8_t *valid, const uint8_t *r,
                           int64_t n, int64_t *len, int64_t *errpos, int64_t *esc) {
    int64_t m = 0;
    *errpos = -1;
    for (int64_t i = 0; i < n;) {
        uint8_t b = r[i];
        if (b == 0x20) {
            if (i + 1 >= n) { *errpos = i; *len = 0; return ZO_ERR_TRUNCATED_ESCAPE; }
            m += 1;
            (*esc)++;
            i += 2;
        } else if (valid[b]) {
            m += exp_len[b];
            i += 1;
        } else {
            *errpos = i;
            *len = 0;
            return ZO_ERR_UNKNOWN_CODE;
        }
    }
    *len = m;
    return 0;
}

static int64_t decode_fill_one(const int64_t *exp_off, const uint8_t *exp_flat, const uint8_t *r,
                               int64_t n, uint8_t *out) {
    int64_t w = 0;
    for (int64_t i = 0; i < n;) {
        uint8_t b = r[i];
        if (b == 0x20) {
            out[w++] = r[i + 1];
            i += 2;
        } else {
            int64_t o = exp_off[b], e = exp_off[b + 1];
            memcpy(out + w, exp_flat + o, (size_t)(e - o));
            w += e - o;
            i += 1;
        }
    }
    return w;
}

void zo_decompress_sizes(const int32_t *exp_len, const uint8_t *valid, const uint8_t *flat,
                         const int64_t *starts, int64_t n_lines, int64_t *out_lens,
                         int8_t *status, int64_t *errpos, int64_t *total, int64_t *escapes) {
    int64_t tot = 0, esc = 0;
    for (int64_t li = 0; li < n_lines; li++) {
        int64_t s = starts[li];
        int st = decode_size_one(exp_len, valid, flat + s, starts[li + 1] - s, &out_lens[li],
                                 &errpos[li], &esc);
        /* status codes of the reference kernel: 1 unknown code, 2 truncated */
        status[li] = (int8_t)(st == 0 ? 0 : (st == ZO_ERR_UNKNOWN_CODE ? 1 : 2));
        tot += out_lens[li];
    }
    *total = tot;
    *escapes = esc;
}

void zo_decompress_fill(const int64_t *exp_off, const uint8_t *exp_flat, const uint8_t *flat,
                        const int64_t *starts, int64_t n_lines, const int8_t *status,
                        uint8_t *out, const int64_t *out_starts) {
    for (int64_t li = 0; li < n_lines; li++) {
        if (status[li] != 0) continue;
        decode_fill_one(exp_off, exp_flat, flat + starts[li], starts[li + 1] - starts[li],
                        out + out_starts[li]);
    }
}

/* ------------------------------------------------------------------ */
/* preprocess: tokenize, pair ring ids, colour intervals, re-emit       */
/* ------------------------------------------------------------------ */

enum { K_ATOM, K_BRACKET, K_BOND, K_BOPEN, K_BCLOSE, K_RING, K_DOT, K_OTHER };

static int is_digit(uint8_t b) { return b >= '0' && b <= '9'; }
static int is_letter(uint8_t b) { return (b >= 'A' && b <= 'Z') || (b >= 'a' && b <= 'z'); }
static int is_bond(uint8_t b) { return b && strchr("-=#$:/\\~", b) != NULL; }

typedef struct { int64_t start, end; int kind, rid; } tok_t;

/*
 * Preprocess one line with strict semantics.  On success returns 0 and writes
 * the renumbered line to out (capacity 3*n+3 is always enough) with *out_len.
 * On failure returns a ZO_ERR_* kind, with err->offset (bracket / percent) or
 * err->ids (unpaired ring ids bitmap) filled.  Lenient handling is the
 * caller's (smiles.py:196-202 vs pipeline.py:108-115).
 */
int zo_preprocess_line(const uint8_t *s, int64_t n, uint8_t *out, int64_t *out_len,
                       zo_err *err) {
    memset(err, 0, sizeof *err);
    err->offset = -1;
    tok_t *tok = (tok_t *)malloc(sizeof(tok_t) * (size_t)(n + 1));
    int64_t nt = 0;
    int ring_ok = 0;
    for (int64_t i = 0; i < n;) {
        uint8_t b = s[i];
        tok_t t = {i, i + 1, K_OTHER, -1};
        if (b == '[') {
            const uint8_t *c = (const uint8_t *)memchr(s + i + 1, ']', (size_t)(n - i - 1 > 0 ? n - i - 1 : 0));
            if (!c) { free(tok); err->offset = i; return ZO_ERR_UNBALANCED_BRACKET; }
            t.end = (c - s) + 1;
            t.kind = K_BRACKET;
        } else if (b == '%') {
            if (i + 2 >= n || !is_digit(s[i + 1]) || !is_digit(s[i + 2])) {
                free(tok);
                err->offset = i;
                return ZO_ERR_MALFORMED_PERCENT;
            }
            t.end = i + 3;
            if (ring_ok) { t.kind = K_RING; t.rid = (s[i + 1] - '0') * 10 + (s[i + 2] - '0'); }
        } else if (is_digit(b)) {
            if (ring_ok) { t.kind = K_RING; t.rid = b - '0'; }
        } else if (is_letter(b) || b == '*') {
            t.kind = K_ATOM;
        } else if (is_bond(b)) {
            t.kind = K_BOND;
        } else if (b == '(') {
            t.kind = K_BOPEN;
        } else if (b == ')') {
            t.kind = K_BCLOSE;
        } else if (b == '.') {
            t.kind = K_DOT;
        }
        tok[nt++] = t;
        i = t.end;
        ring_ok = t.kind == K_ATOM || t.kind == K_BRACKET || t.kind == K_BOND || t.kind == K_RING;
    }
    /* pair: occurrences of one id alternate open/close (smiles.py:140-159) */
    int64_t open_at[100];
    int64_t *partner = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nt + 1));
    int *color = (int *)malloc(sizeof(int) * (size_t)(nt + 1));
    for (int k = 0; k < 100; k++) open_at[k] = -1;
    int64_t n_int = 0;
    for (int64_t t = 0; t < nt; t++) {
        partner[t] = -1;
        color[t] = -1;
        if (tok[t].kind != K_RING) continue;
        int r = tok[t].rid;
        if (open_at[r] >= 0) {
            partner[t] = open_at[r];
            partner[open_at[r]] = t;
            open_at[r] = -1;
            n_int++;
        } else {
            open_at[r] = t;
        }
    }
    int any_open = 0;
    for (int k = 0; k < 100; k++)
        if (open_at[k] >= 0) { any_open = 1; err->ids[k >> 6] |= 1ull << (k & 63); }
    if (any_open) { free(tok); free(partner); free(color); return ZO_ERR_UNPAIRED_RING; }
    if (n_int == 0) {
        memcpy(out, s, (size_t)n);
        *out_len = n;
        free(tok); free(partner); free(color);
        return 0;
    }
    /* colour in closing order: smallest id unused by an already-coloured
     * overlapping interval (smiles.py:162-180).  Intervals coloured so far
     * all close before c, so (o2 < c and o < c2) reduces to c2 > o. */
    for (int64_t c = 0; c < nt; c++) {
        if (tok[c].kind != K_RING || partner[c] < 0 || partner[c] > c) continue;
        int64_t o = partner[c];
        uint64_t used[2] = {0, 0};
        for (int64_t c2 = o + 1; c2 < c; c2++)
            if (tok[c2].kind == K_RING && partner[c2] < c2 && color[c2] >= 0)
                used[color[c2] >> 6] |= 1ull << (color[c2] & 63);
        int col = 0;
        while (col < 128 && (used[col >> 6] >> (col & 63)) & 1) col++;
        if (col > 99) { free(tok); free(partner); free(color); return ZO_ERR_RING_OVERFLOW; }
        color[c] = col;
        color[o] = col;
    }
    int64_t w = 0;
    for (int64_t t = 0; t < nt; t++) {
        if (tok[t].kind == K_RING) {
            int col = color[t];
            if (col < 10) {
                out[w++] = (uint8_t)('0' + col);
            } else {
                out[w++] = '%';
                out[w++] = (uint8_t)('0' + col / 10);
                out[w++] = (uint8_t)('0' + col % 10);
            }
        } else {
            memcpy(out + w, s + tok[t].start, (size_t)(tok[t].end - tok[t].start));
            w += tok[t].end - tok[t].start;
        }
    }
    *out_len = w;
    free(tok); free(partner); free(color);
    return 0;
}

/* ------------------------------------------------------------------ */
/* whole-buffer stream: framing, policies, stats; pthread line shards  */
/* ------------------------------------------------------------------ */

typedef struct {
    /* inputs */
    const zo_tables *tb;
    const uint8_t *buf;
    const int64_t *ls, *le; /* line [start, end) */
    int64_t l0, l1;         /* line range of this shard */
    int direction, preprocess, lenient;
    /* outputs */
    uint8_t *out;
    int64_t out_len, cap;
    int64_t kept, escapes, skipped, flagged;
    int64_t err_line; /* 0-based line index of first strict error, -1 none */
    int err_kind;
    zo_err err;
    int64_t err_code;
    int oom;
} shard_t;

static int shard_grow(shard_t *sh, int64_t need) {
    if (sh->out_len + need <= sh->cap) return 0;
    int64_t c = sh->cap ? sh->cap : 1 << 16;
    while (c < sh->out_len + need) c *= 2;
    uint8_t *p = (uint8_t *)realloc(sh->out, (size_t)c);
    if (!p) { sh->oom = 1; return -1; }
    sh->out = p;
    sh->cap = c;
    return 0;
}

static void *shard_run(void *arg) {
    shard_t *sh = (shard_t *)arg;
    const zo_tables *tb = sh->tb;
    dp_scratch sc = {0};
    uint8_t *pre = NULL;
    int64_t pre_cap = 0;
    sh->err_line = -1;
    for (int64_t li = sh->l0; li < sh->l1; li++) {
        const uint8_t *s = sh->buf + sh->ls[li];
        int64_t n = sh->le[li] - sh->ls[li];
        if (sh->direction == ZO_COMPRESS) {
            if (memchr(s, '\r', (size_t)n)) {
                if (sh->lenient) { sh->skipped++; continue; }
                sh->err_line = li; sh->err_kind = ZO_ERR_CR; break;
            }
            if (sh->preprocess) {
                if (pre_cap < 3 * n + 3) {
                    free(pre);
                    pre_cap = 3 * n + 3;
                    pre = (uint8_t *)malloc((size_t)pre_cap);
                }
                int64_t m;
                zo_err e;
                int k = zo_preprocess_line(s, n, pre, &m, &e);
                if (k) {
                    if (!sh->lenient) { sh->err_line = li; sh->err_kind = k; sh->err = e; break; }
                    sh->flagged++;
                } else {
                    s = pre;
                    n = m;
                }
            }
            if (scratch_reserve(&sc, n) || shard_grow(sh, 2 * n + 1)) { sh->oom = 1; break; }
            sh->out_len += compress_one(tb->children, tb->term_code, s, n, sh->out + sh->out_len,
                                        sc.cost, sc.blen, sc.code, &sh->escapes);
            sh->out[sh->out_len++] = '\n';
            sh->kept++;
        } else {
            int64_t len, ep, esc = 0;
            int st = decode_size_one(tb->exp_len, tb->valid, s, n, &len, &ep, &esc);
            sh->escapes += esc;
            if (st) {
                if (!sh->lenient) {
                    sh->err_line = li;
                    sh->err_kind = st;
                    sh->err.offset = ep;
                    sh->err_code = s[ep];
                    break;
                }
                sh->skipped++;
                continue;
            }
            if (shard_grow(sh, len + 1)) break;
            sh->out_len += decode_fill_one(tb->exp_off, tb->exp_flat, s, n, sh->out + sh->out_len);
            sh->out[sh->out_len++] = '\n';
            sh->kept++;
        }
    }
    scratch_free(&sc);
    free(pre);
    return NULL;
}

/*
 * Whole-buffer compress/decompress with the reference stream semantics.
 * *out is malloc'd (free with zo_free).  Returns 0, or -1 on allocation
 * failure.  A strict-mode error fills st->err_* (err_line 1-based) and
 * leaves *out NULL.
 */
int zo_run_stream(const zo_tables *tb, const uint8_t *buf, int64_t n, int direction,
                  int preprocess, int lenient, int n_threads, uint8_t **out,
                  zo_stats *st) {
    memset(st, 0, sizeof *st);
    *out = NULL;
    st->in_bytes = n;
    /* framing (pipeline.py:49-74): split on 0x0A; a final partial line is a
     * line and clears `trailing` */
    int64_t n_lines = 0;
    for (int64_t i = 0; i < n; i++) n_lines += buf[i] == '\n';
    int trailing = 1;
    if (n > 0 && buf[n - 1] != '\n') { n_lines++; trailing = 0; }
    int64_t *ls = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_lines + 1));
    int64_t *le = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_lines + 1));
    if (!ls || !le) { free(ls); free(le); return -1; }
    int64_t k = 0, s0 = 0;
    for (int64_t i = 0; i < n; i++)
        if (buf[i] == '\n') { ls[k] = s0; le[k] = i; k++; s0 = i + 1; }
    if (!trailing) { ls[k] = s0; le[k] = n; k++; }
    if (n_threads < 1) n_threads = 1;
    if (n_threads > n_lines) n_threads = n_lines > 0 ? (int)n_lines : 1;
    shard_t *sh = (shard_t *)calloc((size_t)n_threads, sizeof(shard_t));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    for (int t = 0; t < n_threads; t++) {
        sh[t].tb = tb; sh[t].buf = buf; sh[t].ls = ls; sh[t].le = le;
        sh[t].l0 = n_lines * t / n_threads;
        sh[t].l1 = n_lines * (t + 1) / n_threads;
        sh[t].direction = direction; sh[t].preprocess = preprocess; sh[t].lenient = lenient;
    }
    for (int t = 1; t < n_threads; t++) pthread_create(&th[t], NULL, shard_run, &sh[t]);
    shard_run(&sh[0]);
    for (int t = 1; t < n_threads; t++) pthread_join(th[t], NULL);
    int rc = 0;
    int64_t total = 0;
    for (int t = 0; t < n_threads; t++) {
        if (sh[t].oom) rc = -1;
        st->escapes += sh[t].escapes;
        st->skipped += sh[t].skipped;
        st->flagged += sh[t].flagged;
        st->lines += sh[t].kept;
        total += sh[t].out_len;
        if (!st->err_line && sh[t].err_line >= 0) {
            /* first shard with an error holds the globally first bad line */
            st->err_line = sh[t].err_line + 1;
            st->err_kind = sh[t].err_kind;
            st->err_offset = sh[t].err.offset;
            st->err_ids[0] = sh[t].err.ids[0];
            st->err_ids[1] = sh[t].err.ids[1];
            st->err_code = sh[t].err_code;
        }
    }
    if (rc == 0 && !st->err_line) {
        /* b"\n".join(kept) + b"\n" iff trailing (pipeline.py:154-164) */
        if (st->lines > 0 && !trailing) total -= 1;
        uint8_t *o = (uint8_t *)malloc((size_t)(total > 0 ? total : 1));
        int64_t w = 0;
        for (int t = 0; t < n_threads && o; t++) {
            int64_t c = sh[t].out_len;
            if (w + c > total) c = total - w;
            memcpy(o + w, sh[t].out, (size_t)c);
            w += c;
        }
        if (!o) rc = -1;
        *out = o;
        st->out_bytes = total;
    }
    for (int t = 0; t < n_threads; t++) free(sh[t].out);
    free(sh); free(th); free(ls); free(le);
    return rc;
}

void zo_free(void *p) { free(p); }
