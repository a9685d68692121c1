/*
 * Synthetic SMILES library generator for the benchmark / parity configs.
 *
 * Byte-exact restatement of the reference corpus generator
 * (pkg/scripts/make_corpus.py:30-136, MoleculeGen) driven by an exact port
 * of CPython's `random.Random` (Mersenne Twister MT19937, init_by_array
 * seeding, random() 53-bit doubles, _randbelow via getrandbits, choice,
 * randint).  Same seed -> same bytes as the reference Python generator, so
 * the golden hashes in tests/golden/corpus_hashes.json (computed by running
 * the reference) pin it.  This is bench/test input plumbing, not part of the
 * codec path.
 *
 * Configs:
 *   kind 0/1/2: MoleculeGen(Random(seed), frac) one molecule per line
 *   kind 3    : C3 skewed lines, molecules joined with LINKERS up to a
 *               U[20,1000] target, never exceeding 1000 bytes.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

/* ---------------- CPython-compatible MT19937 ---------------- */
enum { MT_N = 624, MT_M = 397 };
typedef struct { uint32_t s[MT_N]; int i; } mt_t;

static void mt_init_genrand(mt_t *m, uint32_t seed) {
    m->s[0] = seed;
    for (int k = 1; k < MT_N; k++)
        m->s[k] = 1812433253u * (m->s[k - 1] ^ (m->s[k - 1] >> 30)) + (uint32_t)k;
    m->i = MT_N;
}

static void mt_init_by_array(mt_t *m, const uint32_t *key, int len) {
    mt_init_genrand(m, 19650218u);
    int i = 1, j = 0;
    for (int k = (MT_N > len ? MT_N : len); k; k--) {
        m->s[i] = (m->s[i] ^ ((m->s[i - 1] ^ (m->s[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
        i++; j++;
        if (i >= MT_N) { m->s[0] = m->s[MT_N - 1]; i = 1; }
        if (j >= len) j = 0;
    }
    for (int k = MT_N - 1; k; k--) {
        m->s[i] = (m->s[i] ^ ((m->s[i - 1] ^ (m->s[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
        i++;
        if (i >= MT_N) { m->s[0] = m->s[MT_N - 1]; i = 1; }
    }
    m->s[0] = 0x80000000u;
}

static uint32_t mt_next(mt_t *m) {
    if (m->i >= MT_N) {
        static const uint32_t mag[2] = {0u, 0x9908b0dfu};
        int k;
        for (k = 0; k < MT_N - MT_M; k++) {
            uint32_t y = (m->s[k] & 0x80000000u) | (m->s[k + 1] & 0x7fffffffu);
            m->s[k] = m->s[k + MT_M] ^ (y >> 1) ^ mag[y & 1u];
        }
        for (; k < MT_N - 1; k++) {
            uint32_t y = (m->s[k] & 0x80000000u) | (m->s[k + 1] & 0x7fffffffu);
            m->s[k] = m->s[k + (MT_M - MT_N)] ^ (y >> 1) ^ mag[y & 1u];
        }
        uint32_t y = (m->s[MT_N - 1] & 0x80000000u) | (m->s[0] & 0x7fffffffu);
        m->s[MT_N - 1] = m->s[MT_M - 1] ^ (y >> 1) ^ mag[y & 1u];
        m->i = 0;
    }
    uint32_t y = m->s[m->i++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* random.Random(seed) for a non-negative int seed < 2**64 */
static void py_seed(mt_t *m, uint64_t seed) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    mt_init_by_array(m, key, (seed >> 32) ? 2 : 1);
}

static double py_random(mt_t *m) {
    uint32_t a = mt_next(m) >> 5, b = mt_next(m) >> 6;
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

/* Random._randbelow_with_getrandbits for 1 <= n < 2**32 */
static uint32_t py_below(mt_t *m, uint32_t n) {
    int k = 32 - __builtin_clz(n);
    uint32_t r = mt_next(m) >> (32 - k);
    while (r >= n) r = mt_next(m) >> (32 - k);
    return r;
}

static int py_randint(mt_t *m, int a, int b) { return a + (int)py_below(m, (uint32_t)(b - a + 1)); }

/* ---------------- fragment vocabularies (make_corpus.py:16-28) ---------------- */
#define COUNT(a) ((int)(sizeof(a) / sizeof((a)[0])))
static const char *const ARO_SUB[] = {"F", "Cl", "Br", "I", "C", "CC", "O", "OC", "N", "C#N",
    "C(F)(F)F", "OC(F)F", "N(C)C", "[N+](=O)[O-]", "C(=O)O", "C(=O)N", "C(=O)NC",
    "S(=O)(=O)N", "OCC", "NC(=O)C", "C=O"};
static const char *const CHN_SUB[] = {"C", "CC", "O", "N", "CO", "OC", "F", "C(C)C", "C(=O)O",
    "C(=O)OC", "NC", "C#N", "OCC", "CCO"};
static const char *const LINK[] = {"", "", "C", "CC", "CCC", "O", "N", "CN", "NC", "OC", "S",
    "C(=O)", "C(=O)N", "NC(=O)", "C(=O)O", "OC(=O)", "S(=O)(=O)", "C=C", "/C=C/", "C#C",
    "CNC", "COC", "N(C)"};
static const char *const STEREO[] = {"[C@H](C)", "[C@@H](C)", "[C@H](O)", "[C@@H](N)",
    "[C@H](CC)", "[C@@H](CO)"};
static const char *const BRACK[] = {"[nH]", "[N+](C)(C)C", "[O-]", "[NH3+]", "[13C]", "[2H]",
    "[Si](C)(C)C"};
static const char *const SALT[] = {".Cl", ".Br", ".[Na+]", ".[K+]", ".O", ".OC(=O)C(=O)O"};
static const char *const RARE[] = {"~", ":", "$", "*"};

/* Ring templates.  'a','b','r' = ring-id slots, '0'..'3' = decoration slots.
 * Aromatic: the first template is the fused (two-id, 3-slot) case; the rest
 * are single-id cores selected by the same roll thresholds as the reference. */
typedef struct { double upto; const char *tpl; } core_t;
static const core_t ARO_CORES[] = {
    {0.28, "cr" "nc0c1c2cr"}, {0.38, "crcc0c1or"}, {0.46, "crcc0c1sr"},
    {0.56, "crcc0c1[nH]r"}, {0.62, "crncnc0cr"}, {2.0, "crc0c1c2c3cr"}};
static const core_t ALI_CORES[] = {
    {0.22, "CrCC0C1CCr"}, {0.42, "CrCC0NC1Cr"}, {0.54, "CrCN0CCNr"}, {0.66, "CrCC0OCr"},
    {0.76, "CrCOCC0Nr"}, {0.88, "CrCC0C1Cr"}, {2.0, "CrCCr"}};
static const char *const FUSED = "cacc0cbcc1cc2cbca";

/* ---------------- growable byte buffer ---------------- */
typedef struct { char *p; size_t n, cap; } buf_t;
static void put(buf_t *b, const char *s, size_t k) {
    if (b->n + k > b->cap) {
        size_t c = b->cap ? b->cap : 4096;
        while (c < b->n + k) c *= 2;
        b->p = (char *)realloc(b->p, c);
        b->cap = c;
    }
    memcpy(b->p + b->n, s, k);
    b->n += k;
}
static void puts_(buf_t *b, const char *s) { put(b, s, strlen(s)); }

typedef struct { mt_t mt; double aro; int next_ring; } gen_t;

static void ring_text(int r, char *out) {
    if (r < 10) snprintf(out, 16, "%d", r);
    else snprintf(out, 16, "%%%02d", r);
}

/* MoleculeGen.sub (make_corpus.py:47-53) */
static void sub(gen_t *g, const char *const *pool, int npool, buf_t *o) {
    if (py_random(&g->mt) < 0.06) {
        puts_(o, STEREO[py_below(&g->mt, COUNT(STEREO))]);
        puts_(o, CHN_SUB[py_below(&g->mt, COUNT(CHN_SUB))]);
        return;
    }
    if (py_random(&g->mt) < 0.05) { puts_(o, BRACK[py_below(&g->mt, COUNT(BRACK))]); return; }
    puts_(o, pool[py_below(&g->mt, (uint32_t)npool)]);
}

/* _decorate: slot k is "(" + sub + ")" with probability p, else "" */
static void decorate(gen_t *g, int slots, const char *const *pool, int npool, double p,
                     buf_t deco[4]) {
    for (int k = 0; k < slots; k++) {
        deco[k].n = 0;
        if (py_random(&g->mt) < p) {
            put(&deco[k], "(", 1);
            sub(g, pool, npool, &deco[k]);
            put(&deco[k], ")", 1);
        }
    }
}

static void fill(buf_t *o, const char *tpl, const char *ra, const char *rb, buf_t deco[4]) {
    for (const char *c = tpl; *c; c++) {
        switch (*c) {
        case 'a': case 'r': puts_(o, ra); break;
        case 'b': puts_(o, rb); break;
        case '0': case '1': case '2': case '3': put(o, deco[*c - '0'].p, deco[*c - '0'].n); break;
        default: put(o, c, 1);
        }
    }
}

static void aromatic_ring(gen_t *g, buf_t *o, buf_t deco[4]) {
    double roll = py_random(&g->mt);
    char ra[16], rb[16];
    if (roll < 0.08) {
        ring_text(g->next_ring++, ra);
        ring_text(g->next_ring++, rb);
        decorate(g, 3, ARO_SUB, COUNT(ARO_SUB), 0.25, deco);
        fill(o, FUSED, ra, rb, deco);
        return;
    }
    decorate(g, 4, ARO_SUB, COUNT(ARO_SUB), 0.3, deco);
    ring_text(g->next_ring++, ra);
    int k = 0;
    while (roll >= ARO_CORES[k].upto) k++;
    fill(o, ARO_CORES[k].tpl, ra, ra, deco);
}

static void aliphatic_ring(gen_t *g, buf_t *o, buf_t deco[4]) {
    char r[16];
    ring_text(g->next_ring++, r);
    decorate(g, 3, CHN_SUB, COUNT(CHN_SUB), 0.25, deco);
    double roll = py_random(&g->mt);
    int k = 0;
    while (roll >= ALI_CORES[k].upto) k++;
    fill(o, ALI_CORES[k].tpl, r, r, deco);
}

static void fragment(gen_t *g, buf_t *o, buf_t deco[4]) {
    if (py_random(&g->mt) < g->aro) aromatic_ring(g, o, deco);
    else aliphatic_ring(g, o, deco);
}

static void chain(gen_t *g, buf_t *o) {
    int n = py_randint(&g->mt, 1, 3);
    for (int k = 0; k < n; k++) {
        puts_(o, CHN_SUB[py_below(&g->mt, COUNT(CHN_SUB))]);
        if (py_random(&g->mt) < 0.15) {
            put(o, "(", 1);
            puts_(o, CHN_SUB[py_below(&g->mt, COUNT(CHN_SUB))]);
            put(o, ")", 1);
        }
    }
}

/* MoleculeGen.molecule (make_corpus.py:110-136); appends to o */
static void molecule(gen_t *g, buf_t *o, buf_t scratch[6]) {
    g->next_ring = 1;
    buf_t *deco = scratch;       /* 4 slots */
    buf_t *body = &scratch[4];
    buf_t *pre = &scratch[5];
    if (py_random(&g->mt) < 0.02) {
        int n = py_randint(&g->mt, 10, 14);
        for (int k = 0; k < n; k++) {
            char r[16];
            ring_text(g->next_ring++, r);
            if (k) put(o, "C", 1);
            int four = py_random(&g->mt) < 0.5;
            put(o, "C", 1); puts_(o, r);
            puts_(o, four ? "CC" : "CCC");
            puts_(o, r);
        }
        return;
    }
    body->n = 0;
    fragment(g, body, deco);
    int links = py_randint(&g->mt, 0, 3);
    for (int k = 0; k < links; k++) {
        puts_(body, LINK[py_below(&g->mt, COUNT(LINK))]);
        fragment(g, body, deco);
    }
    pre->n = 0;
    if (py_random(&g->mt) < 0.3) chain(g, pre);
    put(o, pre->p, pre->n);
    put(o, body->p, body->n);
    if (py_random(&g->mt) < 0.25) chain(g, o);
    if (py_random(&g->mt) < 0.04) puts_(o, SALT[py_below(&g->mt, COUNT(SALT))]);
    if (py_random(&g->mt) < 0.004) {
        puts_(o, RARE[py_below(&g->mt, COUNT(RARE))]);
        put(o, "C", 1);
    }
}

/*
 * Generate n_lines newline-terminated lines.  Returns a malloc'd buffer
 * (free with synth_free) and its size in *out_len.
 * kind: 0 mixed (0.5), 1 aromatic (0.92), 2 aliphatic (0.08), 3 skewed (0.5).
 */
char *synth_generate(int kind, uint64_t seed, int64_t n_lines, int64_t *out_len) {
    gen_t g;
    static const double FRAC[4] = {0.5, 0.92, 0.08, 0.5};
    if (kind < 0 || kind > 3) return NULL;
    py_seed(&g.mt, seed);
    g.aro = FRAC[kind];
    buf_t out = {0}, line = {0}, nxt = {0};
    buf_t scratch[6];
    memset(scratch, 0, sizeof scratch);
    for (int64_t i = 0; i < n_lines; i++) {
        if (kind != 3) {
            molecule(&g, &out, scratch);
        } else {
            int target = py_randint(&g.mt, 20, 1000);
            line.n = 0;
            molecule(&g, &line, scratch);
            while ((int)line.n < target) {
                nxt.n = 0;
                puts_(&nxt, LINK[py_below(&g.mt, COUNT(LINK))]);
                molecule(&g, &nxt, scratch);
                if (line.n + nxt.n > 1000) break;
                put(&line, nxt.p, nxt.n);
            }
            put(&out, line.p, line.n);
        }
        put(&out, "\n", 1);
    }
    for (int k = 0; k < 6; k++) free(scratch[k].p);
    free(line.p);
    free(nxt.p);
    *out_len = (int64_t)out.n;
    return out.p;
}

void synth_free(char *p) { free(p); }
