/* ORACLE -- TEST INFRASTRUCTURE ONLY.  See zs_oracle.c. */
#ifndef ZS_ORACLE_H
#define ZS_ORACLE_H
#include <stdint.h>

/* error kinds shared with include/zs.h */
enum {
    ZO_OK = 0,
    ZO_ERR_CR = 1,                 /* pipeline.py:106-107 */
    ZO_ERR_UNBALANCED_BRACKET = 2, /* smiles.py:99 */
    ZO_ERR_MALFORMED_PERCENT = 3,  /* smiles.py:105 */
    ZO_ERR_UNPAIRED_RING = 4,      /* smiles.py:157-158 */
    ZO_ERR_RING_OVERFLOW = 5,      /* smiles.py:176 */
    ZO_ERR_UNKNOWN_CODE = 6,       /* errors.py:64-72 */
    ZO_ERR_TRUNCATED_ESCAPE = 7,   /* errors.py:75-78 */
};

enum { ZO_COMPRESS = 0, ZO_DECOMPRESS = 1 };

typedef struct {
    int64_t offset;
    uint64_t ids[2];
} zo_err;

typedef struct {
    const int32_t *children; /* [n_nodes][256] */
    const int16_t *term_code;
    const int32_t *exp_len;  /* [256] */
    const uint8_t *valid;    /* [256] */
    const int64_t *exp_off;  /* [257] */
    const uint8_t *exp_flat;
} zo_tables;

typedef struct {
    int64_t lines, in_bytes, out_bytes, escapes, skipped, flagged;
    int64_t err_line; /* 1-based; 0 = none */
    int64_t err_kind, err_offset, err_code;
    uint64_t err_ids[2];
} zo_stats;

int64_t zo_compress_batch(const int32_t *children, const int16_t *term_code,
                          const uint8_t *flat, const int64_t *starts, int64_t n_lines,
                          uint8_t *out, int64_t *out_lens);
void zo_decompress_sizes(const int32_t *exp_len, const uint8_t *valid, const uint8_t *flat,
                         const int64_t *starts, int64_t n_lines, int64_t *out_lens,
                         int8_t *status, int64_t *errpos, int64_t *total, int64_t *escapes);
void zo_decompress_fill(const int64_t *exp_off, const uint8_t *exp_flat, const uint8_t *flat,
                        const int64_t *starts, int64_t n_lines, const int8_t *status,
                        uint8_t *out, const int64_t *out_starts);
int zo_preprocess_line(const uint8_t *s, int64_t n, uint8_t *out, int64_t *out_len, zo_err *err);
int zo_run_stream(const zo_tables *tb, const uint8_t *buf, int64_t n, int direction,
                  int preprocess, int lenient, int n_threads, uint8_t **out, zo_stats *st);
void zo_free(void *p);

/* dictionary training (zs_oracle_train.c): rows malloc'd, free with zo_free */
int64_t zo_count_substrings(const uint8_t *buf, int64_t n, int lmin, int lmax, int64_t **pos_out,
                            int32_t **len_out, int64_t **occ_out);
int64_t zo_overlap(const uint8_t *p, int n, const uint8_t *sel, const int32_t *sel_len, int nsel);
int64_t zo_select_patterns(const uint8_t *buf, const int64_t *pos, const int32_t *len, const int64_t *occ,
                           int64_t m, int t, int64_t cap, int64_t *out);
#endif
