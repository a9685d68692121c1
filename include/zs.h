/*
 * zs.h -- C ABI of the B200-native ZSMILES per-line codec (libzs.so).
 *
 * Plain pointers and sizes only; no torch / CUDA types cross this boundary.
 * Every entry point returns an int status (ZS_OK or a negative ZS_E_*) and
 * never throws.  Per-line data errors (decode failures, preprocess errors,
 * carriage returns) are *results*, reported in zs_result, not call failures.
 *
 * Two surfaces, both replacing the reference's Python->numba plugin seam
 * (pkg/src/zsmiles/kernels/__init__.py:28-33, called from codec.py:38-39,
 * 64-70):
 *
 *  1. Fine-grained parity shim with the exact semantics/layouts of the
 *     reference kernels (host pointers; the library stages them through HBM):
 *       zs_compress_batch    <- kernels.compress_batch   numba_impl.py:16-71
 *       zs_decompress_sizes  <- kernels.decompress_sizes numba_impl.py:74-112
 *       zs_decompress_fill   <- kernels.decompress_fill  numba_impl.py:115-139
 *       zs_preprocess_batch  <- smiles.preprocess_line   smiles.py:183-213
 *
 *  2. Coarse whole-buffer API (the hot path): one newline-framed buffer in,
 *     one newline-framed buffer out, with the stream semantics of
 *     pipeline.run_stream (pipeline.py:97-167): framing, CR policy,
 *     strict/lenient, stats, first error with its 1-based line number.
 *       zs_compress_device / zs_decompress_device   (buffers already in HBM)
 *       zs_compress_host   / zs_decompress_host     (host buffers; chunked,
 *                                                    H2D/D2H overlapped)
 *
 * Dictionary tables are passed in the reference's own layouts
 * (Dictionary.encode_trie -> trie.py:22-50; Dictionary.decode_tables ->
 * dictionary.py:112-129); the library derives its device tables from them.
 *
 * Measurement and table-inspection hooks (kernel-variant switches, phase
 * clocks, host-side table builders) are not part of this boundary; they are
 * declared in zs_debug.h.
 */
#ifndef ZS_H
#define ZS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ZS_OK = 0,
    ZS_E_ARG = -1,      /* bad argument */
    ZS_E_CUDA = -2,     /* CUDA runtime error (see zs_last_error) */
    ZS_E_NOMEM = -3,    /* device or host allocation failed */
    ZS_E_NODICT = -4,   /* no dictionary uploaded */
    ZS_E_CAPACITY = -5  /* caller's output buffer too small (result.out_bytes = needed) */
};

/* per-line error kinds (pipeline.py:106-107, smiles.py:99-176, errors.py:64-78) */
enum {
    ZS_ERR_NONE = 0,
    ZS_ERR_CR = 1,                 /* "carriage return in line" */
    ZS_ERR_UNBALANCED_BRACKET = 2, /* "unclosed '[' at offset {offset}" */
    ZS_ERR_MALFORMED_PERCENT = 3,  /* "'%' without two digits at offset {offset}" */
    ZS_ERR_UNPAIRED_RING = 4,      /* "ring id(s) {ids} never close" */
    ZS_ERR_RING_OVERFLOW = 5,      /* "more than 100 mutually overlapping rings" */
    ZS_ERR_UNKNOWN_CODE = 6,       /* "unknown code 0x{code:02x} at offset {offset} ..." */
    ZS_ERR_TRUNCATED_ESCAPE = 7    /* "payload ends with a dangling escape at offset {offset}" */
};

/* flags for the whole-buffer calls */
enum { ZS_F_PREPROCESS = 1, ZS_F_LENIENT = 2 };

typedef struct zs_ctx zs_ctx;

/* CorpusStats (pipeline.py:21-40) + first strict error */
typedef struct {
    int64_t lines;      /* records written */
    int64_t in_bytes;
    int64_t out_bytes;
    int64_t escapes;
    int64_t skipped;
    int64_t flagged;
    int64_t err_line;   /* 1-based line of the first strict-mode error, 0 = none */
    int32_t err_kind;   /* ZS_ERR_* */
    int32_t err_code;   /* offending byte for ZS_ERR_UNKNOWN_CODE */
    int64_t err_offset; /* in-line byte offset (bracket, percent, decode errors) */
    uint64_t err_ids[2];/* bitmap of unpaired ring ids 0..99 (ZS_ERR_UNPAIRED_RING) */
    int32_t gpu_launches; /* kernels launched by this call */
    int32_t pad;
} zs_result;

/* ---- context / dictionary ---- */
int zs_ctx_create(int device, zs_ctx **out);
int zs_ctx_destroy(zs_ctx *ctx);
const char *zs_last_error(zs_ctx *ctx);
int zs_device_count(int *n);

/* children: int32 [n_nodes][256] (-1 = no edge, row 0 = root)
 * term_code: int16 [n_nodes] (-1 = not terminal)
 * exp_len: int32[256], valid: uint8[256], exp_off: int64[257], exp_flat: uint8[exp_off[256]] */
int zs_set_dictionary(zs_ctx *ctx, const int32_t *children, const int16_t *term_code,
                      int32_t n_nodes, const int32_t *exp_len, const uint8_t *valid,
                      const int64_t *exp_off, const uint8_t *exp_flat);
/* DFA window width (2/4/6/8) if the sm_100a fast path (shared-memory DFA)
 * serves the uploaded dictionary, 0 for the generic trie walk */
int zs_dictionary_fast(zs_ctx *ctx);
/* Random access (pkg/README.md:106-110: "grab line i,
 * decode line i") into a compressed library resident in HBM.
 * zs_index_build: d_offsets[r] = first byte of record r (records framed by
 * '\n' as pipeline.py:49-74 splits them), d_offsets[*n_records] = one past
 * the last record's end + 1; needs cap >= records + 1 (else ZS_E_CAPACITY
 * with *n_records set).
 * zs_decode_records: decodes the k records d_idx[] (device) into d_out,
 * record j at d_out_off[j] (k + 1 offsets), with the reference's per-record
 * outcome (numba_impl.py:74-139): d_status 0 ok, 1 unknown code, 2 dangling
 * escape, 3 no such record; d_errpos = offset (| code << 40 for status 1).
 * *total_out = output bytes (ZS_E_CAPACITY when out_cap is smaller). */
int zs_index_build(zs_ctx *ctx, const uint8_t *d_comp, int64_t n, uint64_t *d_offsets, int64_t cap,
                   int64_t *n_records);
int zs_decode_records(zs_ctx *ctx, const uint8_t *d_comp, const uint64_t *d_offsets, int64_t n_records,
                      const int64_t *d_idx, int64_t k, uint8_t *d_out, int64_t out_cap, int64_t *d_out_off,
                      int8_t *d_status, int64_t *d_errpos, int64_t *total_out);
/* ---- dictionary training (dictionary.py:169-320) ----
 * zs_train_count: census of h_buf = b"\n".join(lines) (count_substrings,
 * dictionary.py:169-221): every alphabet-only window of length l_min..l_max
 * (2 <= l_min <= l_max <= 64, n < 2^32), kept on the device as the rank
 * table; *n_rows = its rows.  zs_train_rows copies the rows to the host in
 * the reference's RankTable order (length-major, bytewise ascending): row r
 * is h_buf[pos[r] : pos[r] + len[r]], occurring occ[r] times.
 * zs_train_load replaces the device rank table with a host one (RankTable
 * layout: patterns u8[m][width] zero-padded, lengths, occurrences).
 * zs_train_select: select_patterns(table, t) (dictionary.py:241-307) with
 * working-set cap `cap` (reference default 200000) -> rows_out[0..*n) in
 * code order (0x80 + k).
 * zs_overlap_batch: overlap_batch (numba_impl.py:142-169) on the reference
 * trie layout (children int32[n_nodes][256], term_len int16[n_nodes]). */
int zs_train_count(zs_ctx *ctx, const uint8_t *h_buf, int64_t n, int32_t l_min, int32_t l_max, int64_t *n_rows);
int zs_train_rows(zs_ctx *ctx, int64_t *pos, int32_t *len, int64_t *occ);
int zs_train_load(zs_ctx *ctx, const uint8_t *patterns, int32_t width, const int64_t *lengths, const int64_t *occ,
                  int64_t m);
int zs_train_select(zs_ctx *ctx, int32_t t, int64_t cap, int64_t *rows_out, int32_t *n_selected);
int zs_overlap_batch(zs_ctx *ctx, const int32_t *children, const int16_t *term_len, int32_t n_nodes,
                     const uint8_t *pats, int32_t width, const int64_t *lens, int64_t n, int64_t *out);

/* ---- fine-grained parity shim (reference kernel layouts, host memory) ---- */
/* out must hold 2*starts[n_lines] bytes; record i lands at out[2*starts[i]] */
int zs_compress_batch(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts, int64_t n_lines,
                      uint8_t *out, int64_t *out_lens, int64_t *escapes);
int zs_decompress_sizes(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts,
                        int64_t n_lines, int64_t *out_lens, int8_t *status, int64_t *errpos,
                        int64_t *total, int64_t *escapes);
int zs_decompress_fill(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts, int64_t n_lines,
                       const int8_t *status, uint8_t *out, const int64_t *out_starts);
/* out must hold 3*starts[n_lines] + 3*n_lines bytes; line i lands at
 * out[3*starts[i] + 3*i] with length out_lens[i]; status[i] = ZS_ERR_* with
 * err_off[i] / err_ids[2*i..2*i+1] filled on error (strict semantics). */
int zs_preprocess_batch(zs_ctx *ctx, const uint8_t *flat, const int64_t *starts,
                        int64_t n_lines, uint8_t *out, int64_t *out_lens, int8_t *status,
                        int64_t *err_off, uint64_t *err_ids);

/* ---- whole-buffer stream API (hot path) ---- */
/* device pointers; d_out must hold out_cap bytes.  Runs on the context's
 * stream and synchronises before returning. */
int zs_compress_device(zs_ctx *ctx, const uint8_t *d_in, int64_t n, uint8_t *d_out,
                       int64_t out_cap, int flags, zs_result *res);
int zs_decompress_device(zs_ctx *ctx, const uint8_t *d_in, int64_t n, uint8_t *d_out,
                         int64_t out_cap, int flags, zs_result *res);
/* host pointers (pinned memory gives full PCIe rate) */
int zs_compress_host(zs_ctx *ctx, const uint8_t *h_in, int64_t n, uint8_t *h_out,
                     int64_t out_cap, int flags, zs_result *res);
int zs_decompress_host(zs_ctx *ctx, const uint8_t *h_in, int64_t n, uint8_t *h_out,
                       int64_t out_cap, int flags, zs_result *res);

/* page-locked host memory for the host-pointer calls (cudaHostAlloc):
 * full PCIe rate for run_stream's segments */
int zs_host_alloc(zs_ctx *ctx, int64_t bytes, void **p);
int zs_host_free(zs_ctx *ctx, void *p);

/* upper bound of the output size for an n-byte input (for buffer sizing) */
int64_t zs_compress_bound(int64_t n);
int64_t zs_decompress_bound(zs_ctx *ctx, int64_t n);

/* timing of the last whole-buffer call's main kernel (CUDA events on the
 * launching stream), milliseconds */
float zs_last_kernel_ms(zs_ctx *ctx);
/* name of that kernel (static string) */
const char *zs_last_kernel(zs_ctx *ctx);
/* the cudaStream_t the device API launches on (for events around whole calls) */
void *zs_stream(zs_ctx *ctx);
/* Stream ordering of the device-pointer calls (zs_*_device, zs_index_build,
 * zs_decode_records): each call first waits (cudaStreamWaitEvent) for all
 * work queued so far on `stream` (a cudaStream_t; NULL = the legacy default
 * stream, the initial setting), so buffers a caller's kernels or copies are
 * still writing are not read early.  The calls return after their own work
 * is complete, so their outputs are ready on every stream when they return. */
int zs_set_stream(zs_ctx *ctx, void *stream);

#ifdef __cplusplus
}
#endif
#endif
