/*
 * zs_debug.h -- measurement and inspection hooks of libzs.so.
 *
 * Not part of the drop-in boundary (zs.h): tests and tools use these to pin
 * kernel variants against each other, to read the device tables the library
 * derives from a dictionary without a GPU, and to read per-phase clocks
 * (only in a library built with -DZS_PHASES=1; see tools/phase_cx.py).
 */
#ifndef ZS_DEBUG_H
#define ZS_DEBUG_H
#include "zs.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Host-only inspection (no GPU needed): derive the fast-path tables from a
 * reference trie.  dfa: uint16[256*97], codes: uint8[256*8].  Returns 1 if
 * the fast path applies, 0 if not, <0 on bad arguments. */
int zs_build_tables_host(const int32_t *children, const int16_t *term_code, int32_t n_nodes,
                         uint16_t *dfa, uint8_t *codes, int32_t *n_states, int32_t *max_len);
/* Host-only inspection of the cost-window transducer: dfa2 uint16[256*97],
 * t2 uint32[1024*16].  Returns 1 if built, 0 if the dictionary does not fit. */
int zs_build_t2_host(const int32_t *children, const int16_t *term_code, int32_t n_nodes,
                     uint16_t *dfa2, uint32_t *t2, int32_t *n_windows, int32_t *n_masks);

/* Host-only: the newline-aligned chunk boundaries zs_*_host would use for a
 * buffer with chunk size `chunk` bytes (cuts[0] = 0 ... n).  Writes up to cap
 * entries; returns the number of boundaries, or <0 on bad arguments. */
int64_t zs_debug_chunk_cuts(const uint8_t *h_in, int64_t n, int64_t chunk, int64_t *cuts, int64_t cap);

/* compress-kernel selection for parity tests and ablations (default 3):
 * bits 0+1 clear: the generic key-window / trie-walk kernel (compress_tiles);
 * bit 4: compress_cx parses line-lane ranges instead of byte-exact slices;
 * bit 6: compress_cx parses with the DFA + cost-window transducer instead of
 * the product automaton; bit 7: compress_cx runs every phase on byte-exact
 * slices (balanced lanes, block barriers between phases); bit 8: lines longer
 * than the staged window go to the general routine (one thread each) instead
 * of the block-parallel long-line kernels */
int zs_set_transducer(zs_ctx *ctx, int on);

/* profiling aid: per-phase SM cycles of the tile kernels (summed over CTAs,
 * thread 0's view) for the last device-API call; off by default */
int zs_set_phase_timing(zs_ctx *ctx, int on);
int zs_last_phase_cycles(zs_ctx *ctx, uint64_t *cycles8);

#ifdef __cplusplus
}
#endif
#endif
