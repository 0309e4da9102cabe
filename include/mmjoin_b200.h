/* mmjoin_b200.h -- C ABI of the B200 join-project engine (libmmjoin_b200.so).
 *
 * Every entry point takes plain device pointers, 64-bit sizes and a CUDA
 * stream handle (cudaStream_t passed as void*), returns 0 on success or a
 * positive MMJ_ERR_* status, and never allocates or frees caller memory.
 * Scratch comes from caller workspaces sized by the *_bytes / *_count
 * queries.  The message of the last failure on the calling thread is
 * available from mmj_last_error().
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/mmjoin/):
 *   the only native FFI of the reference is the Cython kernel
 *     matmul_int64(a, b, out, row_start, row_end, block)   matmul/_kernel_cy.pyx:42-47
 *   behind multiply_counts(a, b, cores, backend)            matmul/core.py:95-123;
 *   the remaining entry points replace the numpy operators of the path:
 *     degree split            joinproject.py:100-116, 178-180
 *     heavy_matrices          joinproject.py:119-143
 *     light passes 1..3       joinproject.py:183-203 (+ gather_ranges relation.py:193-204)
 *     merge / np.unique       joinproject.py:220-225, _merge_counts 146-152
 *     full_join_dedup         joinproject.py:228-248
 *     star heavy part         joinproject.py:320-365
 *     bsi_answer_batch        apps.py:314-351
 */
#ifndef MMJOIN_B200_H
#define MMJOIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMJ_OK 0
#define MMJ_ERR_ARG 1          /* -> ValueError                        */
#define MMJ_ERR_CUDA 2         /* -> RuntimeError                      */
#define MMJ_ERR_OVERFLOW 3     /* -> MatrixOverflowError (core.py:33)  */
#define MMJ_ERR_UNSUPPORTED 4  /* -> NotImplementedError               */
#define MMJ_ERR_CAPACITY 5     /* -> output buffer too small           */

#define MMJ_MODE_BITMAP 0      /* nonzero test -> 1 bit per (row, col)  */
#define MMJ_MODE_COUNT32 1     /* exact int32 counts                    */
#define MMJ_MODE_ACC64 2       /* out += count << shift (int64)         */
#define MMJ_MODE_BITMAP_U8 3   /* BITMAP, caller guarantees counts < 256 (<= 255 nonzero K columns) */
#define MMJ_MODE_BITMAP_PAIR 4 /* BITMAP over a z-pair B operand (mmj_build_operand_pairs): b_rows = pair
                                  rows, 2 bits per accumulator; needs every count < 128 (a side whose
                                  heavy degrees are <= 127); ld_out*16 >= b_rows rounded up to 256 */
#define MMJ_MODE_COUNT16 5     /* exact counts as uint16 (caller guarantees every count < 65536); ld_out in
                                  uint16 elements, multiple of 8 */
#define MMJ_MODE_UPPER 16      /* OR-flag: self-join, skip tiles whose columns are all <= their rows
                                  (cells there are left unwritten; consumers keep z > x only) */

int mmj_abi_version(void);
const char* mmj_last_error(void);
int mmj_set_device(int device);
int mmj_sm_count(void);
/* number of kernels this library has launched in the process */
long long mmj_launch_count(void);

/* ---- scans ------------------------------------------------------------- */
size_t mmj_scan_workspace_bytes(int64_t n);
/* out[i] = sum(in[0..i)), out[n] = total  (int32 in, int64 out) */
int mmj_exclusive_scan_i32(const int32_t* in, int64_t* out, int64_t n, void* ws, void* stream);
/* order-sensitive checksum of n codes (parity stamps of chunked outputs):
 * out[0] += sum(codes[i]), out[1] += sum((base+i+1) * codes[i]), mod 2^64;
 * out: 2 x uint64 on the device, accumulated (zero it first); additive over
 * consecutive chunks when base = the number of codes before the chunk. */
int mmj_code_checksum(const int64_t* codes, int64_t n, int64_t base, unsigned long long* out, void* stream);

/* ---- degree split: joinproject.py:178-180 ----------------------------------
 * hpos[y] = rank of y among heavy y (deg_R(y) > delta1 or deg_S(y) > delta1),
 * -1 for light y.  scan_out[dom_y] receives K = number of heavy y.
 * flag_ws: dom_y bytes; scan_out: dom_y+1 int32. */
int mmj_heavy_y_positions(const int32_t* rdeg_y, const int32_t* sdeg_y, int64_t dom_y, int64_t delta1,
                          uint8_t* flag_ws, int32_t* scan_out, int32_t* hpos, void* ws, void* stream);

/* ---- heavy operand build: joinproject.py:119-143 ---------------------------
 * mat[(rows[t]-row0)*kpad + hpos[cols[t]]] = 1 for every tuple t whose left id
 * has degree > delta2 and whose right id is heavy; mat is zeroed first. */
int mmj_build_operand(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t delta2,
                      const int32_t* hpos, uint8_t* mat, int64_t row0, int64_t nrows, int64_t kpad, void* stream);
/* Same, z-pair form for MMJ_MODE_BITMAP_PAIR (nrows a multiple of 32; mat has
 * nrows/2 rows): z = row0 + 32G + k + 8j (k < 8, j < 4) lands in row
 * 16G + 2k + j/2 with weight 1 (j even) or 128 (j odd). */
int mmj_build_operand_pairs(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg,
                            int64_t delta2, const int32_t* hpos, uint8_t* mat, int64_t row0, int64_t nrows,
                            int64_t kpad, void* stream);

/* Heavy-y bit rows of S_h (k x wpr uint32, zeroed first): bit z of row
 * hpos[cols[t]] for every tuple t = (z = rows[t], y = cols[t]) with
 * left_deg[z] > delta2 and heavy y; M2 of joinproject.py:119-143 at one bit
 * per cell, the operand of mmj_merge_emit / mmj_tile_merge has_heavy == 2. */
int mmj_build_heavy_rows(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg,
                         int64_t delta2, const int32_t* hpos, uint32_t* heavy_rows, int64_t k, int64_t wpr,
                         void* stream);
/* stats[0] = #heavy left ids (left_deg > delta2, over dom ids), stats[1] =
 * #tuples with a heavy left id and a heavy y: the mean heavy-y count of a
 * heavy row, which picks the projection's heavy form (engine.py) */
int mmj_heavy_row_stats(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t dom,
                        int64_t delta2, const int32_t* hpos, int64_t* stats, void* stream);

/* ---- light-z CSR of S for pass 3: joinproject.py:195-203 --------------------
 * lz_ptr[dom_y+1]/lz_idx: S.rev(y) restricted to z with deg_S(z) <= delta2.
 * flag_ws: n bytes; pos_ws: n+1 int32. */
int mmj_light_z_csr(const int32_t* rev_ptr, const int32_t* rev_idx, int64_t n, int64_t dom_y,
                    const int32_t* left_deg, int64_t delta2, uint8_t* flag_ws, int32_t* pos_ws, int32_t* lz_ptr,
                    int32_t* lz_idx, void* ws, void* stream);

/* ---- light passes: joinproject.py:183-203 ----------------------------------
 * Tuples t0 .. t0+ntup-1 of R in forward (x-sorted) order each expand one
 * list of S partners (S.rev(y) if y light or x light, else the light-z list).
 * hpos == NULL selects the FULL_JOIN strategy (every y light).
 * mmj_light_lengths writes len[ntup] and offs[ntup+1] (exclusive scan; offs[ntup]
 * is the light intermediate size).  mmj_light_expand sets bit (x-x0, z) of a
 * bitmap (mode 0, ld in words) or adds 1 to count cell (x-x0, z) (mode 1, ld in
 * int32; mode 2, ld in uint16 elements, every count < 65536).  min_deg > 1 (SSJ threshold c) skips rows of sets smaller than c
 * and light-z lists when delta2 < c; upper_only skips witnesses with z <= x. */
int mmj_light_lengths(const int32_t* fwd_row, const int32_t* fwd_idx, int64_t t0, int64_t ntup,
                      const int32_t* rdeg_x, int64_t delta2, const int32_t* hpos, const int32_t* s_rev_ptr,
                      const int32_t* s_rev_idx, const int32_t* lz_ptr, const int32_t* lz_idx, int64_t min_deg,
                      int upper_only, int32_t* len, int64_t* offs, void* ws, void* stream);
int mmj_light_expand(const int32_t* fwd_row, const int32_t* fwd_idx, int64_t t0, int64_t ntup,
                     const int32_t* rdeg_x, int64_t delta2, const int32_t* hpos, const int32_t* s_rev_ptr,
                     const int32_t* s_rev_idx, const int32_t* lz_ptr, const int32_t* lz_idx, int64_t min_deg,
                     int upper_only, const int64_t* offs, int64_t total_hint, int mode, int64_t x0, void* out,
                     int64_t ld, void* stream);

/* ---- heavy contraction on tcgen05: joinproject.py:208-216, core.py:95-123,
 *      _kernel_cy.pyx:42-47 ------------------------------------------------
 * A: a_rows x kpad uint8 (K-major), B: b_rows x kpad uint8 (K-major, one row
 * per output column).  Rows [m_begin, m_begin+m_rows) of A times the K window
 * [k_off, k_off+k_len) (multiples of 128) -> out rows 0..m_rows-1:
 *   MMJ_MODE_BITMAP : uint32 words, ld_out words per row (multiple of 8 and
 *                     >= ceil(b_rows/256)*8); bit j%32 of word j/32 = (C!=0)
 *   MMJ_MODE_COUNT32: int32, ld_out per row (multiple of 4)
 *   MMJ_MODE_ACC64  : int64, out[i][j] += C[i][j] << shift
 * nnz (optional) accumulates the number of nonzero product cells. */
int mmj_heavy_mma(const uint8_t* a, int64_t a_rows, const uint8_t* b, int64_t b_rows, int64_t kpad, int64_t k_off,
                  int64_t k_len, int64_t m_begin, int64_t m_rows, int mode, int shift, void* out, int64_t ld_out,
                  unsigned long long* nnz, int max_ctas, void* stream);

/* digit plane of an int64 matrix for exact multiply_counts: dst[r][c] =
 * (src >> 8*digit) & 255 with src = A (rows x cols) or, if transpose, the
 * transpose of a (cols x rows) source; dst pitch kpad, zero padded. */
int mmj_digit_plane(const int64_t* src, int64_t rows, int64_t cols, int transpose, int digit, uint8_t* dst,
                    int64_t kpad, void* stream);

/* ---- light passes merged into the bitmap + emission (projection, no
 *      counts): joinproject.py:183-203 + 220-225 ------------------------------
 * Chunk bitmap [x0, x0+rows) x [0, dom_z): rows x wpr words, wpr a multiple
 * of 32 (rows start on 1024-cell segments).  mmj_tile_merge runs one CTA per
 * tile (mmj_tile_count(rows, wpr) tiles of <= 65536 cells): the heavy part
 * is staged in shared memory -- has_heavy 0: zeros; 1: the chunk's heavy
 * bitmap already in `bitmap` (the tcgen05 product's output); 2: computed by
 * the tile from the heavy-y bit rows `heavy_rows` (mmj_build_heavy_rows) as
 * OR over the heavy y of each heavy row x, popcount added to *heavy_pairs
 * -- then every light witness of
 * the tile is OR-ed in (shared-memory atomics), the merged tile is written
 * back and segcnt[rows*wpr/32] receives each 32-word segment's popcount;
 * *witnesses accumulates the light intermediate size.  After an exclusive
 * scan of segcnt (mmj_exclusive_scan_i32 -> seg_off), mmj_emit_codes writes
 * the chunk's sorted codes x*dom_z + z to codes[0 .. seg_off[nseg]). */
int64_t mmj_tile_count(int64_t rows, int64_t wpr);
int mmj_tile_merge(uint32_t* bitmap, int has_heavy, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z,
                   const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t delta2,
                   const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr,
                   const int32_t* lz_idx, const uint32_t* heavy_rows, unsigned long long* heavy_pairs, int32_t* segcnt,
                   unsigned long long* witnesses, void* stream);
int mmj_emit_codes(const uint32_t* bitmap, const int64_t* seg_off, int64_t rows, int64_t wpr, int64_t x0,
                   int64_t dom_z, int64_t* codes, void* stream);
/* The same three steps fused into one kernel (no merged-bitmap write-back,
 * no segment-count array): tiles taken in ticket order merge their light
 * witnesses, scan their segments and find their output offset by a
 * decoupled look-back over per-tile status words, then emit.  codes must hold
 * the chunk's output (rows*dom_z is always enough); *total receives its size.
 * ws: caller-owned workspace of mmj_merge_emit_workspace_size(rows, wpr)
 * bytes (reset by the call, on `stream`).  fwd_ptr == NULL: no light merge
 * (the bitmap is complete; e.g. the star path, whose light part is OR-ed in
 * by mmj_star_light): segment scan + look-back + emission only.
 * has_heavy as for mmj_tile_merge; with has_heavy == 2 `bitmap` is the
 * heavy-y bit rows (k x wpr) and no chunk bitmap exists in HBM at all. */
size_t mmj_merge_emit_workspace_size(int64_t rows, int64_t wpr);
int mmj_merge_emit(const uint32_t* bitmap, int has_heavy, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z,
                   const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t delta2,
                   const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr,
                   const int32_t* lz_idx, const int32_t* split_full, const int32_t* split_lz,
                   unsigned long long* witnesses, unsigned long long* heavy_pairs, int64_t* codes, int64_t* total,
                   void* ws, size_t ws_bytes, void* stream);
/* Column blocks per row of the fused kernel's tiles, and the optional list
 * split table it reads instead of bisecting every long list per tile:
 * split[y*(ncb+1)+j] = position in idx of list y's first entry >= the j-th
 * block's first column (dom_y*(ncb+1) int32; NULL split pointers = bisect). */
int mmj_merge_emit_col_blocks(int64_t wpr);
/* profiling aid: per-tile phase timestamps of mmj_merge_emit (8 x uint64 per
 * tile, %globaltimer ns; recorded only by -DMMJ_DEBUG_TIMING builds) */
void mmj_debug_timing_buffer(unsigned long long* buf);
int mmj_list_splits(const int32_t* ptr, const int32_t* idx, int64_t dom_y, int64_t wpr, int32_t* split,
                    void* stream);

/* ---- merge / emission: joinproject.py:220-225 -------------------------------
 * Bitmap chunk of nwords words (wpr words per row, row r <-> x = x0 + r):
 * segment popcounts + exclusive scan (seg_off[nseg+1], seg_off[nseg] = size),
 * then sorted distinct codes x*dom_z + z. */
int64_t mmj_bitmap_segment_count(int64_t nwords);
int mmj_bitmap_segments(const uint32_t* bm, int64_t nwords, int32_t* segcnt, int64_t* seg_off, void* ws,
                        void* stream);
int mmj_bitmap_emit(const uint32_t* bm, int64_t nwords, int64_t wpr, const int64_t* seg_off, int64_t x0,
                    int64_t dom_z, int64_t* codes, void* stream);
/* Count chunk (nrows x ld cells, int32 or uint16 by cell_bytes = 4 / 2, ncols
 * valid columns; uint16 when every count is < 65536): cells with count >=
 * max(min_count, row_min[x0+row]) (row_min may be NULL) -> codes + int32
 * counts.  cell_filter: 0 every cell, 1 col > x0+row (SSJ's a < b,
 * apps.py:57-62), 2 col != x0+row (SCJ's a != b, apps.py:297-304).  ld must be a multiple of 1024
 * (segments of 1024 cells never straddle rows); with cell_filter 1, segments
 * at or below the diagonal are not read. */
int64_t mmj_count_segment_count(int64_t ncell);
int mmj_count_segments(const void* cnt, int cell_bytes, int64_t nrows, int64_t ld, int64_t ncols, int64_t x0,
                       int32_t min_count, const int32_t* row_min, int cell_filter, int32_t* segcnt, int64_t* seg_off,
                       void* ws, void* stream);
int mmj_count_emit(const void* cnt, int cell_bytes, int64_t nrows, int64_t ld, int64_t ncols, int64_t x0,
                   int64_t dom_z, int32_t min_count, const int32_t* row_min, int cell_filter, const int64_t* seg_off,
                   int64_t* codes, int32_t* counts, void* stream);

/* ---- star join-project, k = 2..4: joinproject.py:281-378 -------------------
 * Output as a two-path over composite rows (x1..x_{k-1}) x column x_k.
 * dims / rev_ptr / rev_idx / heavy are HOST arrays of k device pointers or
 * sizes.  mmj_star_split: y heavy iff prod_j deg_j(y) > threshold -> hpos
 * (rank or -1) and the compacted light-y list (prod > 0); flag/scan buffers
 * hold dom_y (+1) entries.  mmj_star_operand: A[r] = AND_{j<k-1} H_j[x_j] for
 * the composite rows r of x1 in [x1_begin, ..) (kpad % 16 == 0).
 * mmj_star_light: every light witness with x1 in [x1_begin, x1_end) is OR-ed
 * (mode 0, ld words) or counted (mode 1, ld int32) into the chunk matrix,
 * balanced by witness index (needs mmj_star_light_workspace_bytes(n_light)). */
int mmj_star_split(int k, const int32_t* const* rev_ptr, int64_t dom_y, double threshold, uint8_t* heavy_flag,
                   uint8_t* light_flag, int32_t* heavy_scan, int32_t* light_scan, int32_t* hpos, int32_t* light_y,
                   void* ws, void* stream);
int mmj_star_operand(int k, const int64_t* dims, const uint8_t* const* heavy, int64_t kpad, int64_t x1_begin,
                     int64_t rows, uint8_t* A, void* stream);
size_t mmj_star_light_workspace_bytes(int64_t n_light);
int mmj_star_light(int k, const int64_t* dims, const int32_t* const* rev_ptr, const int32_t* const* rev_idx,
                   const int32_t* light_y, int64_t n_light, int64_t x1_begin, int64_t x1_end, int mode, void* out,
                   int64_t ld, unsigned long long* witnesses, void* ws, void* stream);

/* ---- batched boolean set intersection: apps.py:314-351 ----------------------
 * Heavy y (hpos >= 0, from mmj_heavy_y_positions) -> one record per left id
 * (mmj_bsi_records, one pass over the forward CSR): `words` bitset words
 * (4, 8, 16 or 32) with bit hpos[y] for each heavy y, then the base and the
 * length of the id's light list, whose y are compacted in place into ovf at
 * the id's own CSR offset (ovf: n int32); rec holds dom_left records of
 * mmj_bsi_record_words(words) uint32 (64-byte multiples).  mmj_bsi_answer
 * resolves raw query ids per side through a direct-address table (table !=
 * NULL), else the sorted raw left values (sorted/order; both NULL = queries
 * are dense ids already), and writes ans[q] = 1 (intersect), 0 (disjoint)
 * or -1 (id unknown to the unreduced relation = None). */
/* histogram of max(rdeg[y], sdeg[y]) > 0: 64 log2 bins (log2mode) or nbins
 * (<= 1024) linear bins over [lo, hi); picks the heavy-y threshold on the device */
int mmj_bsi_degree_histogram(const int32_t* rdeg, const int32_t* sdeg, int64_t dom_y, int64_t lo, int64_t hi,
                             int nbins, int log2mode, int32_t* hist, void* stream);
int mmj_bsi_record_words(int words);
int mmj_bsi_records(const int32_t* fwd_ptr, const int32_t* fwd_idx, int64_t dom_left, const int32_t* hpos, int words,
                    uint32_t* rec, int32_t* ovf, void* stream);
int mmj_bsi_answer(const int64_t* qa, const int64_t* qb, int64_t nq, const int64_t* r_sorted, const int32_t* r_order,
                   int64_t r_n, const int32_t* r_table, int64_t r_min, int64_t r_range, const int64_t* s_sorted,
                   const int32_t* s_order, int64_t s_n, const int32_t* s_table, int64_t s_min, int64_t s_range,
                   const uint32_t* r_rec, const int32_t* r_ovf, const uint32_t* s_rec, const int32_t* s_ovf,
                   int words, int8_t* ans, void* stream);
/* the same answers without any index build: the two queried ids' forward
 * lists (fwd_ptr / fwd_idx int32, each list sorted by the shared y id) are
 * intersected directly (a warp per 32 queries, lists loaded coalesced into
 * registers, shuffle binary search); id maps as for mmj_bsi_answer.  The engine
 * takes this form when the lists are short (mean length <= 64), where a
 * bitset record moves as many DRAM sectors as the list it summarises. */
int mmj_bsi_answer_lists(const int64_t* qa, const int64_t* qb, int64_t nq, const int64_t* r_sorted,
                         const int32_t* r_order, int64_t r_n, const int32_t* r_table, int64_t r_min, int64_t r_range,
                         const int64_t* s_sorted, const int32_t* s_order, int64_t s_n, const int32_t* s_table,
                         int64_t s_min, int64_t s_range, const int32_t* r_fwd_ptr, const int32_t* r_fwd_idx,
                         const int32_t* s_fwd_ptr, const int32_t* s_fwd_idx, int8_t* ans, void* stream);
/* direct-address id map for dense raw id ranges: table[range] = dense id of
 * raw value vmin + i, -1 where absent (one load per query instead of a
 * binary search; range = max - min + 1 < 2^31) */
int mmj_bsi_direct_table(const int64_t* sorted, const int32_t* order, int64_t n, int64_t vmin, int64_t range,
                         int32_t* table, void* stream);
/* span table for dense raw id ranges: table[range] of 8-byte entries, low
 * word = (forward-list offset << len_bits) | min(list length, 2^len_bits - 1)
 * of raw value vmin + i (0xFFFFFFFF where absent; needs n_tuples <
 * 2^(32 - len_bits) - 1), high word = the id's heavy-y signature: bit hpos[y]
 * for each of its y with 0 <= hpos[y] < 32 (hpos over the shared y space, -1 =
 * not heavy; hpos NULL = no signatures).  mmj_bsi_answer_spans resolves each
 * query id with that one load; two ids with a common signature bit share a
 * heavy y and are answered at once (the heavy part of the reference's
 * product, joinproject.py:208-216, on the queried cells only), the others
 * intersect their forward lists (a saturated length falls back to a binary
 * search of the offset in fwd_ptr): the left_ids.get() probes and set
 * intersection of apps.py:321-350, same answers as mmj_bsi_answer_lists */
int mmj_bsi_span_table(const int64_t* sorted, const int32_t* order, int64_t n, int64_t vmin, int64_t range,
                       const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* hpos, int64_t n_tuples,
                       int len_bits, uint64_t* table, void* stream);
int mmj_bsi_answer_spans(const int64_t* qa, const int64_t* qb, int64_t nq, const uint64_t* r_span, int64_t r_min,
                         int64_t r_range, int r_len_bits, const int32_t* r_fwd_ptr, int64_t r_dom,
                         const int32_t* r_fwd_idx, const uint64_t* s_span, int64_t s_min, int64_t s_range,
                         int s_len_bits, const int32_t* s_fwd_ptr, int64_t s_dom, const int32_t* s_fwd_idx,
                         int8_t* ans, void* stream);


/* ---- device ingest: relation.py:37-69, 119-140, 148-186 ----
 * Raw int64 pairs (n x 2, row-major) -> deduplicated, dictionary-encoded,
 * semi-join-reduced relations and their int32 CSR, all in HBM.  Every call
 * takes a caller workspace of >= mmj_ingest_workspace_bytes(n) bytes; counts
 * come back in device int64 scalars (*_out), for the caller to read before
 * sizing the next step.  Ids match the reference's bit for bit. */
size_t mmj_ingest_workspace_bytes(int64_t n);
/* keep-first dedup of (left, right) tuples in input order (dict.fromkeys, relation.py:53) */
int mmj_ingest_dedup(const int64_t* pairs, int64_t n, int64_t* out, int64_t* n_out, void* ws, size_t ws_bytes,
                     void* stream);
/* first-seen dense ids of vals[i*stride] (relation.py:56-66): ids[n] int32, dict[ndict] int64 */
int mmj_ingest_first_seen(const int64_t* vals, int64_t stride, int64_t n, int32_t* ids, int64_t* dict,
                          int64_t* ndict, void* ws, size_t ws_bytes, void* stream);
/* ascending distinct values of vals[i*stride] */
int mmj_ingest_distinct(const int64_t* vals, int64_t stride, int64_t n, int64_t* out, int64_t* n_out, void* ws,
                        size_t ws_bytes, void* stream);
/* sorted-unique a intersect sorted-unique b (relation.py:121-122) */
int mmj_ingest_intersect(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t* out, int64_t* n_out,
                         void* ws, size_t ws_bytes, void* stream);
/* vals (ascending) in repr() order (relation.py:123): out[j] = vals[perm[j]], rank[perm[j]] = j */
int mmj_ingest_repr_order(const int64_t* vals, int64_t n, int64_t* out, int32_t* rank, void* ws, size_t ws_bytes,
                          void* stream);
/* ids[i] = id_of_sorted[p] where sorted[p] == q[i*stride] (p if id_of_sorted is NULL), -1 if absent */
int mmj_ingest_lookup(const int64_t* sorted, const int32_t* id_of_sorted, int64_t nd, const int64_t* q,
                      int64_t stride, int64_t nq, int32_t* ids, void* stream);
/* keep tuples with rid >= 0 in input order (relation.py:128-130): left raw values + right ids */
int mmj_ingest_filter(const int64_t* pairs, const int32_t* rid, int64_t n, int64_t* left_out, int32_t* rid_out,
                      int64_t* n_out, void* ws, size_t ws_bytes, void* stream);
/* CSR of (rows, cols) with each row's cols ascending (relation.py:148-154): ptr[dom_rows+1],
 * idx[n], row_of[n] (may be NULL), deg[dom_rows] (may be NULL); all int32 */
/* ascending vals with their positions: sorted[j] = vals[order[j]] (stable) */
int mmj_ingest_sort_ids(const int64_t* vals, int64_t n, int64_t* sorted, int32_t* order, void* ws, size_t ws_bytes,
                        void* stream);
/* out[i] = map[idx[i]] */
int mmj_ingest_remap(const int32_t* idx, int64_t n, const int32_t* map, int32_t* out, void* stream);
/* out[i] = src[idx[i]] for 4- or 8-byte elements */
int mmj_ingest_gather(const void* src, int elem_bytes, const int32_t* idx, int64_t n, void* out, void* stream);
/* cnt[v] = #{i : idx[i] == v}, v < dom (cnt zeroed first) */
int mmj_ingest_histogram(const int32_t* idx, int64_t n, int64_t dom, int32_t* cnt, void* stream);
/* Row compaction before an SSJ / thresholded count join (apps.py:57-62: a set
 * with fewer than c elements reaches no overlap >= c, so its row and column of
 * the count matrix can be dropped).  Keeps the rows x with left_deg[x] >=
 * min_deg, renumbered 0..dom'-1 in id order (new_id[dom], -1 = dropped;
 * orig[dom'] its inverse), and writes the compacted relation's CSR in both
 * directions without a sort (kept entries keep their order; offsets are the
 * keep-flag scans at the old offsets): fwd_ptr_out[dom'+1], fwd_idx_out /
 * fwd_row_out [n'], left_deg_out[dom'], rev_ptr_out[dom_y+1], rev_idx_out[n'],
 * right_deg_out[dom_y].  Caller sizes the outputs for dom / n.  sizes[0] = dom',
 * sizes[1] = n' (device int64).  Workspace: mmj_ingest_workspace_bytes(max(n,
 * dom, dom_y)). */
int mmj_compact_rows(const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* fwd_row,
                     const int32_t* rev_ptr, const int32_t* rev_idx, const int32_t* left_deg, int64_t n, int64_t dom,
                     int64_t dom_y, int64_t min_deg, int32_t* new_id, int32_t* orig, int32_t* fwd_ptr_out,
                     int32_t* fwd_idx_out, int32_t* fwd_row_out, int32_t* left_deg_out, int32_t* rev_ptr_out,
                     int32_t* rev_idx_out, int32_t* right_deg_out, int64_t* sizes, void* ws, size_t ws_bytes,
                     void* stream);
/* out[i] = orig_l[in[i] / dom_c] * dom_out + orig_r[in[i] % dom_c] (in == out allowed):
 * compact codes back to the caller's dense-id codes; ascending stays ascending */
int mmj_decode_compact_codes(const int64_t* in, int64_t n, int64_t dom_c, const int32_t* orig_l,
                             const int32_t* orig_r, int64_t dom_out, int64_t* out, void* stream);
/* a[i] = codes[i] / dom, b[i] = codes[i] % dom (codes >= 0): the result pairs
 * of SSJ / SCJ as two arrays (apps.py:57-62 unpacks codes the same way) */
int mmj_split_codes(const int64_t* codes, int64_t n, int64_t dom, int64_t* a, int64_t* b, void* stream);
int mmj_ingest_csr(const int32_t* rows, const int32_t* cols, int64_t n, int64_t dom_rows, int64_t dom_cols,
                   int32_t* ptr, int32_t* idx, int32_t* row_of, int32_t* deg, void* ws, size_t ws_bytes,
                   void* stream);

/* ---- result text formats: cli.py:129-136, 154-161, 180-182, 205-206 -----
 * Lines "v0 v1 [v2 [v3]] [count]" of raw dictionary strings, sorted as
 * Python sorts the strings, joined by '\n'.  Columns: ncode code columns
 * (codes mixed radix over dims, as OutputSet.tuples) plus, when counts !=
 * NULL, the count column.  Per column (host arrays of device pointers):
 * rank[c][v] = position of value v's string among the column's sorted
 * strings (nrank[c] entries; count column indexed by the count), soff[c]
 * (nrank[c] + 1 int64 offsets) and blob[c] (UTF-8 bytes).
 *   mmj_format_keys     key[t] = mixed-radix rank tuple (sort it: the line
 *                       order); *bad = 1 if a value is outside its table
 *   mmj_format_lengths  len[p] of line p (tuple order[p], or p if order is
 *                       NULL), separators and the newline included
 *   mmj_format_write    the bytes, line p at line_off[p] (exclusive scan of
 *                       the lengths, mmj_exclusive_scan_i32) */
int mmj_format_keys(const int64_t* codes, const int64_t* counts, int64_t n, int ncode, const int64_t* dims,
                    const int32_t* const* rank, const int64_t* nrank, int64_t* key, int* bad, void* stream);
int mmj_format_lengths(const int64_t* codes, const int64_t* counts, const int32_t* order, int64_t n, int ncode,
                       const int64_t* dims, const int64_t* const* soff, int32_t* len, void* stream);
int mmj_format_write(const int64_t* codes, const int64_t* counts, const int32_t* order, int64_t n, int ncode,
                     const int64_t* dims, const int64_t* const* soff, const uint8_t* const* blob,
                     const int64_t* line_off, uint8_t* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MMJOIN_B200_H */
