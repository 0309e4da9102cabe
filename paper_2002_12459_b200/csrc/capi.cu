// extern "C" boundary of libmmjoin_b200.so (declared in include/mmjoin_b200.h).
#include "../../include/mmjoin_b200.h"
#include "mmj_common.cuh"

namespace mmj {
// format.cu (FmtArgs: mmj_common.cuh)
int fmt_keys(const FmtArgs&, int64_t*, int*, cudaStream_t);
int fmt_lengths(const FmtArgs&, int32_t*, cudaStream_t);
int fmt_write(const FmtArgs&, const int64_t*, uint8_t*, cudaStream_t);
// twopath.cu
int heavy_y_positions(const int32_t*, const int32_t*, int64_t, int64_t, uint8_t*, int32_t*, int32_t*, void*,
                      cudaStream_t);
int build_operand(const int32_t*, const int32_t*, int64_t, const int32_t*, int64_t, const int32_t*, uint8_t*, int64_t,
                  int64_t, int64_t, cudaStream_t);
int build_heavy_rows(const int32_t*, const int32_t*, int64_t, const int32_t*, int64_t, const int32_t*, uint32_t*,
                     int64_t, int64_t, cudaStream_t);
int heavy_row_stats(const int32_t*, const int32_t*, int64_t, const int32_t*, int64_t, int64_t, const int32_t*,
                    int64_t*, cudaStream_t);
int build_operand_pairs(const int32_t*, const int32_t*, int64_t, const int32_t*, int64_t, const int32_t*, uint8_t*,
                        int64_t, int64_t, int64_t, cudaStream_t);
int light_z_csr(const int32_t*, const int32_t*, int64_t, int64_t, const int32_t*, int64_t, uint8_t*, int32_t*,
                int32_t*, int32_t*, void*, cudaStream_t);
int light_lengths(const int32_t*, const int32_t*, int64_t, int64_t, const int32_t*, int64_t, const int32_t*,
                  const int32_t*, const int32_t*, const int32_t*, const int32_t*, int64_t, int, int32_t*, int64_t*, void*,
                  cudaStream_t);
int light_expand(const int32_t*, const int32_t*, int64_t, int64_t, const int32_t*, int64_t, const int32_t*,
                 const int32_t*, const int32_t*, const int32_t*, const int32_t*, int64_t, int, const int64_t*, int64_t,
                 int, int64_t, void*, int64_t, cudaStream_t);
int64_t bitmap_nseg(int64_t);
int64_t count_nseg(int64_t);
int bitmap_segments(const uint32_t*, int64_t, int32_t*, int64_t*, void*, cudaStream_t);
int bitmap_emit(const uint32_t*, int64_t, int64_t, const int64_t*, int64_t, int64_t, int64_t*, cudaStream_t);
int count_segments(const void*, int, int64_t, int64_t, int64_t, int64_t, int32_t, const int32_t*, int, int32_t*,
                   int64_t*, void*, cudaStream_t);
int count_emit(const void*, int, int64_t, int64_t, int64_t, int64_t, int64_t, int32_t, const int32_t*, int,
               const int64_t*, int64_t*, int32_t*, cudaStream_t);
int64_t row_emit_tiles(int64_t, int64_t);
int tile_merge(uint32_t*, int, int64_t, int64_t, int64_t, int64_t, const int32_t*, const int32_t*, const int32_t*,
               int64_t, const int32_t*, const int32_t*, const int32_t*, const int32_t*, const int32_t*,
               const uint32_t*, unsigned long long*, int32_t*, unsigned long long*, cudaStream_t);
int emit_codes(const uint32_t*, const int64_t*, int64_t, int64_t, int64_t, int64_t, int64_t*, cudaStream_t);
size_t merge_emit_ws_bytes(int64_t, int64_t);
int merge_emit(const uint32_t*, int, int64_t, int64_t, int64_t, int64_t, const int32_t*, const int32_t*, const int32_t*,
               int64_t, const int32_t*, const int32_t*, const int32_t*, const int32_t*, const int32_t*,
               const int32_t*, const int32_t*, unsigned long long*, unsigned long long*, int64_t*, int64_t*, void*,
               size_t,
               cudaStream_t);
int merge_emit_col_blocks(int64_t);
extern unsigned long long* tdbg_buffer;
int list_splits(const int32_t*, const int32_t*, int64_t, int64_t, int32_t*, cudaStream_t);
int bsi_record_words(int);
int bsi_records(const int32_t*, const int32_t*, int64_t, const int32_t*, int, uint32_t*, int32_t*, cudaStream_t);
int bsi_answer(const int64_t*, const int64_t*, int64_t, const int64_t*, const int32_t*, int64_t, const int32_t*, int64_t,
               int64_t, const int64_t*, const int32_t*, int64_t, const int32_t*, int64_t, int64_t, const uint32_t*,
               const int32_t*, const uint32_t*, const int32_t*, int, int8_t*, cudaStream_t);
int bsi_direct_table(const int64_t*, const int32_t*, int64_t, int64_t, int64_t, int32_t*, cudaStream_t);
int bsi_span_table(const int64_t*, const int32_t*, int64_t, int64_t, int64_t, const int32_t*, const int32_t*,
                   const int32_t*, int64_t, int, uint2*, cudaStream_t);
int bsi_answer_spans(const int64_t*, const int64_t*, int64_t, const uint2*, int64_t, int64_t, int, const int32_t*,
                     int64_t, const int32_t*, const uint2*, int64_t, int64_t, int, const int32_t*, int64_t,
                     const int32_t*, int8_t*, cudaStream_t);
int bsi_answer_lists(const int64_t*, const int64_t*, int64_t, const int64_t*, const int32_t*, int64_t, const int32_t*,
                     int64_t, int64_t, const int64_t*, const int32_t*, int64_t, const int32_t*, int64_t, int64_t,
                     const int32_t*, const int32_t*, const int32_t*, const int32_t*, int8_t*, cudaStream_t);
int star_split(int, const int32_t* const*, int64_t, double, uint8_t*, uint8_t*, int32_t*, int32_t*, int32_t*, int32_t*,
               void*, cudaStream_t);
int star_operand(int, const int64_t*, const uint8_t* const*, int64_t, int64_t, int64_t, uint8_t*, cudaStream_t);
size_t star_light_ws_bytes(int64_t);
int star_light(int, const int64_t*, const int32_t* const*, const int32_t* const*, const int32_t*, int64_t, int64_t,
               int64_t, int, void*, int64_t, unsigned long long*, void*, cudaStream_t);
int bsi_degree_histogram(const int32_t*, const int32_t*, int64_t, int64_t, int64_t, int, int, int32_t*, cudaStream_t);
namespace mma {
int launch_heavy_mma(const uint8_t*, int64_t, const uint8_t*, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t,
                     int, int, void*, int64_t, unsigned long long*, int, cudaStream_t);
}

namespace {
__global__ void k_digit_plane(const int64_t* __restrict__ src, int64_t rows, int64_t cols, int transpose, int digit,
                              uint8_t* __restrict__ dst, int64_t kpad) {
  const int64_t total = rows * kpad;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / kpad, c = i - r * kpad;
    uint8_t v = 0;
    if (c < cols) {
      const int64_t x = transpose ? src[c * rows + r] : src[r * cols + c];
      v = (uint8_t)((x >> (8 * digit)) & 255);
    }
    dst[i] = v;
  }
}
}  // namespace
}  // namespace mmj

#define ST(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

int mmj_abi_version(void) { return 1; }

const char* mmj_last_error(void) { return mmj::last_error(); }

int mmj_set_device(int device) { return mmj::cuda_status(cudaSetDevice(device), "cudaSetDevice"); }

int mmj_sm_count(void) { return mmj::sm_count(); }

long long mmj_launch_count(void) { return mmj::launch_count(); }

size_t mmj_scan_workspace_bytes(int64_t n) { return mmj::scan_ws_bytes(n); }

int mmj_exclusive_scan_i32(const int32_t* in, int64_t* out, int64_t n, void* ws, void* stream) {
  return mmj::scan_i32_i64(in, out, n, ws, ST(stream));
}

int mmj_code_checksum(const int64_t* codes, int64_t n, int64_t base, unsigned long long* out, void* stream) {
  return mmj::code_checksum(codes, n, base, out, ST(stream));
}

int mmj_heavy_y_positions(const int32_t* rdeg_y, const int32_t* sdeg_y, int64_t dom_y, int64_t delta1,
                          uint8_t* flag_ws, int32_t* scan_out, int32_t* hpos, void* ws, void* stream) {
  if (delta1 < 1) {
    mmj::set_error("thresholds must be >= 1");
    return MMJ_ERR_ARG;
  }
  return mmj::heavy_y_positions(rdeg_y, sdeg_y, dom_y, delta1, flag_ws, scan_out, hpos, ws, ST(stream));
}

int mmj_build_operand(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t delta2,
                      const int32_t* hpos, uint8_t* mat, int64_t row0, int64_t nrows, int64_t kpad, void* stream) {
  return mmj::build_operand(rows, cols, n, left_deg, delta2, hpos, mat, row0, nrows, kpad, ST(stream));
}

int mmj_build_operand_pairs(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg,
                            int64_t delta2, const int32_t* hpos, uint8_t* mat, int64_t row0, int64_t nrows,
                            int64_t kpad, void* stream) {
  return mmj::build_operand_pairs(rows, cols, n, left_deg, delta2, hpos, mat, row0, nrows, kpad, ST(stream));
}

int mmj_heavy_row_stats(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t dom,
                        int64_t delta2, const int32_t* hpos, int64_t* stats, void* stream) {
  return mmj::heavy_row_stats(rows, cols, n, left_deg, dom, delta2, hpos, stats, ST(stream));
}

int mmj_build_heavy_rows(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg,
                         int64_t delta2, const int32_t* hpos, uint32_t* heavy_rows, int64_t k, int64_t wpr,
                         void* stream) {
  return mmj::build_heavy_rows(rows, cols, n, left_deg, delta2, hpos, heavy_rows, k, wpr, ST(stream));
}

int mmj_light_z_csr(const int32_t* rev_ptr, const int32_t* rev_idx, int64_t n, int64_t dom_y,
                    const int32_t* left_deg, int64_t delta2, uint8_t* flag_ws, int32_t* pos_ws, int32_t* lz_ptr,
                    int32_t* lz_idx, void* ws, void* stream) {
  return mmj::light_z_csr(rev_ptr, rev_idx, n, dom_y, left_deg, delta2, flag_ws, pos_ws, lz_ptr, lz_idx, ws,
                          ST(stream));
}

int mmj_light_lengths(const int32_t* fwd_row, const int32_t* fwd_idx, int64_t t0, int64_t ntup,
                      const int32_t* rdeg_x, int64_t delta2, const int32_t* hpos, const int32_t* s_rev_ptr,
                      const int32_t* s_rev_idx, const int32_t* lz_ptr, const int32_t* lz_idx, int64_t min_deg,
                      int upper_only, int32_t* len, int64_t* offs, void* ws, void* stream) {
  return mmj::light_lengths(fwd_row, fwd_idx, t0, ntup, rdeg_x, delta2, hpos, s_rev_ptr, s_rev_idx, lz_ptr, lz_idx,
                            min_deg, upper_only, len, offs, ws, ST(stream));
}

int mmj_light_expand(const int32_t* fwd_row, const int32_t* fwd_idx, int64_t t0, int64_t ntup,
                     const int32_t* rdeg_x, int64_t delta2, const int32_t* hpos, const int32_t* s_rev_ptr,
                     const int32_t* s_rev_idx, const int32_t* lz_ptr, const int32_t* lz_idx, int64_t min_deg,
                     int upper_only, const int64_t* offs, int64_t total_hint, int mode, int64_t x0, void* out,
                     int64_t ld, void* stream) {
  if (mode < 0 || mode > 2) {
    mmj::set_error("light_expand: mode must be 0 (bitmap), 1 (int32 counts) or 2 (uint16 counts)");
    return MMJ_ERR_ARG;
  }
  return mmj::light_expand(fwd_row, fwd_idx, t0, ntup, rdeg_x, delta2, hpos, s_rev_ptr, s_rev_idx, lz_ptr, lz_idx,
                           min_deg, upper_only, offs, total_hint, mode, x0, out, ld, ST(stream));
}

int mmj_heavy_mma(const uint8_t* a, int64_t a_rows, const uint8_t* b, int64_t b_rows, int64_t kpad, int64_t k_off,
                  int64_t k_len, int64_t m_begin, int64_t m_rows, int mode, int shift, void* out, int64_t ld_out,
                  unsigned long long* nnz, int max_ctas, void* stream) {
  const int base_mode = mode & ~MMJ_MODE_UPPER;
  const int upper = mode & MMJ_MODE_UPPER;
  if (base_mode < 0 || base_mode > MMJ_MODE_COUNT16 ||
      (upper && base_mode != MMJ_MODE_COUNT32 && base_mode != MMJ_MODE_COUNT16)) {
    mmj::set_error("heavy_mma: unknown mode %d (MMJ_MODE_UPPER combines with the count modes only)", mode);
    return MMJ_ERR_ARG;
  }
  return mmj::mma::launch_heavy_mma(a, a_rows, b, b_rows, kpad, k_off, k_len, m_begin, m_rows, mode, shift, out,
                                    ld_out, nnz, max_ctas, ST(stream));
}

int mmj_digit_plane(const int64_t* src, int64_t rows, int64_t cols, int transpose, int digit, uint8_t* dst,
                    int64_t kpad, void* stream) {
  if (digit < 0 || digit > 7 || kpad < cols) {
    mmj::set_error("digit_plane: bad digit/pitch");
    return MMJ_ERR_ARG;
  }
  const int64_t total = rows * kpad;
  if (total == 0) return MMJ_OK;
  int64_t g = mmj::ceil_div(total, 256);
  if (g > (int64_t)mmj::sm_count() * 32) g = (int64_t)mmj::sm_count() * 32;
  mmj::k_digit_plane<<<(unsigned)g, 256, 0, ST(stream)>>>(src, rows, cols, transpose, digit, dst, kpad);
  MMJ_CHECK_LAUNCH("k_digit_plane");
  return MMJ_OK;
}

int64_t mmj_tile_count(int64_t rows, int64_t wpr) { return mmj::row_emit_tiles(rows, wpr); }

int mmj_tile_merge(uint32_t* bitmap, int has_heavy, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z,
                   const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t delta2,
                   const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr,
                   const int32_t* lz_idx, const uint32_t* heavy_rows, unsigned long long* heavy_pairs, int32_t* segcnt,
                   unsigned long long* witnesses, void* stream) {
  return mmj::tile_merge(bitmap, has_heavy, x0, rows, wpr, dom_z, fwd_ptr, fwd_idx, rdeg_x, delta2, hpos, s_rev_ptr,
                         s_rev_idx, lz_ptr, lz_idx, heavy_rows, heavy_pairs, segcnt, witnesses, ST(stream));
}

size_t mmj_merge_emit_workspace_size(int64_t rows, int64_t wpr) { return mmj::merge_emit_ws_bytes(rows, wpr); }

int mmj_merge_emit(const uint32_t* bitmap, int has_heavy, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z,
                   const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t delta2,
                   const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr,
                   const int32_t* lz_idx, const int32_t* split_full, const int32_t* split_lz,
                   unsigned long long* witnesses, unsigned long long* heavy_pairs, int64_t* codes, int64_t* total,
                   void* ws, size_t ws_bytes, void* stream) {
  return mmj::merge_emit(bitmap, has_heavy, x0, rows, wpr, dom_z, fwd_ptr, fwd_idx, rdeg_x, delta2, hpos, s_rev_ptr,
                         s_rev_idx, lz_ptr, lz_idx, split_full, split_lz, witnesses, heavy_pairs, codes, total, ws,
                         ws_bytes, ST(stream));
}

int mmj_merge_emit_col_blocks(int64_t wpr) { return mmj::merge_emit_col_blocks(wpr); }

/* profiling aid: per-tile phase timestamps of mmj_merge_emit (8 x uint64 per
 * tile; recorded only by -DMMJ_DEBUG_TIMING builds); NULL switches it off */
void mmj_debug_timing_buffer(unsigned long long* buf) { mmj::tdbg_buffer = buf; }

int mmj_list_splits(const int32_t* ptr, const int32_t* idx, int64_t dom_y, int64_t wpr, int32_t* split,
                    void* stream) {
  return mmj::list_splits(ptr, idx, dom_y, wpr, split, ST(stream));
}

int mmj_emit_codes(const uint32_t* bitmap, const int64_t* seg_off, int64_t rows, int64_t wpr, int64_t x0,
                   int64_t dom_z, int64_t* codes, void* stream) {
  return mmj::emit_codes(bitmap, seg_off, rows, wpr, x0, dom_z, codes, ST(stream));
}

int mmj_bsi_degree_histogram(const int32_t* rdeg, const int32_t* sdeg, int64_t dom_y, int64_t lo, int64_t hi,
                             int nbins, int log2mode, int32_t* hist, void* stream) {
  return mmj::bsi_degree_histogram(rdeg, sdeg, dom_y, lo, hi, nbins, log2mode, hist, ST(stream));
}

int mmj_bsi_record_words(int words) { return mmj::bsi_record_words(words); }

int mmj_bsi_records(const int32_t* fwd_ptr, const int32_t* fwd_idx, int64_t dom_left, const int32_t* hpos, int words,
                    uint32_t* rec, int32_t* ovf, void* stream) {
  return mmj::bsi_records(fwd_ptr, fwd_idx, dom_left, hpos, words, rec, ovf, ST(stream));
}

int mmj_bsi_answer(const int64_t* qa, const int64_t* qb, int64_t nq, const int64_t* r_sorted, const int32_t* r_order,
                   int64_t r_n, const int32_t* r_table, int64_t r_min, int64_t r_range, const int64_t* s_sorted,
                   const int32_t* s_order, int64_t s_n, const int32_t* s_table, int64_t s_min, int64_t s_range,
                   const uint32_t* r_rec, const int32_t* r_ovf, const uint32_t* s_rec, const int32_t* s_ovf,
                   int words, int8_t* ans, void* stream) {
  return mmj::bsi_answer(qa, qb, nq, r_sorted, r_order, r_n, r_table, r_min, r_range, s_sorted, s_order, s_n, s_table,
                         s_min, s_range, r_rec, r_ovf, s_rec, s_ovf, words, ans, ST(stream));
}

int mmj_bsi_answer_lists(const int64_t* qa, const int64_t* qb, int64_t nq, const int64_t* r_sorted,
                         const int32_t* r_order, int64_t r_n, const int32_t* r_table, int64_t r_min, int64_t r_range,
                         const int64_t* s_sorted, const int32_t* s_order, int64_t s_n, const int32_t* s_table,
                         int64_t s_min, int64_t s_range, const int32_t* r_fwd_ptr, const int32_t* r_fwd_idx,
                         const int32_t* s_fwd_ptr, const int32_t* s_fwd_idx, int8_t* ans, void* stream) {
  return mmj::bsi_answer_lists(qa, qb, nq, r_sorted, r_order, r_n, r_table, r_min, r_range, s_sorted, s_order, s_n,
                               s_table, s_min, s_range, r_fwd_ptr, r_fwd_idx, s_fwd_ptr, s_fwd_idx, ans, ST(stream));
}

int mmj_bsi_span_table(const int64_t* sorted, const int32_t* order, int64_t n, int64_t vmin, int64_t range,
                       const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* hpos, int64_t n_tuples,
                       int len_bits, uint64_t* table, void* stream) {
  return mmj::bsi_span_table(sorted, order, n, vmin, range, fwd_ptr, fwd_idx, hpos, n_tuples, len_bits,
                             reinterpret_cast<uint2*>(table), ST(stream));
}

int mmj_bsi_answer_spans(const int64_t* qa, const int64_t* qb, int64_t nq, const uint64_t* r_span, int64_t r_min,
                         int64_t r_range, int r_len_bits, const int32_t* r_fwd_ptr, int64_t r_dom,
                         const int32_t* r_fwd_idx, const uint64_t* s_span, int64_t s_min, int64_t s_range,
                         int s_len_bits, const int32_t* s_fwd_ptr, int64_t s_dom, const int32_t* s_fwd_idx,
                         int8_t* ans, void* stream) {
  return mmj::bsi_answer_spans(qa, qb, nq, reinterpret_cast<const uint2*>(r_span), r_min, r_range, r_len_bits,
                               r_fwd_ptr, r_dom, r_fwd_idx, reinterpret_cast<const uint2*>(s_span), s_min, s_range,
                               s_len_bits, s_fwd_ptr, s_dom, s_fwd_idx, ans, ST(stream));
}

int mmj_bsi_direct_table(const int64_t* sorted, const int32_t* order, int64_t n, int64_t vmin, int64_t range,
                         int32_t* table, void* stream) {
  return mmj::bsi_direct_table(sorted, order, n, vmin, range, table, ST(stream));
}


int mmj_star_split(int k, const int32_t* const* rev_ptr, int64_t dom_y, double threshold, uint8_t* heavy_flag,
                   uint8_t* light_flag, int32_t* heavy_scan, int32_t* light_scan, int32_t* hpos, int32_t* light_y,
                   void* ws, void* stream) {
  return mmj::star_split(k, rev_ptr, dom_y, threshold, heavy_flag, light_flag, heavy_scan, light_scan, hpos, light_y,
                         ws, ST(stream));
}

int mmj_star_operand(int k, const int64_t* dims, const uint8_t* const* heavy, int64_t kpad, int64_t x1_begin,
                     int64_t rows, uint8_t* A, void* stream) {
  return mmj::star_operand(k, dims, heavy, kpad, x1_begin, rows, A, ST(stream));
}

size_t mmj_star_light_workspace_bytes(int64_t n_light) { return mmj::star_light_ws_bytes(n_light); }

int mmj_star_light(int k, const int64_t* dims, const int32_t* const* rev_ptr, const int32_t* const* rev_idx,
                   const int32_t* light_y, int64_t n_light, int64_t x1_begin, int64_t x1_end, int mode, void* out,
                   int64_t ld, unsigned long long* witnesses, void* ws, void* stream) {
  return mmj::star_light(k, dims, rev_ptr, rev_idx, light_y, n_light, x1_begin, x1_end, mode, out, ld, witnesses,
                         ws, ST(stream));
}

int64_t mmj_bitmap_segment_count(int64_t nwords) { return mmj::bitmap_nseg(nwords); }

int mmj_bitmap_segments(const uint32_t* bm, int64_t nwords, int32_t* segcnt, int64_t* seg_off, void* ws,
                        void* stream) {
  return mmj::bitmap_segments(bm, nwords, segcnt, seg_off, ws, ST(stream));
}

int mmj_bitmap_emit(const uint32_t* bm, int64_t nwords, int64_t wpr, const int64_t* seg_off, int64_t x0,
                    int64_t dom_z, int64_t* codes, void* stream) {
  return mmj::bitmap_emit(bm, nwords, wpr, seg_off, x0, dom_z, codes, ST(stream));
}

int64_t mmj_count_segment_count(int64_t ncell) { return mmj::count_nseg(ncell); }

int mmj_count_segments(const void* cnt, int cell_bytes, int64_t nrows, int64_t ld, int64_t ncols, int64_t x0,
                       int32_t min_count, const int32_t* row_min, int cell_filter, int32_t* segcnt, int64_t* seg_off,
                       void* ws, void* stream) {
  if (cell_bytes != 2 && cell_bytes != 4) {
    mmj::set_error("count_segments: cell_bytes must be 2 (uint16) or 4 (int32)");
    return MMJ_ERR_ARG;
  }
  if (cell_filter < 0 || cell_filter > 2) {
    mmj::set_error("count_segments: cell_filter must be 0, 1 or 2");
    return MMJ_ERR_ARG;
  }
  return mmj::count_segments(cnt, cell_bytes, nrows, ld, ncols, x0, min_count, row_min, cell_filter, segcnt, seg_off, ws,
                             ST(stream));
}

int mmj_count_emit(const void* cnt, int cell_bytes, int64_t nrows, int64_t ld, int64_t ncols, int64_t x0,
                   int64_t dom_z, int32_t min_count, const int32_t* row_min, int cell_filter, const int64_t* seg_off,
                   int64_t* codes, int32_t* counts, void* stream) {
  if (cell_bytes != 2 && cell_bytes != 4) {
    mmj::set_error("count_emit: cell_bytes must be 2 (uint16) or 4 (int32)");
    return MMJ_ERR_ARG;
  }
  if (cell_filter < 0 || cell_filter > 2) {
    mmj::set_error("count_emit: cell_filter must be 0, 1 or 2");
    return MMJ_ERR_ARG;
  }
  return mmj::count_emit(cnt, cell_bytes, nrows, ld, ncols, x0, dom_z, min_count, row_min, cell_filter, seg_off, codes,
                         counts,
                         ST(stream));
}

}  // extern "C"


// ---- result text formats (cli.py:129-136, 154-161, 180-182, 205-206) ----
static int fmt_args(mmj::FmtArgs& f, const int64_t* codes, const int64_t* counts, const int32_t* order, int64_t n,
                    int ncode, const int64_t* dims, const int32_t* const* rank, const int64_t* nrank,
                    const int64_t* const* soff, const uint8_t* const* blob) {
  const int ncol = ncode + (counts ? 1 : 0);
  if (ncode < 1 || ncol > 5 || n < 0 || (n > 0 && codes == nullptr)) {
    mmj::set_error("format: 1 <= code columns, columns (+ count) <= 5, n >= 0");
    return MMJ_ERR_ARG;
  }
  f.codes = codes;
  f.counts = counts;
  f.order = order;
  f.n = n;
  f.ncode = ncode;
  for (int c = 0; c < 5; ++c) {
    f.dims[c] = c < ncode ? dims[c] : 1;
    f.rank[c] = (c < ncol && rank) ? rank[c] : nullptr;
    f.nrank[c] = (c < ncol && nrank) ? nrank[c] : 1;
    f.soff[c] = (c < ncol && soff) ? soff[c] : nullptr;
    f.blob[c] = (c < ncol && blob) ? blob[c] : nullptr;
    if (c < ncode && f.dims[c] < 1) {
      mmj::set_error("format: dims must be >= 1");
      return MMJ_ERR_ARG;
    }
  }
  return MMJ_OK;
}

int mmj_format_keys(const int64_t* codes, const int64_t* counts, int64_t n, int ncode, const int64_t* dims,
                    const int32_t* const* rank, const int64_t* nrank, int64_t* key, int* bad, void* stream) {
  mmj::FmtArgs f;
  MMJ_TRY(fmt_args(f, codes, counts, nullptr, n, ncode, dims, rank, nrank, nullptr, nullptr));
  double span = 1.0;
  for (int c = 0; c < ncode + (counts ? 1 : 0); ++c) span *= (double)f.nrank[c];
  if (span >= 9.2e18) {
    mmj::set_error("format_keys: the columns' rank product exceeds int64");
    return MMJ_ERR_ARG;
  }
  return mmj::fmt_keys(f, key, bad, ST(stream));
}

int mmj_format_lengths(const int64_t* codes, const int64_t* counts, const int32_t* order, int64_t n, int ncode,
                       const int64_t* dims, const int64_t* const* soff, int32_t* len, void* stream) {
  mmj::FmtArgs f;
  MMJ_TRY(fmt_args(f, codes, counts, order, n, ncode, dims, nullptr, nullptr, soff, nullptr));
  return mmj::fmt_lengths(f, len, ST(stream));
}

int mmj_format_write(const int64_t* codes, const int64_t* counts, const int32_t* order, int64_t n, int ncode,
                     const int64_t* dims, const int64_t* const* soff, const uint8_t* const* blob,
                     const int64_t* line_off, uint8_t* out, void* stream) {
  mmj::FmtArgs f;
  MMJ_TRY(fmt_args(f, codes, counts, order, n, ncode, dims, nullptr, nullptr, soff, blob));
  return mmj::fmt_write(f, line_off, out, ST(stream));
}
