// Degree split, heavy-operand build, light expansion and the merge/emission
// kernels of the two-path join-project path.
//
// Reference (paths relative to /root/reference/pkg/src/mmjoin/):
//   degree split            joinproject.py:178-180, 100-116
//   heavy 0/1 matrices      joinproject.py:119-143
//   light passes 1-3        joinproject.py:183-203 (gather_ranges relation.py:193-204)
//   merge / dedup           joinproject.py:220-225, _merge_counts 146-152
//   full join               joinproject.py:228-248
//
// Layout in HBM (all dense ids int32):
//   relation CSR            fwd_ptr[dom_l+1], fwd_idx[n] (right id per tuple),
//                           fwd_row[n] (left id per tuple), rev_ptr[dom_r+1], rev_idx[n]
//   heavy position of y     hpos[dom_y] = rank among heavy y, -1 if light
//   operands                A[x][Kp], B[z][Kp] uint8 0/1, K-major (row = dense id)
//   light-z CSR of S        lz_ptr[dom_y+1], lz_idx[.]: S.rev(y) restricted to light z
//   output chunk            bitmap rows x words (1 bit per (x, z)), or int32 counts
//   codes                   int64 x*dom_z + z, strictly increasing (bitmap order)
#include "mmj_common.cuh"

namespace mmj {

namespace {

constexpr int TPB = 256;

inline int grid_for(int64_t work, int per_block, int cap_waves = 32) {
  int64_t g = ceil_div(work, per_block);
  int64_t cap = (int64_t)sm_count() * cap_waves;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ------------------------------------------------------------------ split
__global__ void k_heavy_y_flags(const int32_t* __restrict__ rdeg, const int32_t* __restrict__ sdeg,
                                int64_t dom_y, int64_t d1, uint8_t* __restrict__ flag) {
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < dom_y;
       y += (int64_t)gridDim.x * blockDim.x) {
    // joinproject.py:178: light iff deg_R(y) <= d1 and deg_S(y) <= d1
    flag[y] = (rdeg[y] > d1 || sdeg[y] > d1) ? 1 : 0;
  }
}

__global__ void k_heavy_y_pos(const uint8_t* __restrict__ flag, const int32_t* __restrict__ scanned,
                              int64_t dom_y, int32_t* __restrict__ hpos) {
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < dom_y;
       y += (int64_t)gridDim.x * blockDim.x)
    hpos[y] = flag[y] ? scanned[y] : -1;
}

// --------------------------------------------------------- operand build
// mat[(row - row0) * kpad + hpos[col]] = 1 for every tuple whose left id is
// heavy (deg > d2) -- joinproject.py:135-141 / 337-344.
__global__ void k_build_operand(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                int64_t n, const int32_t* __restrict__ left_deg, int64_t d2,
                                const int32_t* __restrict__ hpos, uint8_t* __restrict__ mat,
                                int64_t row0, int64_t nrows, int64_t kpad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[t] - row0;
    if (r < 0 || r >= nrows) continue;
    if (left_deg[rows[t]] <= d2) continue;
    const int32_t k = hpos[cols[t]];
    if (k >= 0) mat[r * kpad + k] = 1;
  }
}

// Heavy-y bit rows of S_h for the in-tile heavy product (rowemit.cu
// heavy_or_rows): bit z of row hpos[y] is set for every S tuple (z, y) with
// heavy z (deg_S(z) > d2) and heavy y -- the rows of joinproject.py:119-143's
// M2 stored one bit per cell.
__global__ void k_build_heavy_rows(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols, int64_t n,
                                   const int32_t* __restrict__ left_deg, int64_t d2, const int32_t* __restrict__ hpos,
                                   uint32_t* __restrict__ hbits, int64_t wpr) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t z = rows[t];
    if (left_deg[z] <= d2) continue;
    const int32_t k = hpos[cols[t]];
    MMJ_DCHECK(z >= 0 && (z >> 5) < wpr, "heavy row bit outside the row pitch");
    if (k >= 0) atomicOr(&hbits[(int64_t)k * wpr + (z >> 5)], 1u << (z & 31));
  }
}

// z-pair operand for MMJ_MODE_BITMAP_PAIR: z = 32G + b (b = k + 8j) goes to
// row 16G + 2k + (j >> 1) with weight 1 (j even) or 128 (j odd) -- the
// placement the heavy_mma pair epilogue unpacks (mma_i8.cu pack_bits_pair).
// The two halves of a byte come from different tuples -> word atomicOr.
__global__ void k_build_operand_pairs(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                      int64_t n, const int32_t* __restrict__ left_deg, int64_t d2,
                                      const int32_t* __restrict__ hpos, uint8_t* __restrict__ mat, int64_t row0,
                                      int64_t nrows, int64_t kpad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[t] - row0;
    if (r < 0 || r >= nrows) continue;
    if (left_deg[rows[t]] <= d2) continue;
    const int32_t k = hpos[cols[t]];
    if (k < 0) continue;
    const int b = (int)(r & 31), kk = b & 7, j = b >> 3;
    const int64_t prow = (r >> 5) * 16 + 2 * kk + (j >> 1);
    const int64_t off = prow * kpad + k;
    const uint32_t v = (j & 1) ? 0x80u : 0x01u;
    atomicOr(reinterpret_cast<unsigned int*>(mat + (off & ~int64_t(3))), v << (8 * (off & 3)));
  }
}

// ----------------------------------------------------------- light-z CSR
__global__ void k_lz_flags(const int32_t* __restrict__ rev_idx, int64_t n,
                           const int32_t* __restrict__ left_deg, int64_t d2, uint8_t* __restrict__ flag) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = left_deg[rev_idx[j]] <= d2 ? 1 : 0;
}

__global__ void k_lz_scatter(const int32_t* __restrict__ rev_idx, const uint8_t* __restrict__ flag,
                             const int32_t* __restrict__ pos, int64_t n, int32_t* __restrict__ lz_idx) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    if (flag[j]) lz_idx[pos[j]] = rev_idx[j];
}

__global__ void k_lz_ptr(const int32_t* __restrict__ rev_ptr, const int32_t* __restrict__ pos, int64_t dom_y,
                         int32_t* __restrict__ lz_ptr) {
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y <= dom_y;
       y += (int64_t)gridDim.x * blockDim.x)
    lz_ptr[y] = pos[rev_ptr[y]];
}

// -------------------------------------------------------- light passes
// x-driven restatement of the three witness-disjoint passes: every R tuple
// (x, y) of the chunk expands one list of S-side partners
//   y light                -> S.rev(y)                 (pass 1, joinproject.py:183-186)
//   y heavy, x light       -> S.rev(y)                 (pass 2, 188-193)
//   y heavy, x heavy       -> S.rev(y) ∩ light z       (pass 3, 195-203)
// hpos == nullptr means "no heavy y" (FULL_JOIN plan, joinproject.py:228-248).
struct LightArgs {
  const int32_t* fwd_row;
  const int32_t* fwd_idx;
  int64_t t0;
  const int32_t* rdeg_x;
  int64_t d2;
  const int32_t* hpos;
  const int32_t* s_rev_ptr;
  const int32_t* s_rev_idx;
  const int32_t* lz_ptr;
  const int32_t* lz_idx;
  int64_t min_deg;   // SSJ c-prefilter: left ids with degree < min_deg cannot reach overlap >= c
  int upper_only;    // SSJ: only z > x cells are ever emitted
};

__device__ __forceinline__ void list_of(const LightArgs& a, int64_t t, int32_t& x, const int32_t*& base,
                                        int32_t& len, bool& lz) {
  x = a.fwd_row[t];
  const int32_t y = a.fwd_idx[t];
  const bool full_list = (a.hpos == nullptr) || (a.hpos[y] < 0) || (a.rdeg_x[x] <= a.d2);
  lz = !full_list;
  if (full_list) {
    const int32_t b = a.s_rev_ptr[y];
    base = a.s_rev_idx + b;
    len = a.s_rev_ptr[y + 1] - b;
  } else {
    const int32_t b = a.lz_ptr[y];
    base = a.lz_idx + b;
    len = a.lz_ptr[y + 1] - b;
  }
}

__global__ void k_light_len(LightArgs a, int64_t ntup, int32_t* __restrict__ len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ntup;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t x, l;
    const int32_t* b;
    bool lz;
    list_of(a, a.t0 + i, x, b, l, lz);
    // c-prefilter (ssj_mmjoin, apps.py:57-62): a row whose set has fewer than c
    // elements, or a light-z list (all its z have degree <= d2 < c), cannot
    // produce a pair with overlap >= c; skipping them leaves the output unchanged
    if (a.min_deg > 1 && (a.rdeg_x[x] < a.min_deg || (lz && a.d2 < a.min_deg))) l = 0;
    len[i] = l;
  }
}

constexpr int EXP_THREADS = 256;
constexpr int EXP_ITEMS = 8;
constexpr int EXP_SPAN = EXP_THREADS * EXP_ITEMS;

__device__ __forceinline__ int64_t upper_bound_i64(const int64_t* __restrict__ v, int64_t lo, int64_t hi,
                                                   int64_t key) {
  // first index in [lo, hi) with v[idx] > key
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (v[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// mode 0: bitmap atomicOr; mode 1: int32 counts atomicAdd; mode 2: uint16 counts
template <int MODE>
__global__ void __launch_bounds__(EXP_THREADS) k_light_expand(LightArgs a, const int64_t* __restrict__ offs,
                                                              int64_t ntup, int64_t x0, void* __restrict__ out,
                                                              int64_t ld) {
  __shared__ int64_t s_lo, s_hi;
  const int64_t total = offs[ntup];
  for (int64_t span0 = (int64_t)blockIdx.x * EXP_SPAN; span0 < total; span0 += (int64_t)gridDim.x * EXP_SPAN) {
    const int64_t span1 = min(span0 + (int64_t)EXP_SPAN, total);
    if (threadIdx.x == 0) {
      s_lo = upper_bound_i64(offs, 0, ntup + 1, span0) - 1;
      s_hi = upper_bound_i64(offs, 0, ntup + 1, span1 - 1);
    }
    __syncthreads();
    const int64_t lo = s_lo, hi = s_hi;
#pragma unroll 2
    for (int it = 0; it < EXP_ITEMS; ++it) {
      const int64_t s = span0 + (int64_t)it * EXP_THREADS + threadIdx.x;
      if (s >= span1) break;
      const int64_t i = upper_bound_i64(offs, lo, hi, s) - 1;
      int32_t x, l;
      const int32_t* base;
      bool lz;
      list_of(a, a.t0 + i, x, base, l, lz);
      const int32_t z = base[s - offs[i]];
      const int64_t row = (int64_t)x - x0;
      if (a.upper_only == 1 && z <= x) continue;  // SSJ keeps a < b only (apps.py:60)
      MMJ_DCHECK(row >= 0 && z >= 0 && (MODE == 0 ? (z >> 5) < ld : (MODE == 1 ? z < ld : (z >> 1) < (ld >> 1))),
                 "light witness outside the chunk's output block");
      if (MODE == 0) {
        atomicOr(reinterpret_cast<uint32_t*>(out) + row * ld + (z >> 5), 1u << (z & 31));
      } else if (MODE == 1) {
        atomicAdd(reinterpret_cast<int32_t*>(out) + row * ld + z, 1);
      } else {   // uint16 counts, two per word (no carry: every count < 2^16)
        atomicAdd(reinterpret_cast<unsigned int*>(out) + row * (ld >> 1) + (z >> 1), (z & 1) ? 0x10000u : 1u);
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- emission
// A segment is 32 consecutive bitmap words (1024 (x, z) cells); codes come
// out in bitmap order = ascending code order, so the merge needs no sort.
constexpr int SEG_WORDS = 32;

__global__ void k_seg_popc(const uint32_t* __restrict__ bm, int64_t nwords, int32_t* __restrict__ segcnt,
                           int64_t nseg) {
  for (int64_t sgi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; sgi < nseg;
       sgi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w0 = sgi * SEG_WORDS;
    int c = 0;
    if (w0 + SEG_WORDS <= nwords) {
      const uint4* p = reinterpret_cast<const uint4*>(bm + w0);
#pragma unroll
      for (int i = 0; i < SEG_WORDS / 4; ++i) {
        uint4 v = p[i];
        c += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
      }
    } else {
      for (int64_t w = w0; w < nwords; ++w) c += __popc(bm[w]);
    }
    segcnt[sgi] = c;
  }
}

constexpr int EMIT_WARPS = 4;   // 4 x 8 KB staging (static smem limit 48 KB)

__global__ void __launch_bounds__(EMIT_WARPS * 32) k_bitmap_emit(const uint32_t* __restrict__ bm, int64_t nwords,
                                                                 int64_t wpr, const int64_t* __restrict__ seg_off,
                                                                 int64_t nseg, int64_t x0, int64_t dom_z,
                                                                 int64_t* __restrict__ codes) {
  __shared__ int64_t stage[EMIT_WARPS][SEG_WORDS * 32];
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int64_t* st = stage[wib];
  for (int64_t sgi = (int64_t)blockIdx.x * EMIT_WARPS + wib; sgi < nseg; sgi += (int64_t)gridDim.x * EMIT_WARPS) {
    const int64_t w = sgi * SEG_WORDS + lane;
    uint32_t word = w < nwords ? bm[w] : 0u;
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int k = incl - c;
    const int64_t row = w / wpr;
    const int64_t code0 = (x0 + row) * dom_z + (w - row * wpr) * 32;
    while (word) {
      const int b = __ffs(word) - 1;
      st[k++] = code0 + b;
      word &= word - 1;
    }
    __syncwarp();
    const int64_t base = seg_off[sgi];
    for (int i = lane; i < total; i += 32) codes[base + i] = st[i];
    __syncwarp();
  }
}

// count matrix (rows x ld cells of int32 or uint16, ld a multiple of CSEG,
// ncols valid): keep cells with value >= min_count (per-row max(min_count,
// row_min[x])) that pass the cell filter.  One warp per 1024-cell segment,
// which always lies inside one row; lane l loads VEC cells per int4 (4 int32
// or 8 uint16), ITS coalesced int4s per lane.  Segments entirely at or below
// the diagonal (filter 1) or right of ncols are never read - the MMA leaves
// the former unwritten.
constexpr int CSEG = 1024;   // cells per count segment

template <typename CellT>
struct CellGeo {
  static constexpr int VEC = 16 / (int)sizeof(CellT);    // cells per int4
  static constexpr int ITS = CSEG / (32 * VEC);            // int4 loads per lane
  static constexpr int FIELD = 32 * VEC >= 256 ? 16 : 8;   // bits of a per-iteration count field
};

struct CountSeg {
  int64_t row, col0;
  bool live;
};

__device__ __forceinline__ CountSeg count_seg(int64_t sgi, int64_t spr, int64_t ncols, int64_t x0, int upper_only) {
  CountSeg g;
  g.row = sgi / spr;
  g.col0 = (sgi - g.row * spr) * CSEG;
  g.live = g.col0 < ncols && !(upper_only == 1 && g.col0 + CSEG - 1 <= x0 + g.row);
  return g;
}

template <typename CellT>
__device__ __forceinline__ int32_t cell_of(int4 v, int j) {
  const int32_t words[4] = {v.x, v.y, v.z, v.w};
  if constexpr (sizeof(CellT) == 4) {
    return words[j];
  } else {
    const uint32_t w = (uint32_t)words[j >> 1];
    return (int32_t)((j & 1) ? (w >> 16) : (w & 0xFFFFu));   // low half = even column
  }
}

// keep flags of one int4 of cells (VEC bits, cell j -> bit j)
// cell filters: 0 every cell, 1 z > x (SSJ's a < b), 2 z != x (SCJ's a != b)
template <typename CellT>
__device__ __forceinline__ uint32_t keep_mask(int4 v, int64_t col, int64_t x, int64_t ncols, int32_t min_count,
                                              int filter) {
  const int64_t lo = filter == 1 ? x + 1 : 0;   // first kept column
  const int64_t skip = filter == 2 ? x : -1;    // the one excluded column
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < CellGeo<CellT>::VEC; ++j) {
    const int64_t c = col + j;
    m |= (cell_of<CellT>(v, j) >= min_count && c >= lo && c < ncols && c != skip) ? (1u << j) : 0u;
  }
  return m;
}

// interior segments (no cell filter or pitch edge inside): value test only,
// two uint16 cells per SIMD compare
template <typename CellT>
__device__ __forceinline__ uint32_t keep_mask_fast(int4 v, int32_t thr) {
  if constexpr (sizeof(CellT) == 4) {
    return (uint32_t)(v.x >= thr) | ((uint32_t)(v.y >= thr) << 1) | ((uint32_t)(v.z >= thr) << 2) |
           ((uint32_t)(v.w >= thr) << 3);
  } else {
    if (thr > 65535) return 0u;
    const uint32_t t2 = (uint32_t)thr * 0x00010001u;
    const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t c = __vcmpgeu2(w[k], t2);
      m |= ((c & 1u) | ((c >> 15) & 2u)) << (2 * k);
    }
    return m;
  }
}

__device__ __forceinline__ bool interior_seg(const CountSeg& g, int64_t x, int64_t ncols, int filter) {
  const int64_t lo = filter == 1 ? x + 1 : 0;
  return g.col0 >= lo && g.col0 + CSEG <= ncols && !(filter == 2 && x >= g.col0 && x < g.col0 + CSEG);
}

template <typename CellT>
__global__ void __launch_bounds__(256) k_count_seg_nnz(const CellT* __restrict__ cnt, int64_t nseg, int64_t spr,
                                                       int64_t ld, int64_t ncols, int64_t x0, int32_t min_count,
                                                       const int32_t* __restrict__ row_min, int upper_only,
                                                       int32_t* __restrict__ segcnt) {
  using G = CellGeo<CellT>;
  const int lane = threadIdx.x & 31;
  for (int64_t sgi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; sgi < nseg;
       sgi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const CountSeg g = count_seg(sgi, spr, ncols, x0, upper_only);
    int n = 0;
    if (g.live) {
      const int4* src = reinterpret_cast<const int4*>(cnt + g.row * ld + g.col0) + lane;
      const int32_t thr = row_min ? max(min_count, row_min[x0 + g.row]) : min_count;
      int4 v[G::ITS];
#pragma unroll
      for (int it = 0; it < G::ITS; ++it) v[it] = __ldcs(src + it * 32);
      if (interior_seg(g, x0 + g.row, ncols, upper_only)) {
#pragma unroll
        for (int it = 0; it < G::ITS; ++it) n += __popc(keep_mask_fast<CellT>(v[it], thr));
      } else {
#pragma unroll
        for (int it = 0; it < G::ITS; ++it)
          n += __popc(keep_mask<CellT>(v[it], g.col0 + (it * 32 + lane) * G::VEC, x0 + g.row, ncols, thr,
                                       upper_only));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    }
    if (lane == 0) segcnt[sgi] = n;
  }
}

template <typename CellT>
__global__ void __launch_bounds__(256) k_count_emit(const CellT* __restrict__ cnt, int64_t nseg, int64_t spr,
                                                    int64_t ld, int64_t ncols, int64_t x0, int64_t dom_z,
                                                    int32_t min_count, const int32_t* __restrict__ row_min,
                                                    int upper_only, const int64_t* __restrict__ seg_off,
                                                    int64_t* __restrict__ codes, int32_t* __restrict__ counts) {
  using G = CellGeo<CellT>;
  constexpr uint64_t FMASK = (1ull << G::FIELD) - 1;
  // per-warp staging of the segment's kept cells (column offset, count), so
  // the codes and counts leave as coalesced runs instead of one scattered
  // 8-B / 4-B store per kept cell per lane
  __shared__ uint16_t s_col[8][CSEG];
  __shared__ int32_t s_cnt[8][CSEG];
  const int lane = threadIdx.x & 31;
  const int wib = (threadIdx.x >> 5) & 7;
  for (int64_t sgi = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; sgi < nseg;
       sgi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const CountSeg g = count_seg(sgi, spr, ncols, x0, upper_only);
    if (!g.live) continue;
    const int64_t base = seg_off[sgi];
    if (seg_off[sgi + 1] == base) continue;
    const int4* src = reinterpret_cast<const int4*>(cnt + g.row * ld + g.col0) + lane;
    const int32_t thr = row_min ? max(min_count, row_min[x0 + g.row]) : min_count;
    int4 v[G::ITS];
#pragma unroll
    for (int it = 0; it < G::ITS; ++it) v[it] = __ldcs(src + it * 32);
    // a count field per iteration, packed, warp-scanned in one pass
    uint32_t msk[G::ITS];
    uint64_t packed = 0;
    const bool inner = interior_seg(g, x0 + g.row, ncols, upper_only);
#pragma unroll
    for (int it = 0; it < G::ITS; ++it) {
      msk[it] = inner ? keep_mask_fast<CellT>(v[it], thr)
                      : keep_mask<CellT>(v[it], g.col0 + (it * 32 + lane) * G::VEC, x0 + g.row, ncols, thr,
                                         upper_only);
      packed |= (uint64_t)__popc(msk[it]) << (G::FIELD * it);
    }
    uint64_t incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const uint64_t tot = __shfl_sync(0xffffffffu, incl, 31);   // per-iteration totals
    const uint64_t excl = incl - packed;
    const int64_t code_row = (x0 + g.row) * dom_z + g.col0;
    int it_base = 0;
#pragma unroll
    for (int it = 0; it < G::ITS; ++it) {
      const uint32_t m = msk[it];
      int k = it_base + (int)((excl >> (G::FIELD * it)) & FMASK);
#pragma unroll
      for (int j = 0; j < G::VEC; ++j) {
        if (m & (1u << j)) {
          s_col[wib][k] = (uint16_t)((it * 32 + lane) * G::VEC + j);
          s_cnt[wib][k] = cell_of<CellT>(v[it], j);
          ++k;
        }
      }
      it_base += (int)((tot >> (G::FIELD * it)) & FMASK);
    }
    __syncwarp();
    for (int p = lane; p < it_base; p += 32) {
      __stcs(codes + base + p, code_row + s_col[wib][p]);
      __stcs(counts + base + p, s_cnt[wib][p]);
    }
    __syncwarp();
  }
}

}  // namespace

// ============================================================== host API
int heavy_y_positions(const int32_t* rdeg_y, const int32_t* sdeg_y, int64_t dom_y, int64_t d1, uint8_t* flag_ws,
                      int32_t* scan_ws_out /*dom_y+1*/, int32_t* hpos, void* ws, cudaStream_t st) {
  if (dom_y == 0) return cuda_status(cudaMemsetAsync(scan_ws_out, 0, 4, st), "memset");
  k_heavy_y_flags<<<grid_for(dom_y, TPB), TPB, 0, st>>>(rdeg_y, sdeg_y, dom_y, d1, flag_ws);
  MMJ_CHECK_LAUNCH("k_heavy_y_flags");
  MMJ_TRY(scan_u8_i32(flag_ws, scan_ws_out, dom_y, ws, st));
  k_heavy_y_pos<<<grid_for(dom_y, TPB), TPB, 0, st>>>(flag_ws, scan_ws_out, dom_y, hpos);
  MMJ_CHECK_LAUNCH("k_heavy_y_pos");
  return MMJ_OK;
}

int build_operand(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t d2,
                  const int32_t* hpos, uint8_t* mat, int64_t row0, int64_t nrows, int64_t kpad, cudaStream_t st) {
  MMJ_TRY(cuda_status(cudaMemsetAsync(mat, 0, (size_t)(nrows * kpad), st), "memset operand"));
  if (n == 0) return MMJ_OK;
  k_build_operand<<<grid_for(n, TPB), TPB, 0, st>>>(rows, cols, n, left_deg, d2, hpos, mat, row0, nrows, kpad);
  MMJ_CHECK_LAUNCH("k_build_operand");
  return MMJ_OK;
}

// stats[0] = #{x : left_deg[x] > d2}, stats[1] = #{tuples (x, y) : left_deg[x] > d2 and hpos[y] >= 0}
// (the engine's choice between the tcgen05 product and the in-tile OR)
__global__ void k_heavy_row_stats(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols, int64_t n,
                                  const int32_t* __restrict__ left_deg, int64_t dom, int64_t d2,
                                  const int32_t* __restrict__ hpos, unsigned long long* __restrict__ stats) {
  unsigned long long nh = 0, nt = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dom; i += stride) nh += left_deg[i] > d2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride)
    nt += (left_deg[rows[t]] > d2) && hpos[cols[t]] >= 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nh += __shfl_xor_sync(0xffffffffu, nh, o);
    nt += __shfl_xor_sync(0xffffffffu, nt, o);
  }
  if ((threadIdx.x & 31) == 0 && (nh | nt)) {
    atomicAdd(stats, nh);
    atomicAdd(stats + 1, nt);
  }
}

int heavy_row_stats(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t dom,
                    int64_t d2, const int32_t* hpos, int64_t* stats, cudaStream_t st) {
  MMJ_TRY(cuda_status(cudaMemsetAsync(stats, 0, 2 * sizeof(int64_t), st), "memset heavy row stats"));
  if (n == 0 && dom == 0) return MMJ_OK;
  k_heavy_row_stats<<<grid_for(n > dom ? n : dom, TPB), TPB, 0, st>>>(
      rows, cols, n, left_deg, dom, d2, hpos, reinterpret_cast<unsigned long long*>(stats));
  MMJ_CHECK_LAUNCH("k_heavy_row_stats");
  return MMJ_OK;
}

int build_heavy_rows(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t d2,
                     const int32_t* hpos, uint32_t* hbits, int64_t k, int64_t wpr, cudaStream_t st) {
  if (k < 0 || wpr <= 0 || wpr % 4 != 0) {
    set_error("build_heavy_rows: k >= 0 and a positive row pitch (multiple of 4 words) are required");
    return MMJ_ERR_ARG;
  }
  MMJ_TRY(cuda_status(cudaMemsetAsync(hbits, 0, (size_t)(k * wpr) * 4, st), "memset heavy rows"));
  if (n == 0 || k == 0) return MMJ_OK;
  k_build_heavy_rows<<<grid_for(n, TPB), TPB, 0, st>>>(rows, cols, n, left_deg, d2, hpos, hbits, wpr);
  MMJ_CHECK_LAUNCH("k_build_heavy_rows");
  return MMJ_OK;
}

int build_operand_pairs(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* left_deg, int64_t d2,
                        const int32_t* hpos, uint8_t* mat, int64_t row0, int64_t nrows, int64_t kpad,
                        cudaStream_t st) {
  if (kpad % 4 != 0 || reinterpret_cast<uintptr_t>(mat) % 4 != 0 || nrows % 32 != 0) {
    set_error("build_operand_pairs: kpad and mat must be 4-byte aligned, nrows a multiple of 32");
    return MMJ_ERR_ARG;
  }
  MMJ_TRY(cuda_status(cudaMemsetAsync(mat, 0, (size_t)((nrows / 2) * kpad), st), "memset operand"));
  if (n == 0) return MMJ_OK;
  k_build_operand_pairs<<<grid_for(n, TPB), TPB, 0, st>>>(rows, cols, n, left_deg, d2, hpos, mat, row0, nrows,
                                                          kpad);
  MMJ_CHECK_LAUNCH("k_build_operand_pairs");
  return MMJ_OK;
}

int light_z_csr(const int32_t* rev_ptr, const int32_t* rev_idx, int64_t n, int64_t dom_y, const int32_t* left_deg,
                int64_t d2, uint8_t* flag_ws, int32_t* pos_ws /*n+1*/, int32_t* lz_ptr, int32_t* lz_idx, void* ws,
                cudaStream_t st) {
  if (n > 0) {
    k_lz_flags<<<grid_for(n, TPB), TPB, 0, st>>>(rev_idx, n, left_deg, d2, flag_ws);
    MMJ_CHECK_LAUNCH("k_lz_flags");
  }
  MMJ_TRY(scan_u8_i32(flag_ws, pos_ws, n, ws, st));
  if (n > 0) {
    k_lz_scatter<<<grid_for(n, TPB), TPB, 0, st>>>(rev_idx, flag_ws, pos_ws, n, lz_idx);
    MMJ_CHECK_LAUNCH("k_lz_scatter");
  }
  k_lz_ptr<<<grid_for(dom_y + 1, TPB), TPB, 0, st>>>(rev_ptr, pos_ws, dom_y, lz_ptr);
  MMJ_CHECK_LAUNCH("k_lz_ptr");
  return MMJ_OK;
}

int light_lengths(const int32_t* fwd_row, const int32_t* fwd_idx, int64_t t0, int64_t ntup, const int32_t* rdeg_x,
                  int64_t d2, const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx,
                  const int32_t* lz_ptr, const int32_t* lz_idx, int64_t min_deg, int upper_only, int32_t* len,
                  int64_t* offs, void* ws, cudaStream_t st) {
  LightArgs a{fwd_row, fwd_idx, t0, rdeg_x, d2, hpos, s_rev_ptr, s_rev_idx, lz_ptr, lz_idx, min_deg, upper_only};
  if (ntup > 0) {
    k_light_len<<<grid_for(ntup, TPB), TPB, 0, st>>>(a, ntup, len);
    MMJ_CHECK_LAUNCH("k_light_len");
  }
  return scan_i32_i64(len, offs, ntup, ws, st);
}

int light_expand(const int32_t* fwd_row, const int32_t* fwd_idx, int64_t t0, int64_t ntup, const int32_t* rdeg_x,
                 int64_t d2, const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx,
                 const int32_t* lz_ptr, const int32_t* lz_idx, int64_t min_deg, int upper_only, const int64_t* offs,
                 int64_t total_hint, int mode, int64_t x0, void* out, int64_t ld, cudaStream_t st) {
  if (ntup == 0 || total_hint == 0) return MMJ_OK;
  LightArgs a{fwd_row, fwd_idx, t0, rdeg_x, d2, hpos, s_rev_ptr, s_rev_idx, lz_ptr, lz_idx, min_deg, upper_only};
  const int64_t work = total_hint > 0 ? total_hint : ntup;
  const int grid = grid_for(work, EXP_SPAN, 8);
  if (mode == 0)
    k_light_expand<0><<<grid, EXP_THREADS, 0, st>>>(a, offs, ntup, x0, out, ld);
  else if (mode == 1)
    k_light_expand<1><<<grid, EXP_THREADS, 0, st>>>(a, offs, ntup, x0, out, ld);
  else
    k_light_expand<2><<<grid, EXP_THREADS, 0, st>>>(a, offs, ntup, x0, out, ld);
  MMJ_CHECK_LAUNCH("k_light_expand");
  return MMJ_OK;
}

int64_t bitmap_nseg(int64_t nwords) { return ceil_div(nwords, SEG_WORDS); }
int64_t count_nseg(int64_t ncell) { return ceil_div(ncell, CSEG); }

int bitmap_segments(const uint32_t* bm, int64_t nwords, int32_t* segcnt, int64_t* seg_off, void* ws,
                    cudaStream_t st) {
  const int64_t nseg = bitmap_nseg(nwords);
  if (nseg > 0) {
    k_seg_popc<<<grid_for(nseg, TPB), TPB, 0, st>>>(bm, nwords, segcnt, nseg);
    MMJ_CHECK_LAUNCH("k_seg_popc");
  }
  return scan_i32_i64(segcnt, seg_off, nseg, ws, st);
}

int bitmap_emit(const uint32_t* bm, int64_t nwords, int64_t wpr, const int64_t* seg_off, int64_t x0, int64_t dom_z,
                int64_t* codes, cudaStream_t st) {
  const int64_t nseg = bitmap_nseg(nwords);
  if (nseg == 0) return MMJ_OK;
  k_bitmap_emit<<<grid_for(nseg, EMIT_WARPS, 16), EMIT_WARPS * 32, 0, st>>>(bm, nwords, wpr, seg_off, nseg, x0,
                                                                            dom_z, codes);
  MMJ_CHECK_LAUNCH("k_bitmap_emit");
  return MMJ_OK;
}

static int check_count_pitch(int64_t ld, int64_t ncols) {
  if (ld % CSEG != 0 || ld < ncols) {
    set_error("count matrix pitch %lld must be a multiple of %d and >= %lld columns", (long long)ld, CSEG,
              (long long)ncols);
    return MMJ_ERR_ARG;
  }
  return MMJ_OK;
}

static int count_grid(int64_t nseg) {
  // 8 warps per CTA, 8 CTAs per SM resident; grid-stride beyond that
  const int64_t ctas = ceil_div(nseg, (int64_t)8);
  const int64_t cap = (int64_t)sm_count() * 8;
  return (int)(ctas < cap ? ctas : cap);
}

int count_segments(const void* cnt, int cell_bytes, int64_t nrows, int64_t ld, int64_t ncols, int64_t x0,
                   int32_t min_count, const int32_t* row_min, int upper_only, int32_t* segcnt, int64_t* seg_off,
                   void* ws, cudaStream_t st) {
  MMJ_TRY(check_count_pitch(ld, ncols));
  const int64_t nseg = count_nseg(nrows * ld);
  if (nseg > 0) {
    if (cell_bytes == 2)
      k_count_seg_nnz<uint16_t><<<count_grid(nseg), 256, 0, st>>>(static_cast<const uint16_t*>(cnt), nseg, ld / CSEG,
                                                                   ld, ncols, x0, min_count, row_min, upper_only,
                                                                   segcnt);
    else
      k_count_seg_nnz<int32_t><<<count_grid(nseg), 256, 0, st>>>(static_cast<const int32_t*>(cnt), nseg, ld / CSEG, ld,
                                                                  ncols, x0, min_count, row_min, upper_only, segcnt);
    MMJ_CHECK_LAUNCH("k_count_seg_nnz");
  }
  return scan_i32_i64(segcnt, seg_off, nseg, ws, st);
}

int count_emit(const void* cnt, int cell_bytes, int64_t nrows, int64_t ld, int64_t ncols, int64_t x0, int64_t dom_z,
               int32_t min_count, const int32_t* row_min, int upper_only, const int64_t* seg_off, int64_t* codes,
               int32_t* counts, cudaStream_t st) {
  MMJ_TRY(check_count_pitch(ld, ncols));
  const int64_t nseg = count_nseg(nrows * ld);
  if (nseg == 0) return MMJ_OK;
  if (cell_bytes == 2)
    k_count_emit<uint16_t><<<count_grid(nseg), 256, 0, st>>>(static_cast<const uint16_t*>(cnt), nseg, ld / CSEG, ld,
                                                              ncols, x0, dom_z, min_count, row_min, upper_only,
                                                              seg_off, codes, counts);
  else
    k_count_emit<int32_t><<<count_grid(nseg), 256, 0, st>>>(static_cast<const int32_t*>(cnt), nseg, ld / CSEG, ld,
                                                             ncols, x0, dom_z, min_count, row_min, upper_only,
                                                             seg_off, codes, counts);
  MMJ_CHECK_LAUNCH("k_count_emit");
  return MMJ_OK;
}

}  // namespace mmj
