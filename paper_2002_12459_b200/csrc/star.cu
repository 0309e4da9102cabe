// Star join-project pi_{x1..xk}(R1(x1,y) ... Rk(xk,y)), k = 2..4
// (joinproject.py:281-378, star_join).
//
// The output is laid out as a two-path over composite rows: row =
// (x1, .., x_{k-1}) in mixed radix, column = x_k, so code = row * d_k + x_k
// is exactly the reference's _encode (joinproject.py:80-84).  For a chunk of
// x1 values:
//   * k_star_operand builds the A operand of the tensor-core product: row
//     (x1..x_{k-1}) = AND of the heavy-y rows H_1[x1] & .. & H_{k-1}[x_{k-1}]
//     (the Khatri-Rao rows of joinproject.py:346-351, generated on the fly
//     per chunk instead of materialising all prod(|x_h|) rows); B = H_k;
//     the heavy product (mma_i8.cu) then writes the nonzero bitmap or exact
//     counts of the chunk;
//   * k_star_light_count / _expand enumerate the light witnesses balanced by
//     witness index: per light y its count inside the chunk's x1 range, a
//     scan, then contiguous witness runs per thread, each OR-ed (or counted)
//     into the chunk's bitmap;
// heavy and light y are disjoint, so bits OR and counts add exactly.
#include "mmj_common.cuh"

namespace mmj {
namespace {

constexpr int TPB = 256;

struct StarRels {
  int k;
  int64_t dims[4];
  const int32_t* rev_ptr[4];
  const int32_t* rev_idx[4];
  const uint8_t* heavy[4];    // H_j[x][kpad] uint8 0/1 (heavy y columns)
};

__global__ void k_star_operand(StarRels s, int64_t kpad, int64_t x1_begin, int64_t rows, uint8_t* __restrict__ A) {
  const int64_t q16 = kpad / 16;
  const int64_t total = rows * q16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / q16, q = i - r * q16;
    // decompose the composite row (x1 - x1_begin, x2, .., x_{k-1})
    int64_t rem = r;
    int64_t x[4];
    for (int j = s.k - 2; j >= 1; --j) {
      x[j] = rem % s.dims[j];
      rem /= s.dims[j];
    }
    x[0] = x1_begin + rem;
    uint4 v = reinterpret_cast<const uint4*>(s.heavy[0] + x[0] * kpad)[q];
    for (int j = 1; j <= s.k - 2; ++j) {
      const uint4 w = reinterpret_cast<const uint4*>(s.heavy[j] + x[j] * kpad)[q];
      v.x &= w.x;
      v.y &= w.y;
      v.z &= w.z;
      v.w &= w.w;
    }
    reinterpret_cast<uint4*>(A + r * kpad)[q] = v;
  }
}

__device__ __forceinline__ int lb32(const int32_t* v, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// mode 0: bitmap (ld words per row), mode 1: int32 counts (ld per row)
// Witness-balanced form: per light y its witness count inside the chunk
// (x1 list restricted by binary search) and restricted list start, a scan,
// then every thread expands a contiguous run of witness indices: the product
// of a few large light y no longer serialises on one warp.
__global__ void k_star_light_count(StarRels s, const int32_t* __restrict__ light_y, int64_t nly, int64_t x1_begin,
                                   int64_t x1_end, int64_t* __restrict__ cnt, int32_t* __restrict__ start0) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < nly; li += (int64_t)gridDim.x * blockDim.x) {
    const int32_t y = light_y[li];
    const int32_t b0 = s.rev_ptr[0][y];
    const int n0 = s.rev_ptr[0][y + 1] - b0;
    const int lo = lb32(s.rev_idx[0] + b0, n0, (int32_t)x1_begin);
    const int hi = lb32(s.rev_idx[0] + b0, n0, (int32_t)x1_end);
    int64_t total = hi - lo;
    for (int j = 1; j < s.k; ++j) total *= (int64_t)(s.rev_ptr[j][y + 1] - s.rev_ptr[j][y]);
    cnt[li] = total;
    start0[li] = b0 + lo;
  }
}

constexpr int SL_THREADS = 256;
constexpr int SL_ITEMS = 8;
constexpr int SL_SPAN = SL_THREADS * SL_ITEMS;

__device__ __forceinline__ int64_t ub64(const int64_t* __restrict__ v, int64_t lo, int64_t hi, int64_t key) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (v[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(SL_THREADS) k_star_light_expand(StarRels s, const int32_t* __restrict__ light_y,
                                                                  int64_t nly, const int64_t* __restrict__ offs,
                                                                  const int32_t* __restrict__ start0,
                                                                  int64_t x1_begin, int mode, void* __restrict__ out,
                                                                  int64_t ld) {
  __shared__ int64_t s_lo, s_hi;
  const int64_t total = offs[nly];
  for (int64_t span0 = (int64_t)blockIdx.x * SL_SPAN; span0 < total; span0 += (int64_t)gridDim.x * SL_SPAN) {
    const int64_t span1 = min(span0 + (int64_t)SL_SPAN, total);
    if (threadIdx.x == 0) {
      s_lo = ub64(offs, 0, nly + 1, span0) - 1;
      s_hi = ub64(offs, 0, nly + 1, span1 - 1);
    }
    __syncthreads();
    const int64_t lo = s_lo, hi = s_hi;
    for (int it = 0; it < SL_ITEMS; ++it) {
      const int64_t w = span0 + (int64_t)it * SL_THREADS + threadIdx.x;
      if (w >= span1) break;
      const int64_t li = ub64(offs, lo, hi, w) - 1;
      const int32_t y = light_y[li];
      int64_t rem = w - offs[li];
      int32_t xv[4];
      // mixed radix over the k lists, x_k fastest (32-bit when the lists allow)
      for (int j = s.k - 1; j >= 1; --j) {
        const int32_t b = s.rev_ptr[j][y];
        const int32_t n = s.rev_ptr[j][y + 1] - b;
        const int64_t q = rem / n;
        xv[j] = s.rev_idx[j][b + (int32_t)(rem - q * n)];
        rem = q;
      }
      xv[0] = s.rev_idx[0][start0[li] + (int32_t)rem];
      int64_t row = xv[0] - x1_begin;
      for (int j = 1; j <= s.k - 2; ++j) row = row * s.dims[j] + xv[j];
      const int32_t col = xv[s.k - 1];
      MMJ_DCHECK(row >= 0 && col >= 0 && (mode == 0 ? (col >> 5) < ld : col < ld), "star witness outside its block");
      if (mode == 0)
        atomicOr(reinterpret_cast<uint32_t*>(out) + row * ld + (col >> 5), 1u << (col & 31));
      else
        atomicAdd(reinterpret_cast<int32_t*>(out) + row * ld + col, 1);
    }
    __syncthreads();
  }
}

__global__ void k_add_total(const int64_t* __restrict__ total, unsigned long long* __restrict__ acc) {
  *acc += (unsigned long long)*total;
}

// y is "heavy" for the tensor-core product when prod_j deg_j(y) > threshold;
// heavy[y] / light[y] flags feed two scans (positions / compacted light list)
__global__ void k_star_split(StarRels s, int64_t dom_y, double threshold, uint8_t* __restrict__ heavy,
                             uint8_t* __restrict__ light) {
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < dom_y; y += (int64_t)gridDim.x * blockDim.x) {
    double prod = 1.0;
    for (int j = 0; j < s.k; ++j) prod *= (double)(s.rev_ptr[j][y + 1] - s.rev_ptr[j][y]);
    const bool h = prod > threshold;
    heavy[y] = h ? 1 : 0;
    light[y] = (!h && prod > 0.0) ? 1 : 0;
  }
}

__global__ void k_star_positions(const uint8_t* __restrict__ heavy, const int32_t* __restrict__ hscan,
                                 const uint8_t* __restrict__ light, const int32_t* __restrict__ lscan, int64_t dom_y,
                                 int32_t* __restrict__ hpos, int32_t* __restrict__ light_y) {
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < dom_y; y += (int64_t)gridDim.x * blockDim.x) {
    hpos[y] = heavy[y] ? hscan[y] : -1;
    if (light[y]) light_y[lscan[y]] = (int32_t)y;
  }
}

}  // namespace

int star_split(int k, const int32_t* const* rev_ptr, int64_t dom_y, double threshold, uint8_t* hflag, uint8_t* lflag,
               int32_t* hscan, int32_t* lscan, int32_t* hpos, int32_t* light_y, void* ws, cudaStream_t st) {
  if (k < 2 || k > 4) {
    set_error("star_split: 2 <= k <= 4 required");
    return MMJ_ERR_ARG;
  }
  StarRels s{};
  s.k = k;
  for (int j = 0; j < k; ++j) s.rev_ptr[j] = rev_ptr[j];
  if (dom_y > 0) {
    int64_t g = ceil_div(dom_y, TPB);
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    k_star_split<<<(unsigned)g, TPB, 0, st>>>(s, dom_y, threshold, hflag, lflag);
    MMJ_CHECK_LAUNCH("k_star_split");
  }
  MMJ_TRY(scan_u8_i32(hflag, hscan, dom_y, ws, st));
  MMJ_TRY(scan_u8_i32(lflag, lscan, dom_y, ws, st));
  if (dom_y > 0) {
    int64_t g = ceil_div(dom_y, TPB);
    if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
    k_star_positions<<<(unsigned)g, TPB, 0, st>>>(hflag, hscan, lflag, lscan, dom_y, hpos, light_y);
    MMJ_CHECK_LAUNCH("k_star_positions");
  }
  return MMJ_OK;
}

int star_operand(int k, const int64_t* dims, const uint8_t* const* heavy, int64_t kpad, int64_t x1_begin,
                 int64_t rows, uint8_t* A, cudaStream_t st) {
  if (k < 2 || k > 4 || kpad % 16 != 0) {
    set_error("star_operand: 2 <= k <= 4 and kpad % 16 == 0 required");
    return MMJ_ERR_ARG;
  }
  StarRels s{};
  s.k = k;
  for (int j = 0; j < k; ++j) {
    s.dims[j] = dims[j];
    s.heavy[j] = heavy[j];
  }
  const int64_t total = rows * (kpad / 16);
  if (total == 0) return MMJ_OK;
  int64_t g = ceil_div(total, TPB);
  if (g > (int64_t)sm_count() * 32) g = (int64_t)sm_count() * 32;
  k_star_operand<<<(unsigned)g, TPB, 0, st>>>(s, kpad, x1_begin, rows, A);
  MMJ_CHECK_LAUNCH("k_star_operand");
  return MMJ_OK;
}

size_t star_light_ws_bytes(int64_t nly) {
  return (size_t)(nly + 1) * 8 * 2 + (size_t)(nly + 1) * 4 + scan_ws_bytes(nly + 1) + 1024;
}

int star_light(int k, const int64_t* dims, const int32_t* const* rev_ptr, const int32_t* const* rev_idx,
               const int32_t* light_y, int64_t nly, int64_t x1_begin, int64_t x1_end, int mode, void* out, int64_t ld,
               unsigned long long* witnesses, void* ws, cudaStream_t st) {
  if (k < 2 || k > 4) {
    set_error("star_light: 2 <= k <= 4 required");
    return MMJ_ERR_ARG;
  }
  if (nly == 0) return MMJ_OK;
  if (ws == nullptr) {
    set_error("star_light: workspace of mmj_star_light_workspace_bytes(n_light) bytes required");
    return MMJ_ERR_ARG;
  }
  StarRels s{};
  s.k = k;
  for (int j = 0; j < k; ++j) {
    s.dims[j] = dims[j];
    s.rev_ptr[j] = rev_ptr[j];
    s.rev_idx[j] = rev_idx[j];
  }
  char* w = static_cast<char*>(ws);
  int64_t* cnt = reinterpret_cast<int64_t*>(w);
  int64_t* offs = cnt + (nly + 1);
  int32_t* start0 = reinterpret_cast<int32_t*>(offs + (nly + 1));
  void* scan_ws = reinterpret_cast<char*>(start0) + (((nly + 1) * 4 + 255) / 256) * 256;
  const int64_t gc = ceil_div(nly, TPB) < (int64_t)sm_count() * 16 ? ceil_div(nly, TPB) : (int64_t)sm_count() * 16;
  k_star_light_count<<<(unsigned)gc, TPB, 0, st>>>(s, light_y, nly, x1_begin, x1_end, cnt, start0);
  MMJ_CHECK_LAUNCH("k_star_light_count");
  MMJ_TRY(scan_i64_i64(cnt, offs, nly, scan_ws, st));
  const int grid = sm_count() * 8;
  k_star_light_expand<<<grid, SL_THREADS, 0, st>>>(s, light_y, nly, offs, start0, x1_begin, mode, out, ld);
  MMJ_CHECK_LAUNCH("k_star_light_expand");
  // witness statistic: the scan total, added on the device
  k_add_total<<<1, 1, 0, st>>>(offs + nly, witnesses);
  MMJ_CHECK_LAUNCH("k_add_total");
  return MMJ_OK;
}

}  // namespace mmj
