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
//   * k_star_light enumerates, one warp per light y, the cross product of the
//     k adjacency lists restricted to the chunk's x1 range and ORs (or counts)
//     each witness into the chunk's bitmap;
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
__global__ void k_star_light(StarRels s, const int32_t* __restrict__ light_y, int64_t nly, int64_t x1_begin,
                             int64_t x1_end, int mode, void* __restrict__ out, int64_t ld,
                             unsigned long long* __restrict__ witnesses) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long mine = 0;
  for (int64_t li = warp_global; li < nly; li += nwarps) {
    const int32_t y = light_y[li];
    const int32_t* lst[4];
    int64_t len[4];
    for (int j = 0; j < s.k; ++j) {
      const int32_t b = s.rev_ptr[j][y];
      lst[j] = s.rev_idx[j] + b;
      len[j] = s.rev_ptr[j][y + 1] - b;
    }
    // x1 list restricted to the chunk (lists are sorted by x)
    const int lo = lb32(lst[0], (int)len[0], (int32_t)x1_begin);
    const int hi = lb32(lst[0], (int)len[0], (int32_t)x1_end);
    lst[0] += lo;
    len[0] = hi - lo;
    int64_t total = 1;
    for (int j = 0; j < s.k; ++j) total *= len[j];
    for (int64_t t = lane; t < total; t += 32) {
      int64_t rem = t;
      int32_t xv[4];
      for (int j = s.k - 1; j >= 0; --j) {
        xv[j] = lst[j][rem % len[j]];
        rem /= len[j];
      }
      int64_t row = xv[0] - x1_begin;
      for (int j = 1; j <= s.k - 2; ++j) row = row * s.dims[j] + xv[j];
      const int32_t col = xv[s.k - 1];
      if (mode == 0)
        atomicOr(reinterpret_cast<uint32_t*>(out) + row * ld + (col >> 5), 1u << (col & 31));
      else
        atomicAdd(reinterpret_cast<int32_t*>(out) + row * ld + col, 1);
    }
    mine += (unsigned long long)total;
  }
  if (lane == 0 && mine) atomicAdd(witnesses, mine);
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

int star_light(int k, const int64_t* dims, const int32_t* const* rev_ptr, const int32_t* const* rev_idx,
               const int32_t* light_y, int64_t nly, int64_t x1_begin, int64_t x1_end, int mode, void* out, int64_t ld,
               unsigned long long* witnesses, cudaStream_t st) {
  if (k < 2 || k > 4) {
    set_error("star_light: 2 <= k <= 4 required");
    return MMJ_ERR_ARG;
  }
  if (nly == 0) return MMJ_OK;
  StarRels s{};
  s.k = k;
  for (int j = 0; j < k; ++j) {
    s.dims[j] = dims[j];
    s.rev_ptr[j] = rev_ptr[j];
    s.rev_idx[j] = rev_idx[j];
  }
  int64_t g = ceil_div(nly * 32, TPB);
  if (g > (int64_t)sm_count() * 16) g = (int64_t)sm_count() * 16;
  k_star_light<<<(unsigned)g, TPB, 0, st>>>(s, light_y, nly, x1_begin, x1_end, mode, out, ld, witnesses);
  MMJ_CHECK_LAUNCH("k_star_light");
  return MMJ_OK;
}

}  // namespace mmj
