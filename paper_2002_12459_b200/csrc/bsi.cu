// Batched boolean set intersection (apps.py:314-351, bsi_answer_batch).
//
// The reference answers a batch by filtering R and S to the queried ids and
// running the two-path join on the filtered relations, then probing the
// output.  At cfg5 scale (64M + 64M tuples, 4M queries over a 4M x 4M space)
// a dense product would be 0.25 ppm dense, so the B200 path evaluates the
// "sampled" product instead -- only the queried (a, b) cells:
//   * heavy y (the H most frequent join values) become H-bit rows per left
//     id (Rbits[a], Sbits[b]); a query is decided by popc(Rbits & Sbits) > 0
//     whenever a heavy witness exists -- the heavy part of the reference's
//     matrix product with its nonzero test, restricted to queried cells;
//   * otherwise the light lists (each left id's y list without heavy y, in
//     y order) are merge-intersected;
//   * raw query ids are resolved against each relation's own dictionary on
//     device (binary search over the sorted raw values); an id unknown to
//     the unreduced relation answers -1 (the reference's None marker).
#include "mmj_common.cuh"

namespace mmj {
namespace {

constexpr int TPB = 256;

inline int grid_for(int64_t n, int per = TPB, int waves = 32) {
  int64_t g = ceil_div(n, per);
  const int64_t cap = (int64_t)sm_count() * waves;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

// bits[left * words + hpos[y] / 32] |= bit, for every tuple (left, y) with heavy y
__global__ void k_bsi_bits(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols, int64_t n,
                           const int32_t* __restrict__ hpos, int words, uint32_t* __restrict__ bits) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t h = hpos[cols[t]];
    if (h >= 0) atomicOr(&bits[(int64_t)rows[t] * words + (h >> 5)], 1u << (h & 31));
  }
}

__global__ void k_bsi_light_flags(const int32_t* __restrict__ cols, int64_t n, const int32_t* __restrict__ hpos,
                                  uint8_t* __restrict__ flag) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    flag[t] = hpos[cols[t]] < 0 ? 1 : 0;
}

__global__ void k_bsi_light_scatter(const int32_t* __restrict__ cols, const uint8_t* __restrict__ flag,
                                    const int32_t* __restrict__ pos, int64_t n, int32_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    if (flag[t]) out[pos[t]] = cols[t];
}

__global__ void k_bsi_light_ptr(const int32_t* __restrict__ ptr, const int32_t* __restrict__ pos, int64_t dom,
                                int32_t* __restrict__ lptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= dom; i += (int64_t)gridDim.x * blockDim.x)
    lptr[i] = pos[ptr[i]];
}

__device__ __forceinline__ int32_t lookup(const int64_t* __restrict__ sorted, const int32_t* __restrict__ order,
                                          int64_t n, int64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && sorted[lo] == key) ? order[lo] : -1;
}

struct BsiArgs {
  const int64_t* qa;            // raw query ids (or dense ids when sorted == nullptr)
  const int64_t* qb;
  int64_t nq;
  const int64_t* r_sorted;      // sorted raw left values of R and their dense ids
  const int32_t* r_order;
  int64_t r_n;
  const int64_t* s_sorted;
  const int32_t* s_order;
  int64_t s_n;
  const uint32_t* r_bits;       // [dom_R x words]
  const uint32_t* s_bits;
  int words;
  const int32_t* r_lptr;        // light lists (y ids ascending)
  const int32_t* r_lidx;
  const int32_t* s_lptr;
  const int32_t* s_lidx;
  int8_t* ans;
};

// raw id -> dense id: binary search over the sorted raw values, or one load
// from a direct-address table (dense_of[raw - vmin], -1 = unknown id)
struct IdMap {
  const int64_t* sorted;
  const int32_t* order;
  int64_t n;
  const int32_t* table;
  int64_t vmin, range;
};

__device__ __forceinline__ int32_t map_id(const IdMap& m, int64_t v) {
  if (m.table) {
    const int64_t o = v - m.vmin;
    return (o >= 0 && o < m.range) ? __ldg(m.table + o) : -1;
  }
  return m.sorted ? lookup(m.sorted, m.order, m.n, v) : (int32_t)v;
}

__global__ void k_bsi_answer(const BsiArgs a, const IdMap ma, const IdMap mb) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.nq; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t ia = map_id(ma, a.qa[q]);
    const int32_t ib = map_id(mb, a.qb[q]);
    if (ia < 0 || ib < 0) {
      a.ans[q] = -1;
      continue;
    }
    bool hit = false;
    const uint32_t* ra = a.r_bits + (int64_t)ia * a.words;
    const uint32_t* sb = a.s_bits + (int64_t)ib * a.words;
    for (int w = 0; w < a.words && !hit; w += 4) {
      const uint4 x = *reinterpret_cast<const uint4*>(ra + w);
      const uint4 y = *reinterpret_cast<const uint4*>(sb + w);
      hit = ((x.x & y.x) | (x.y & y.y) | (x.z & y.z) | (x.w & y.w)) != 0u;
    }
    if (!hit) {
      int32_t i = a.r_lptr[ia], ie = a.r_lptr[ia + 1];
      int32_t j = a.s_lptr[ib], je = a.s_lptr[ib + 1];
      while (i < ie && j < je) {
        const int32_t u = a.r_lidx[i], v = a.s_lidx[j];
        if (u == v) {
          hit = true;
          break;
        }
        if (u < v) ++i;
        else ++j;
      }
    }
    a.ans[q] = hit ? 1 : 0;
  }
}

__global__ void k_direct_table(const int64_t* __restrict__ sorted, const int32_t* __restrict__ order, int64_t n,
                               int64_t vmin, int64_t range, int32_t* __restrict__ table) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = sorted[i] - vmin;
    if (o >= 0 && o < range) table[o] = order[i];
  }
}

}  // namespace

// histogram of m(y) = max(rdeg[y], sdeg[y]) over y with m > 0: log2 bins
// (bin b holds m in [2^b, 2^(b+1))) or nbins linear bins over [lo, hi)
__global__ void k_bsi_deg_hist(const int32_t* __restrict__ rdeg, const int32_t* __restrict__ sdeg, int64_t dom_y,
                               int64_t lo, int64_t hi, int nbins, int log2mode, int32_t* __restrict__ hist) {
  __shared__ int32_t sh[1024];
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y < dom_y; y += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = max(rdeg[y], sdeg[y]);
    if (m <= 0) continue;
    if (log2mode) {
      atomicAdd(&sh[63 - __clzll((unsigned long long)m)], 1);
    } else if (m >= lo && m < hi) {
      atomicAdd(&sh[(int)((m - lo) * nbins / (hi - lo))], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nbins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

int bsi_bits(const int32_t* rows, const int32_t* cols, int64_t n, const int32_t* hpos, int words, uint32_t* bits,
             int64_t dom, cudaStream_t st) {
  MMJ_TRY(cuda_status(cudaMemsetAsync(bits, 0, (size_t)dom * words * 4, st), "memset bits"));
  if (n == 0) return MMJ_OK;
  k_bsi_bits<<<grid_for(n), TPB, 0, st>>>(rows, cols, n, hpos, words, bits);
  MMJ_CHECK_LAUNCH("k_bsi_bits");
  return MMJ_OK;
}

int bsi_light_lists(const int32_t* ptr, const int32_t* cols, int64_t n, int64_t dom, const int32_t* hpos,
                    uint8_t* flag_ws, int32_t* pos_ws, int32_t* lptr, int32_t* lidx, void* ws, cudaStream_t st) {
  if (n > 0) {
    k_bsi_light_flags<<<grid_for(n), TPB, 0, st>>>(cols, n, hpos, flag_ws);
    MMJ_CHECK_LAUNCH("k_bsi_light_flags");
  }
  MMJ_TRY(scan_u8_i32(flag_ws, pos_ws, n, ws, st));
  if (n > 0) {
    k_bsi_light_scatter<<<grid_for(n), TPB, 0, st>>>(cols, flag_ws, pos_ws, n, lidx);
    MMJ_CHECK_LAUNCH("k_bsi_light_scatter");
  }
  k_bsi_light_ptr<<<grid_for(dom + 1), TPB, 0, st>>>(ptr, pos_ws, dom, lptr);
  MMJ_CHECK_LAUNCH("k_bsi_light_ptr");
  return MMJ_OK;
}

int bsi_answer(const int64_t* qa, const int64_t* qb, int64_t nq, const int64_t* r_sorted, const int32_t* r_order,
               int64_t r_n, const int64_t* s_sorted, const int32_t* s_order, int64_t s_n, const uint32_t* r_bits,
               const uint32_t* s_bits, int words, const int32_t* r_lptr, const int32_t* r_lidx,
               const int32_t* s_lptr, const int32_t* s_lidx, int8_t* ans, const int32_t* r_table, int64_t r_min,
               int64_t r_range, const int32_t* s_table, int64_t s_min, int64_t s_range, cudaStream_t st) {
  if (words % 4 != 0 || words <= 0) {
    set_error("bsi_answer: bitset words must be a positive multiple of 4");
    return MMJ_ERR_ARG;
  }
  if (nq == 0) return MMJ_OK;
  BsiArgs a{qa, qb, nq, r_sorted, r_order, r_n, s_sorted, s_order, s_n, r_bits, s_bits, words,
            r_lptr, r_lidx, s_lptr, s_lidx, ans};
  const IdMap ma{r_sorted, r_order, r_n, r_table, r_min, r_range};
  const IdMap mb{s_sorted, s_order, s_n, s_table, s_min, s_range};
  k_bsi_answer<<<grid_for(nq, TPB, 16), TPB, 0, st>>>(a, ma, mb);
  MMJ_CHECK_LAUNCH("k_bsi_answer");
  return MMJ_OK;
}

int bsi_direct_table(const int64_t* sorted, const int32_t* order, int64_t n, int64_t vmin, int64_t range,
                     int32_t* table, cudaStream_t st) {
  if (range <= 0 || range >= (1ll << 31)) {
    set_error("bsi_direct_table: range %lld out of (0, 2^31)", (long long)range);
    return MMJ_ERR_ARG;
  }
  MMJ_TRY(cuda_status(cudaMemsetAsync(table, 0xFF, (size_t)range * 4, st), "memset direct table"));
  if (n == 0) return MMJ_OK;
  k_direct_table<<<grid_for(n), TPB, 0, st>>>(sorted, order, n, vmin, range, table);
  MMJ_CHECK_LAUNCH("k_direct_table");
  return MMJ_OK;
}

int bsi_degree_histogram(const int32_t* rdeg, const int32_t* sdeg, int64_t dom_y, int64_t lo, int64_t hi, int nbins,
                         int log2mode, int32_t* hist, cudaStream_t st) {
  if (nbins < 1 || nbins > 1024 || (!log2mode && hi <= lo) || (log2mode && nbins < 64)) {
    set_error("bsi_degree_histogram: 1 <= nbins <= 1024 (64 for log2 bins), lo < hi");
    return MMJ_ERR_ARG;
  }
  MMJ_TRY(cuda_status(cudaMemsetAsync(hist, 0, (size_t)nbins * 4, st), "memset hist"));
  if (dom_y == 0) return MMJ_OK;
  int64_t g = ceil_div(dom_y, TPB);
  if (g > (int64_t)sm_count() * 4) g = (int64_t)sm_count() * 4;
  k_bsi_deg_hist<<<(unsigned)g, TPB, 0, st>>>(rdeg, sdeg, dom_y, lo, hi, nbins, log2mode, hist);
  MMJ_CHECK_LAUNCH("k_bsi_deg_hist");
  return MMJ_OK;
}

}  // namespace mmj
