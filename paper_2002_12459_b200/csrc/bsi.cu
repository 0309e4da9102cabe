// Batched boolean set intersection (apps.py:314-351, bsi_answer_batch).
//
// The reference answers a batch by filtering R and S to the queried ids and
// running the two-path join on the filtered relations, then probing the
// output.  At cfg5 scale (64M + 64M tuples, 4M queries over a 4M x 4M space)
// a dense product would be 0.25 ppm dense, so the B200 path evaluates the
// "sampled" product instead -- only the queried (a, b) cells:
//   * index build, one pass over each side's forward CSR (k_bsi_records,
//     thread per left id): a record of RECORD_WORDS(words) uint32 (64-byte
//     multiples, so one DRAM access fetches it) holding the H-bit row of the
//     id's heavy y (the H most frequent join values), the base and length of
//     its light list, which is compacted IN PLACE into the id's own CSR span
//     (no scan, no offsets array);
//   * per query (k_bsi_answer): raw ids -> dense ids (direct-address table
//     or binary search; -1 = unknown id = the reference's None), both records
//     loaded together, popc(Rbits & Sbits) > 0 decides whenever a heavy
//     witness exists -- the heavy part of the reference's matrix product
//     with its nonzero test, restricted to queried cells; otherwise the two
//     light lists (sectors prefetched to L1 first) are merge-intersected.
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

// Record of left id x (rec + x * stride uint32): words bitset words (bit
// hpos[y] for every heavy y of x), then [words] = base of x's light list in
// ovf (= fwd_ptr[x]) and [words + 1] = its length; the light y of x are
// written to ovf[fwd_ptr[x] ...] in forward (ascending y) order.
template <int WORDS>
__global__ void __launch_bounds__(TPB) k_bsi_records(const int32_t* __restrict__ fwd_ptr,
                                                     const int32_t* __restrict__ fwd_idx, int64_t dom,
                                                     const int32_t* __restrict__ hpos, int stride,
                                                     uint32_t* __restrict__ rec, int32_t* __restrict__ ovf) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < dom; x += (int64_t)gridDim.x * blockDim.x) {
    uint32_t b[WORDS];
#pragma unroll
    for (int w = 0; w < WORDS; ++w) b[w] = 0u;
    const int32_t p0 = fwd_ptr[x], p1 = fwd_ptr[x + 1];
    int32_t k = p0;
    for (int32_t p = p0; p < p1; ++p) {
      const int32_t y = fwd_idx[p];
      const int32_t h = hpos[y];
      if (h >= 0) {
        const uint32_t m = 1u << (h & 31);
#pragma unroll
        for (int w = 0; w < WORDS; ++w) b[w] |= ((h >> 5) == w) ? m : 0u;
      } else {
        ovf[k++] = y;
      }
    }
    uint32_t* r = rec + x * (int64_t)stride;
#pragma unroll
    for (int w = 0; w < WORDS; w += 4) *reinterpret_cast<uint4*>(r + w) = make_uint4(b[w], b[w + 1], b[w + 2], b[w + 3]);
    *reinterpret_cast<uint2*>(r + WORDS) = make_uint2((uint32_t)p0, (uint32_t)(k - p0));
  }
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

// L2 eviction-priority hints for the lists form: the id tables and list
// offsets (4 x 16 MB at cfg5, every 64-byte granule read ~16 times per batch)
// are kept (evict_last) while the lists themselves (each read about once)
// stream through (evict_first) -- otherwise the lists push the tables out and
// every 4-byte table / offset read costs a DRAM granule.
__device__ __forceinline__ uint64_t l2_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_stream() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ld_pol(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t map_id_pol(const IdMap& m, int64_t v, uint64_t pol) {
  if (m.table) {
    const int64_t o = v - m.vmin;
    return (o >= 0 && o < m.range) ? ld_pol(m.table + o, pol) : -1;
  }
  return m.sorted ? lookup(m.sorted, m.order, m.n, v) : (int32_t)v;
}

struct BsiSideArgs {
  IdMap map;
  const uint32_t* rec;
  const int32_t* ovf;
};

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <int WORDS>
__global__ void __launch_bounds__(TPB) k_bsi_answer(const int64_t* __restrict__ qa, const int64_t* __restrict__ qb,
                                                    int64_t nq, const BsiSideArgs ra, const BsiSideArgs sb, int stride,
                                                    int8_t* __restrict__ ans) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t ia = map_id(ra.map, qa[q]);
    const int32_t ib = map_id(sb.map, qb[q]);
    if (ia < 0 || ib < 0) {
      ans[q] = -1;
      continue;
    }
    const uint32_t* pa = ra.rec + (int64_t)ia * stride;
    const uint32_t* pb = sb.rec + (int64_t)ib * stride;
    // both records' bit rows and list headers in flight together
    uint4 xa[WORDS / 4], xb[WORDS / 4];
#pragma unroll
    for (int w = 0; w < WORDS / 4; ++w) {
      xa[w] = __ldg(reinterpret_cast<const uint4*>(pa) + w);
      xb[w] = __ldg(reinterpret_cast<const uint4*>(pb) + w);
    }
    const uint2 ha = __ldg(reinterpret_cast<const uint2*>(pa + WORDS));
    const uint2 hb = __ldg(reinterpret_cast<const uint2*>(pb + WORDS));
    uint32_t any = 0u;
#pragma unroll
    for (int w = 0; w < WORDS / 4; ++w)
      any |= (xa[w].x & xb[w].x) | (xa[w].y & xb[w].y) | (xa[w].z & xb[w].z) | (xa[w].w & xb[w].w);
    bool hit = any != 0u;
    if (!hit && ha.y && hb.y) {
      const int32_t* la = ra.ovf + ha.x;
      const int32_t* lb = sb.ovf + hb.x;
      const int32_t na = (int32_t)ha.y, nb = (int32_t)hb.y;
      // every 32-byte sector of both lists requested before the (dependent) merge
      for (int32_t i = 0; i < na; i += 8) prefetch_l1(la + i);
      for (int32_t j = 0; j < nb; j += 8) prefetch_l1(lb + j);
      prefetch_l1(la + na - 1);
      prefetch_l1(lb + nb - 1);
      int32_t i = 0, j = 0;
      int32_t u = la[0], v = lb[0];
      while (true) {
        if (u == v) {
          hit = true;
          break;
        }
        if (u < v) {
          if (++i == na) break;
          u = la[i];
        } else {
          if (++j == nb) break;
          v = lb[j];
        }
      }
    }
    ans[q] = hit ? 1 : 0;
  }
}

// ---- "lists" form: warp-cooperative intersection of the forward lists ------
// Both lists of a query are sorted by the shared y id, so the index IS the
// relations' CSR and nothing is built per batch.  Taken when the lists are
// short (cfg5: 16 y per id on average), where a bitset record (64 B) costs as
// many DRAM granules as the list itself.
//
// A warp takes 32 queries: every lane resolves its own query's two list spans
// (the table loads of 32 queries in flight together), then the warp walks the
// queries, PIPE at a time: lane l loads element l of each list (one coalesced
// request per list, every sector fetched once, straight into registers), and
// the two 32-entry chunks are intersected by a shuffle binary search (5
// steps) + ballot.  Lists longer than 32 take a chunked merge.  cfg5, 4M
// queries: 0.41 ms at PIPE = 2 (r3d/r3e; PIPE = 1 / 3 / 4 / 8: 0.46 / 0.48 /
// 0.47 / 0.54 ms -- occupancy beats a deeper pipeline) against 0.48 ms for the
// thread-per-query merge it replaces (r3b; 0.64 ms before the span tables).
// It is issue-bound (r3f ncu: 76 warp instructions per query, issue slots 71%
// busy, DRAM 40%); __match_any_sync over both lists in one register row
// (na + nb <= 32) was slower (0.67 ms, r3h), as was staging 64-byte aligned
// list copies in shared memory by cp.async and merging per lane (0.44, r3g).
//
// Raw id -> list, three ways per side (ListSide):
//   * span table (mmj_bsi_span_table): table[raw - vmin] = {(offset <<
//     len_bits) | min(length, 2^len_bits - 1), signature}, the first word
//     0xFFFFFFFF for an id the relation does not hold -- one 8-byte load
//     instead of the id table -> fwd_ptr[id], fwd_ptr[id + 1] chain (two more
//     DRAM granules per side); a saturated length field sends the query to a
//     binary search of its offset in fwd_ptr.  The signature holds one bit
//     per heaviest join value (up to 32, chosen by the caller): two ids with
//     a common bit intersect, so that query never touches the lists -- the
//     heavy part of the reference's product with its nonzero test
//     (joinproject.py:208-216), restricted to the queried cells;
//   * direct id table or binary search over the sorted raw ids, then fwd_ptr;
//   * dense ids already (map all null).
struct ListSide {
  IdMap map;                // raw id -> dense id (when span == nullptr)
  const uint2* span;        // raw id -> {packed (offset, length), heavy-y signature}, or nullptr
  int64_t vmin, range;      // span table window
  int len_bits;             // length bits of a span entry
  const int32_t* fwd_ptr;   // dom + 1 CSR offsets (searched when a span's length saturates)
  int64_t dom;
  const int32_t* lists;     // fwd_idx
};

__device__ __forceinline__ uint2 ld_pol_u32x2(const uint2* p, uint64_t pol) {
  uint2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.b32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}

// (first entry index in s.lists, length) of raw id v's list; length -1 for an
// unknown id; sig = the id's heavy-y signature (0 without a span table)
__device__ __forceinline__ int2 resolve_list(const ListSide& s, int64_t v, uint64_t keep, uint32_t& sig) {
  sig = 0u;
  if (s.span) {
    const int64_t o = v - s.vmin;
    if (o < 0 || o >= s.range) return make_int2(0, -1);
    const uint2 es = ld_pol_u32x2(s.span + o, keep);
    const uint32_t e = es.x;
    if (e == 0xFFFFFFFFu) return make_int2(0, -1);
    sig = es.y;
    const uint32_t cap = (1u << s.len_bits) - 1u;
    const int32_t off = (int32_t)(e >> s.len_bits);
    int32_t len = (int32_t)(e & cap);
    if (len == (int32_t)cap) {
      // saturated: the (non-empty) list's id is the last i with fwd_ptr[i] <= off
      int64_t lo = 0, hi = s.dom;          // answer in [lo, hi)
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(s.fwd_ptr + mid) <= off) lo = mid;
        else hi = mid;
      }
      len = __ldg(s.fwd_ptr + lo + 1) - off;
      MMJ_DCHECK(__ldg(s.fwd_ptr + lo) == off && len >= (int32_t)cap, "span escape");
    }
    return make_int2(off, len);
  }
  const int32_t id = map_id_pol(s.map, v, keep);
  if (id < 0) return make_int2(0, -1);
  const int32_t p0 = ld_pol(s.fwd_ptr + id, keep), p1 = ld_pol(s.fwd_ptr + id + 1, keep);
  MMJ_DCHECK(p0 >= 0 && p1 >= p0, "list bounds");
  return make_int2(p0, p1 - p0);
}

constexpr int32_t PAD_Y = 0x7FFFFFFF;   // beyond every y id (dom_y < 2^31 - 1)
constexpr unsigned FULL = 0xFFFFFFFFu;

// does any of the first ca values of `a` (one per lane) occur among the first
// cb values of `b` (ascending, padded with PAD_Y)?  warp-uniform result
__device__ __forceinline__ bool chunk_match(int32_t a, int32_t b, int ca, int cb, int lane) {
  int lo = 0;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int32_t v = __shfl_sync(FULL, b, lo + s - 1);
    if (v < a) lo += s;
  }
  const int32_t v = __shfl_sync(FULL, b, lo);
  return __any_sync(FULL, lane < ca && lo < cb && v == a);
}

// lists of any length, 32-entry chunks of each side; the chunk with the
// smaller last value advances
__device__ __noinline__ bool long_intersect(const int32_t* __restrict__ la, int na, const int32_t* __restrict__ lb,
                                            int nb, int lane) {
  int ia = 0, ib = 0;
  int32_t a = lane < na ? __ldg(la + lane) : PAD_Y;
  int32_t b = lane < nb ? __ldg(lb + lane) : PAD_Y;
  while (true) {
    const int ca = min(32, na - ia), cb = min(32, nb - ib);
    if (chunk_match(a, b, ca, cb, lane)) return true;
    const int32_t amax = __shfl_sync(FULL, a, ca - 1), bmax = __shfl_sync(FULL, b, cb - 1);
    if (amax <= bmax) {
      ia += ca;
      if (ia >= na) return false;
      a = ia + lane < na ? __ldg(la + ia + lane) : PAD_Y;
    }
    if (bmax <= amax) {
      ib += cb;
      if (ib >= nb) return false;
      b = ib + lane < nb ? __ldg(lb + ib + lane) : PAD_Y;
    }
  }
}

constexpr int PIPE = 2;   // queries whose list loads are in flight together per warp

__global__ void __launch_bounds__(TPB) k_bsi_answer_lists(const int64_t* __restrict__ qa,
                                                          const int64_t* __restrict__ qb, int64_t nq,
                                                          const ListSide sa, const ListSide sb,
                                                          int8_t* __restrict__ ans) {
  // L2 hints: tables and offsets are re-read across the batch (evict_last),
  // the lists are read about once (evict_first)
  const uint64_t keep = l2_keep(), stream = l2_stream();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 32; base < nq; base += nwarps * 32) {
    const int64_t q = base + lane;
    int2 ra = make_int2(0, -1), rb = make_int2(0, -1);
    uint32_t ga = 0u, gb = 0u;
    if (q < nq) {
      ra = resolve_list(sa, __ldcs(qa + q), keep, ga);
      rb = resolve_list(sb, __ldcs(qb + q), keep, gb);
    }
    // a shared signature bit is a shared heavy y: answered without the lists
    const bool heavy_hit = (ga & gb) != 0u;
    int res = (ra.y < 0 || rb.y < 0) ? -1 : (heavy_hit ? 1 : 0);
    unsigned todo = __ballot_sync(FULL, ra.y > 0 && rb.y > 0 && !heavy_hit);
    while (todo) {
      int j[PIPE], na[PIPE], nb[PIPE], oa[PIPE], ob[PIPE];
      int32_t a[PIPE], b[PIPE];
#pragma unroll
      for (int p = 0; p < PIPE; ++p) {
        j[p] = todo ? __ffs(todo) - 1 : -1;
        todo &= todo - 1;            // 0 stays 0
        const int src = j[p] & 31;
        oa[p] = __shfl_sync(FULL, ra.x, src);
        na[p] = j[p] >= 0 ? __shfl_sync(FULL, ra.y, src) : 0;
        ob[p] = __shfl_sync(FULL, rb.x, src);
        nb[p] = j[p] >= 0 ? __shfl_sync(FULL, rb.y, src) : 0;
        a[p] = lane < na[p] ? ld_pol(sa.lists + oa[p] + lane, stream) : PAD_Y;
        b[p] = lane < nb[p] ? ld_pol(sb.lists + ob[p] + lane, stream) : PAD_Y;
      }
#pragma unroll
      for (int p = 0; p < PIPE; ++p) {
        if (j[p] < 0) continue;      // warp-uniform
        bool hit;
        if (na[p] <= 32 && nb[p] <= 32) hit = chunk_match(a[p], b[p], na[p], nb[p], lane);
        else hit = long_intersect(sa.lists + oa[p], na[p], sb.lists + ob[p], nb[p], lane);
        if (lane == j[p]) res = hit ? 1 : 0;
      }
    }
    if (q < nq) ans[q] = (int8_t)res;
  }
}

// span entry of every held raw id: {(fwd_ptr[dense] << len_bits) | min(length,
// cap), signature}: signature bit hpos[y] for each of the id's y with 0 <=
// hpos[y] < 32 (the heaviest join values: at cfg5's Zipf(1.0) the top 32 y
// decide 63% of the queries -- 98% of the intersecting pairs -- from the
// two table entries alone)
__global__ void k_span_table(const int64_t* __restrict__ sorted, const int32_t* __restrict__ order, int64_t n,
                             int64_t vmin, int64_t range, const int32_t* __restrict__ fwd_ptr,
                             const int32_t* __restrict__ fwd_idx, const int32_t* __restrict__ hpos, int len_bits,
                             uint2* __restrict__ table) {
  const uint32_t cap = (1u << len_bits) - 1u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = sorted[i] - vmin;
    if (o < 0 || o >= range) continue;
    const int32_t d = order[i];
    const int32_t p0 = fwd_ptr[d], p1 = fwd_ptr[d + 1];
    const uint32_t off = (uint32_t)p0, len = (uint32_t)(p1 - p0);
    uint32_t sig = 0u;
    if (hpos != nullptr)
      for (int32_t p = p0; p < p1; ++p) {
        const int32_t h = __ldg(hpos + __ldg(fwd_idx + p));
        if (h >= 0 && h < 32) sig |= 1u << h;
      }
    table[o] = make_uint2((off << len_bits) | (len < cap ? len : cap), sig);
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

int bsi_record_words(int words) { return (int)round_up(words + 2, 16); }

int bsi_records(const int32_t* fwd_ptr, const int32_t* fwd_idx, int64_t dom, const int32_t* hpos, int words,
                uint32_t* rec, int32_t* ovf, cudaStream_t st) {
  if (dom == 0) return MMJ_OK;
  const int stride = bsi_record_words(words);
  const int g = grid_for(dom);
  switch (words) {
    case 4: k_bsi_records<4><<<g, TPB, 0, st>>>(fwd_ptr, fwd_idx, dom, hpos, stride, rec, ovf); break;
    case 8: k_bsi_records<8><<<g, TPB, 0, st>>>(fwd_ptr, fwd_idx, dom, hpos, stride, rec, ovf); break;
    case 16: k_bsi_records<16><<<g, TPB, 0, st>>>(fwd_ptr, fwd_idx, dom, hpos, stride, rec, ovf); break;
    case 32: k_bsi_records<32><<<g, TPB, 0, st>>>(fwd_ptr, fwd_idx, dom, hpos, stride, rec, ovf); break;
    default:
      set_error("bsi_records: words must be 4, 8, 16 or 32 (128 .. 1024 heavy bits)");
      return MMJ_ERR_ARG;
  }
  MMJ_CHECK_LAUNCH("k_bsi_records");
  return MMJ_OK;
}

int bsi_answer(const int64_t* qa, const int64_t* qb, int64_t nq, const int64_t* r_sorted, const int32_t* r_order,
               int64_t r_n, const int32_t* r_table, int64_t r_min, int64_t r_range, const int64_t* s_sorted,
               const int32_t* s_order, int64_t s_n, const int32_t* s_table, int64_t s_min, int64_t s_range,
               const uint32_t* r_rec, const int32_t* r_ovf, const uint32_t* s_rec, const int32_t* s_ovf, int words,
               int8_t* ans, cudaStream_t st) {
  if (words != 4 && words != 8 && words != 16 && words != 32) {
    set_error("bsi_answer: words must be 4, 8, 16 or 32 (128 .. 1024 heavy bits)");
    return MMJ_ERR_ARG;
  }
  if (nq == 0) return MMJ_OK;
  const BsiSideArgs a{IdMap{r_sorted, r_order, r_n, r_table, r_min, r_range}, r_rec, r_ovf};
  const BsiSideArgs b{IdMap{s_sorted, s_order, s_n, s_table, s_min, s_range}, s_rec, s_ovf};
  const int stride = bsi_record_words(words);
  const int g = grid_for(nq, TPB, 16);
  switch (words) {
    case 4: k_bsi_answer<4><<<g, TPB, 0, st>>>(qa, qb, nq, a, b, stride, ans); break;
    case 8: k_bsi_answer<8><<<g, TPB, 0, st>>>(qa, qb, nq, a, b, stride, ans); break;
    case 16: k_bsi_answer<16><<<g, TPB, 0, st>>>(qa, qb, nq, a, b, stride, ans); break;
    default: k_bsi_answer<32><<<g, TPB, 0, st>>>(qa, qb, nq, a, b, stride, ans); break;
  }
  MMJ_CHECK_LAUNCH("k_bsi_answer");
  return MMJ_OK;
}

static int launch_answer_lists(const int64_t* qa, const int64_t* qb, int64_t nq, const ListSide& a,
                               const ListSide& b, int8_t* ans, cudaStream_t st) {
  // a warp per 32 queries, 16 waves of resident CTAs at most
  k_bsi_answer_lists<<<grid_for(nq, TPB, 16), TPB, 0, st>>>(qa, qb, nq, a, b, ans);
  MMJ_CHECK_LAUNCH("k_bsi_answer_lists");
  return MMJ_OK;
}

int bsi_answer_lists(const int64_t* qa, const int64_t* qb, int64_t nq, const int64_t* r_sorted,
                     const int32_t* r_order, int64_t r_n, const int32_t* r_table, int64_t r_min, int64_t r_range,
                     const int64_t* s_sorted, const int32_t* s_order, int64_t s_n, const int32_t* s_table,
                     int64_t s_min, int64_t s_range, const int32_t* r_fwd_ptr, const int32_t* r_fwd_idx,
                     const int32_t* s_fwd_ptr, const int32_t* s_fwd_idx, int8_t* ans, cudaStream_t st) {
  if (nq == 0) return MMJ_OK;
  if (r_fwd_ptr == nullptr || s_fwd_ptr == nullptr) {
    set_error("bsi_answer_lists: both forward CSRs are required");
    return MMJ_ERR_ARG;
  }
  const ListSide a{IdMap{r_sorted, r_order, r_n, r_table, r_min, r_range}, nullptr, 0, 0, 0, r_fwd_ptr, 0, r_fwd_idx};
  const ListSide b{IdMap{s_sorted, s_order, s_n, s_table, s_min, s_range}, nullptr, 0, 0, 0, s_fwd_ptr, 0, s_fwd_idx};
  return launch_answer_lists(qa, qb, nq, a, b, ans, st);
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

int bsi_span_table(const int64_t* sorted, const int32_t* order, int64_t n, int64_t vmin, int64_t range,
                   const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* hpos, int64_t n_tuples,
                   int len_bits, uint2* table, cudaStream_t st) {
  if (range <= 0 || range >= (1ll << 31)) {
    set_error("bsi_span_table: range %lld out of (0, 2^31)", (long long)range);
    return MMJ_ERR_ARG;
  }
  if (len_bits < 1 || len_bits > 16 || n_tuples < 0 || n_tuples >= (1ll << (32 - len_bits)) - 1) {
    set_error("bsi_span_table: %lld tuples do not leave %d length bits in a 32-bit span", (long long)n_tuples,
              len_bits);
    return MMJ_ERR_ARG;
  }
  MMJ_TRY(cuda_status(cudaMemsetAsync(table, 0xFF, (size_t)range * 8, st), "memset span table"));
  if (n == 0) return MMJ_OK;
  k_span_table<<<grid_for(n), TPB, 0, st>>>(sorted, order, n, vmin, range, fwd_ptr, fwd_idx, hpos, len_bits, table);
  MMJ_CHECK_LAUNCH("k_span_table");
  return MMJ_OK;
}

int bsi_answer_spans(const int64_t* qa, const int64_t* qb, int64_t nq, const uint2* r_span, int64_t r_min,
                     int64_t r_range, int r_len_bits, const int32_t* r_fwd_ptr, int64_t r_dom,
                     const int32_t* r_fwd_idx, const uint2* s_span, int64_t s_min, int64_t s_range, int s_len_bits,
                     const int32_t* s_fwd_ptr, int64_t s_dom, const int32_t* s_fwd_idx, int8_t* ans,
                     cudaStream_t st) {
  if (nq == 0) return MMJ_OK;
  if (!r_span || !s_span || !r_fwd_ptr || !s_fwd_ptr || r_len_bits < 1 || r_len_bits > 16 || s_len_bits < 1 ||
      s_len_bits > 16) {
    set_error("bsi_answer_spans: both span tables (1..16 length bits) and forward CSRs are required");
    return MMJ_ERR_ARG;
  }
  const ListSide a{IdMap{}, r_span, r_min, r_range, r_len_bits, r_fwd_ptr, r_dom, r_fwd_idx};
  const ListSide b{IdMap{}, s_span, s_min, s_range, s_len_bits, s_fwd_ptr, s_dom, s_fwd_idx};
  return launch_answer_lists(qa, qb, nq, a, b, ans, st);
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
