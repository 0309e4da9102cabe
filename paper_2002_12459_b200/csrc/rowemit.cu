// Fused light expansion + merge + emission, one row group per CTA.
//
// Replaces, for the projection (no counts) two-path path, the light passes
// (joinproject.py:183-203) and the np.unique merge (joinproject.py:220-225):
//   1. the heavy product's bitmap rows of the group are copied into shared
//      memory (or zeroed when there is no heavy part);
//   2. every light witness (x, z) of the group's rows -- R tuples of those x,
//      each expanding its S-side list exactly as the reference's three
//      witness-disjoint passes do -- is OR-ed into the shared bitmap with a
//      shared-memory atomic (no global atomics, no materialised keys);
//   3. per-32-word segment popcounts are block-scanned, the group's global
//      output offset comes from a single-pass decoupled look-back over the
//      groups (tickets taken in order, so predecessors are always resident);
//   4. each warp stages a segment's codes x*dom_z + z in shared memory and
//      writes them with coalesced 16-byte streaming stores.
// The bitmap is read once, every code is written once: the kernel is bound by
// the HBM write of the sorted output (8 B per distinct (x, z)).
#include <cub/block/block_scan.cuh>

#include "mmj_common.cuh"

namespace mmj {
namespace {

constexpr int RE_THREADS = 512;
constexpr int RE_WARPS = RE_THREADS / 32;
constexpr int TUP_BATCH = RE_THREADS;   // light tuples staged per round
constexpr int STAGE = 1024 + 64;        // codes staged per warp (one segment max) + bank padding

// staging slot of the k-th code of a segment: one pad slot per 16 codes.
// Lanes start ~16 codes apart (a 49%-dense word has ~16 set bits), so an
// unpadded layout puts every lane's k-th store in the same bank.
__device__ __forceinline__ int stage_slot(int k) { return k + (k >> 4); }

constexpr unsigned long long FLAG_AGG = 1ull << 62;
constexpr unsigned long long FLAG_INC = 2ull << 62;
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

struct RowEmitArgs {
  const uint32_t* heavy_bm;   // rows x wpr words of the chunk (nullptr: no heavy part)
  int64_t x0, rows, wpr, dom_z;
  int G;                      // rows per group
  int64_t ngroups;
  const int32_t* fwd_ptr;     // R forward CSR (x -> tuples)
  const int32_t* fwd_idx;
  const int32_t* rdeg_x;
  int64_t d2;
  const int32_t* hpos;        // nullptr: FULL_JOIN (every y light)
  const int32_t* s_rev_ptr;
  const int32_t* s_rev_idx;
  const int32_t* lz_ptr;
  const int32_t* lz_idx;
  int64_t* codes;
  unsigned long long* status;          // per group look-back word (zeroed)
  int* ticket;                         // zeroed
  unsigned long long* witnesses;       // += light witnesses processed
  unsigned long long* total;           // chunk size (written by the last group)
};

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_stream_v2(int64_t* p, int64_t a, int64_t b) {
  asm volatile("st.global.cs.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_stream(int64_t* p, int64_t a) {
  asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}

__global__ void __launch_bounds__(RE_THREADS, 1) k_row_light_emit(const RowEmitArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  using BScan = cub::BlockScan<int, RE_THREADS>;
  __shared__ typename BScan::TempStorage scan_tmp;
  __shared__ int s_group;
  __shared__ long long s_prefix;
  __shared__ int s_tb_len[TUP_BATCH + 1];      // exclusive prefix of list lengths
  __shared__ const int32_t* s_tb_base[TUP_BATCH];
  __shared__ int s_tb_row[TUP_BATCH];
  __shared__ int s_carry;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t gw = (int64_t)a.G * a.wpr;            // words per group
  uint32_t* sbm = reinterpret_cast<uint32_t*>(smem);  // gw words
  int64_t* stage = reinterpret_cast<int64_t*>(smem + ((gw * 4 + 15) & ~15ll)) + warp * STAGE;
  int* segcnt = reinterpret_cast<int*>(smem + ((gw * 4 + 15) & ~15ll) + (size_t)RE_WARPS * STAGE * 8);
  const int nseg = (int)((gw + 31) / 32);

  if (tid == 0) s_group = atomicAdd(a.ticket, 1);
  __syncthreads();
  const int64_t g = s_group;
  const int64_t r0 = g * a.G;
  const int64_t r1 = min(r0 + (int64_t)a.G, a.rows);
  const int64_t words = (r1 - r0) * a.wpr;

  // ---- 1. heavy rows -> shared bitmap
  if (a.heavy_bm != nullptr) {
    const uint4* src = reinterpret_cast<const uint4*>(a.heavy_bm + r0 * a.wpr);
    uint4* dst = reinterpret_cast<uint4*>(sbm);
    for (int64_t i = tid; i < words / 4; i += RE_THREADS) dst[i] = src[i];
  } else {
    uint4* dst = reinterpret_cast<uint4*>(sbm);
    for (int64_t i = tid; i < words / 4; i += RE_THREADS) dst[i] = make_uint4(0, 0, 0, 0);
  }
  for (int64_t i = words + tid; i < (int64_t)nseg * 32; i += RE_THREADS) sbm[i] = 0;   // tail segment pad

  // ---- 2. light witnesses of the group's rows, OR-ed in shared memory
  const int64_t xa = a.x0 + r0, xb = a.x0 + r1;
  const int64_t t_begin = a.fwd_ptr[xa], t_end = a.fwd_ptr[xb];
  unsigned long long my_w = 0;
  __syncthreads();
  for (int64_t tb = t_begin; tb < t_end; tb += TUP_BATCH) {
    const int64_t t = tb + tid;
    int len = 0;
    const int32_t* base = nullptr;
    int row = 0;
    if (t < t_end) {
      // the row of tuple t: x with fwd_ptr[x] <= t < fwd_ptr[x+1] inside [xa, xb)
      int64_t lo = xa, hi = xb;   // upper_bound over fwd_ptr
      while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (a.fwd_ptr[mid] <= t) lo = mid;
        else hi = mid;
      }
      const int64_t x = lo;
      row = (int)(x - xa);
      const int32_t y = a.fwd_idx[t];
      const bool full = (a.hpos == nullptr) || (a.hpos[y] < 0) || (a.rdeg_x[x] <= a.d2);
      if (full) {
        const int32_t b = a.s_rev_ptr[y];
        base = a.s_rev_idx + b;
        len = a.s_rev_ptr[y + 1] - b;
      } else {
        const int32_t b = a.lz_ptr[y];
        base = a.lz_idx + b;
        len = a.lz_ptr[y + 1] - b;
      }
    }
    int excl, tot;
    BScan(scan_tmp).ExclusiveSum(len, excl, tot);
    s_tb_len[tid] = excl;
    s_tb_base[tid] = base;
    s_tb_row[tid] = row;
    if (tid == 0) s_tb_len[TUP_BATCH] = tot;
    __syncthreads();
    const int nt = (int)min((int64_t)TUP_BATCH, t_end - tb);
    for (int s = tid; s < tot; s += RE_THREADS) {
      int lo = 0, hi = nt;   // last i with s_tb_len[i] <= s
      while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (s_tb_len[mid] <= s) lo = mid;
        else hi = mid;
      }
      const int32_t z = s_tb_base[lo][s - s_tb_len[lo]];
      atomicOr(&sbm[(int64_t)s_tb_row[lo] * a.wpr + (z >> 5)], 1u << (z & 31));
    }
    my_w += (tid == 0) ? (unsigned long long)tot : 0ull;
    __syncthreads();
  }
  if (tid == 0 && my_w) atomicAdd(a.witnesses, my_w);

  // ---- 3. segment counts, block scan, decoupled look-back
  for (int s = warp; s < nseg; s += RE_WARPS) {
    int c = __popc(sbm[(int64_t)s * 32 + lane]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) segcnt[s] = c;
  }
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (int s0 = 0; s0 < nseg; s0 += RE_THREADS) {
    const int s = s0 + tid;
    const int v = s < nseg ? segcnt[s] : 0;
    int excl, tot;
    BScan(scan_tmp).ExclusiveSum(v, excl, tot);
    const int carry = s_carry;
    __syncthreads();
    if (s < nseg) segcnt[s] = carry + excl;
    if (tid == 0) s_carry = carry + tot;
    __syncthreads();
  }
  if (tid == 0) {
    const unsigned long long cnt = (unsigned long long)s_carry;
    unsigned long long prefix = 0;
    if (g == 0) {
      st_release(&a.status[0], FLAG_INC | cnt);
    } else {
      st_release(&a.status[g], FLAG_AGG | cnt);
      int64_t j = g - 1;
      while (true) {
        const unsigned long long v = ld_acquire(&a.status[j]);
        if (v == 0) continue;
        prefix += v & VAL_MASK;
        if (v & FLAG_INC) break;
        --j;
      }
      st_release(&a.status[g], FLAG_INC | (prefix + cnt));
    }
    s_prefix = (long long)prefix;
    if (g == a.ngroups - 1) *a.total = prefix + cnt;
  }
  __syncthreads();
  const int64_t gbase = s_prefix;

  // ---- 4. emission: per segment, stage codes, coalesced streaming stores
  for (int s = warp; s < nseg; s += RE_WARPS) {
    const int64_t w = (int64_t)s * 32 + lane;         // word within the group
    uint32_t word = sbm[w];
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    int k = incl - c;
    const int64_t row = w / a.wpr;
    const int64_t code0 = (xa + row) * a.dom_z + (w - row * a.wpr) * 32;
    while (word) {
      const int b = __ffs(word) - 1;
      stage[stage_slot(k++)] = code0 + b;
      word &= word - 1;
    }
    __syncwarp();
    int64_t* out = a.codes + gbase + segcnt[s];
    // peel to a 16-byte boundary, then pairs, then the tail
    const int head = (int)(((reinterpret_cast<uintptr_t>(out) >> 3) & 1));
    const int h = min(head, tot);
    if (lane < h) st_stream(out + lane, stage[stage_slot(lane)]);
    const int npair = (tot - h) >> 1;
    for (int p = lane; p < npair; p += 32) {
      const int i = h + 2 * p;
      st_stream_v2(out + i, stage[stage_slot(i)], stage[stage_slot(i + 1)]);
    }
    const int done = h + 2 * npair;
    if (lane < tot - done) st_stream(out + done + lane, stage[stage_slot(done + lane)]);
    __syncwarp();
  }
}

}  // namespace

size_t row_emit_smem(int64_t G, int64_t wpr) {
  const int64_t gw = G * wpr;
  const int nseg = (int)((gw + 31) / 32);
  return (size_t)(((gw * 4 + 15) & ~15ll) + (int64_t)RE_WARPS * STAGE * 8 + (int64_t)nseg * 4 + 16);
}

int row_light_emit(const uint32_t* heavy_bm, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z, int G,
                   const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t d2,
                   const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr,
                   const int32_t* lz_idx, int64_t* codes, unsigned long long* status, int* ticket,
                   unsigned long long* witnesses, unsigned long long* total, cudaStream_t st) {
  if (rows <= 0) return MMJ_OK;
  if (G < 1 || wpr % 8 != 0) {
    set_error("row_light_emit: G >= 1 and wpr % 8 == 0 required");
    return MMJ_ERR_ARG;
  }
  const size_t smem = row_emit_smem(G, wpr);
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t static_smem = sizeof(int) * (TUP_BATCH * 2 + 1) + sizeof(void*) * TUP_BATCH + 4096;
  if (smem + static_smem > (size_t)maxsm) {
    set_error("row_light_emit: row group needs %zu B of shared memory (max %d)", smem, maxsm);
    return MMJ_ERR_UNSUPPORTED;
  }
  static size_t attr = 0;
  if (smem > attr) {
    MMJ_TRY(cuda_status(cudaFuncSetAttribute(k_row_light_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(maxsm - static_smem)),
                        "cudaFuncSetAttribute(row_light_emit)"));
    attr = maxsm - static_smem;
  }
  RowEmitArgs a;
  a.heavy_bm = heavy_bm;
  a.x0 = x0;
  a.rows = rows;
  a.wpr = wpr;
  a.dom_z = dom_z;
  a.G = G;
  a.ngroups = ceil_div(rows, G);
  a.fwd_ptr = fwd_ptr;
  a.fwd_idx = fwd_idx;
  a.rdeg_x = rdeg_x;
  a.d2 = d2;
  a.hpos = hpos;
  a.s_rev_ptr = s_rev_ptr;
  a.s_rev_idx = s_rev_idx;
  a.lz_ptr = lz_ptr;
  a.lz_idx = lz_idx;
  a.codes = codes;
  a.status = status;
  a.ticket = ticket;
  a.witnesses = witnesses;
  a.total = total;
  k_row_light_emit<<<(unsigned)a.ngroups, RE_THREADS, smem, st>>>(a);
  MMJ_CHECK_LAUNCH("k_row_light_emit");
  return MMJ_OK;
}

}  // namespace mmj
