// Fused light expansion + merge + emission over bitmap tiles.
//
// Replaces, for the projection (no counts) two-path path, the light passes
// (joinproject.py:183-203) and the np.unique merge (joinproject.py:220-225).
// The chunk's output space (rows x dom_z bits) is cut into tiles of at most
// TILE_BITS bits -- several whole rows when dom_z is small, otherwise one row
// and a column block -- processed in row-major tile order, one CTA per tile:
//   1. the heavy product's bitmap tile is copied into shared memory (or zeroed
//      when there is no heavy part);
//   2. every light witness (x, z) with x in the tile's rows and z in its
//      column block -- R tuples of those x, each expanding its S-side list
//      (sorted by z, so the column block is a contiguous slice) exactly as the
//      reference's three witness-disjoint passes do -- is OR-ed into the tile
//      with a shared-memory atomic (no global atomics, no materialised keys);
//   3. per-32-word segment popcounts are block-scanned and the tile's global
//      output offset comes from a single-pass decoupled look-back over tiles
//      (blockIdx order: lower tiles are always already resident or done);
//   4. each warp stages a segment's codes (as 32-bit offsets from the tile's
//      first code, in an XOR-swizzled conflict-free layout) and writes them
//      with coalesced 16-byte streaming stores.
// The bitmap is read once and every code written once: the kernel is bound by
// the HBM write of the sorted output (8 B per distinct (x, z)).
#include <cub/block/block_scan.cuh>

#include "mmj_common.cuh"

namespace mmj {
namespace {

constexpr int RE_THREADS = 256;
constexpr int RE_WARPS = RE_THREADS / 32;
constexpr int TUP_BATCH = RE_THREADS;   // light tuples staged per round
constexpr int TILE_WORDS = 2048;        // 8 KB of bitmap per tile (65536 cells)
constexpr int TILE_SEGS = TILE_WORDS / 32;
constexpr int STAGE = 1024;             // codes staged per warp (one segment)
constexpr int SHORT_LIST = 96;          // lists up to this length are filtered, longer ones bisected

constexpr unsigned long long FLAG_AGG = 1ull << 62;
constexpr unsigned long long FLAG_INC = 2ull << 62;
constexpr unsigned long long VAL_MASK = (1ull << 62) - 1;

struct RowEmitArgs {
  const uint32_t* heavy_bm;   // rows x wpr words of the chunk (nullptr: no heavy part)
  int64_t x0, rows, wpr, dom_z;
  int G;                      // rows per tile (1 when a row spans several column blocks)
  int cb_words;               // words per column block (== wpr when G > 1)
  int ncb;                    // column blocks per row
  int64_t ntiles;
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
  unsigned long long* status;          // per tile look-back word (zeroed)
  unsigned long long* witnesses;       // += light witnesses processed
  unsigned long long* total;           // chunk size (written by the last tile)
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

// staging slot of the k-th code of a segment.  Lanes start their runs at
// unrelated offsets; XOR-ing bits [2,5) with bits [5,8) spreads a warp's
// stores over the banks while keeping each aligned quad (k & ~3) contiguous
// and in order, so the reader can fetch four codes with one LDS.128.
__device__ __forceinline__ int stage_slot(int k) { return k ^ ((k >> 3) & 0x1C); }

__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ v, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(RE_THREADS) k_row_light_emit(const RowEmitArgs a) {
  using BScan = cub::BlockScan<int, RE_THREADS>;
  __shared__ typename BScan::TempStorage scan_tmp;
  __shared__ __align__(16) uint32_t sbm[TILE_WORDS];
  __shared__ __align__(16) uint32_t stage_all[RE_WARPS][STAGE + 4];
  __shared__ int segoff[TILE_SEGS];
  __shared__ int s_tb_len[TUP_BATCH + 1];      // exclusive prefix of (clipped) list lengths
  __shared__ const int32_t* s_tb_base[TUP_BATCH];
  __shared__ int s_tb_row[TUP_BATCH];
  __shared__ int s_tb_zlo[TUP_BATCH];          // z range filter for short lists (zlo,zhi) or -1
  __shared__ long long s_prefix;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  uint32_t* stage = stage_all[warp];

  const int64_t tile = blockIdx.x;
  const int64_t rg = tile / a.ncb;               // row group
  const int cbi = (int)(tile - rg * a.ncb);     // column block
  const int64_t r0 = rg * a.G;
  const int64_t r1 = min(r0 + (int64_t)a.G, a.rows);
  const int64_t c0w = (int64_t)cbi * a.cb_words;                 // first word of the block
  const int cw = (int)min((int64_t)a.cb_words, a.wpr - c0w);      // words per row in this block
  const int nrow = (int)(r1 - r0);
  const int words = nrow * cw;                                     // <= TILE_WORDS
  const int nseg = (words + 31) >> 5;
  const int32_t zlo = (int32_t)(c0w * 32);
  const int32_t zhi = (int32_t)min((c0w + cw) * 32, a.dom_z);

  // ---- 1. heavy bitmap tile -> shared memory (row pieces of cw words)
  if (a.heavy_bm != nullptr) {
    const int q4 = cw >> 2;   // cw is a multiple of 8
    for (int i = tid; i < nrow * q4; i += RE_THREADS) {
      const int rr = i / q4, qq = i - rr * q4;
      reinterpret_cast<uint4*>(sbm)[rr * q4 + qq] =
          reinterpret_cast<const uint4*>(a.heavy_bm + (r0 + rr) * a.wpr + c0w)[qq];
    }
  } else {
    for (int i = tid; i < words; i += RE_THREADS) sbm[i] = 0;
  }
  for (int i = words + tid; i < nseg * 32; i += RE_THREADS) sbm[i] = 0;

  // ---- 2. light witnesses of the tile, OR-ed in shared memory
  const int64_t xa = a.x0 + r0, xb = a.x0 + r1;
  const int64_t t_begin = a.fwd_ptr[xa], t_end = a.fwd_ptr[xb];
  unsigned long long my_w = 0;
  __syncthreads();
  for (int64_t tb = t_begin; tb < t_end; tb += TUP_BATCH) {
    const int64_t t = tb + tid;
    int len = 0, row = 0, filt = -1;
    const int32_t* base = nullptr;
    if (t < t_end) {
      int64_t lo = xa, hi = xb;   // row of tuple t: last x with fwd_ptr[x] <= t
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (a.fwd_ptr[mid] <= t) lo = mid;
        else hi = mid;
      }
      const int64_t x = lo;
      row = (int)(x - xa);
      const int32_t y = a.fwd_idx[t];
      const bool full = (a.hpos == nullptr) || (a.hpos[y] < 0) || (a.rdeg_x[x] <= a.d2);
      int32_t b, e;
      if (full) {
        b = a.s_rev_ptr[y];
        e = a.s_rev_ptr[y + 1];
        base = a.s_rev_idx + b;
      } else {
        b = a.lz_ptr[y];
        e = a.lz_ptr[y + 1];
        base = a.lz_idx + b;
      }
      len = e - b;
      if (a.ncb > 1) {
        if (len > SHORT_LIST) {   // z-sorted list: bisect to the column block
          const int lb = lower_bound_i32(base, len, zlo);
          const int ub = lb + lower_bound_i32(base + lb, len - lb, zhi);
          base += lb;
          len = ub - lb;
        } else {
          filt = 1;               // scan it, keep z in [zlo, zhi)
        }
      }
    }
    int excl, tot;
    BScan(scan_tmp).ExclusiveSum(len, excl, tot);
    s_tb_len[tid] = excl;
    s_tb_base[tid] = base;
    s_tb_row[tid] = row;
    s_tb_zlo[tid] = filt;
    if (tid == 0) s_tb_len[TUP_BATCH] = tot;
    __syncthreads();
    const int nt = (int)min((int64_t)TUP_BATCH, t_end - tb);
    int kept = 0;
    for (int s = tid; s < tot; s += RE_THREADS) {
      int lo = 0, hi = nt;   // last i with s_tb_len[i] <= s
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_tb_len[mid] <= s) lo = mid;
        else hi = mid;
      }
      const int32_t z = s_tb_base[lo][s - s_tb_len[lo]];
      if (s_tb_zlo[lo] >= 0 && (z < zlo || z >= zhi)) continue;
      const int wz = (z - zlo) >> 5;
      atomicOr(&sbm[s_tb_row[lo] * cw + wz], 1u << (z & 31));
      ++kept;
    }
    my_w += kept;
    __syncthreads();
  }
  {
    unsigned long long w = my_w;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0 && w) atomicAdd(a.witnesses, w);
  }

  // ---- 3. segment counts, block scan, decoupled look-back
  for (int s = warp; s < nseg; s += RE_WARPS) {
    int c = __popc(sbm[s * 32 + lane]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) segoff[s] = c;
  }
  __syncthreads();
  {
    // TILE_SEGS (64) <= RE_THREADS: one scan round
    const int v = tid < nseg ? segoff[tid] : 0;
    int excl, tot;
    BScan(scan_tmp).ExclusiveSum(v, excl, tot);
    __syncthreads();
    if (tid < nseg) segoff[tid] = excl;
    if (tid == 0) {
      const unsigned long long cnt = (unsigned long long)tot;
      unsigned long long prefix = 0;
      if (tile == 0) {
        st_release(&a.status[0], FLAG_INC | cnt);
      } else {
        st_release(&a.status[tile], FLAG_AGG | cnt);
        int64_t j = tile - 1;
        while (true) {
          const unsigned long long v2 = ld_acquire(&a.status[j]);
          if (v2 == 0) continue;
          prefix += v2 & VAL_MASK;
          if (v2 & FLAG_INC) break;
          --j;
        }
        st_release(&a.status[tile], FLAG_INC | (prefix + cnt));
      }
      s_prefix = (long long)prefix;
      if (tile == a.ntiles - 1) *a.total = prefix + cnt;
    }
  }
  __syncthreads();
  const int64_t tbase_code = xa * a.dom_z + zlo;    // code of the tile's first cell
  int64_t* const out_tile = a.codes + s_prefix;

  // ---- 4. emission: per segment, stage code offsets, coalesced streaming stores
  for (int s = warp; s < nseg; s += RE_WARPS) {
    const int w = s * 32 + lane;                   // word within the tile
    uint32_t word = sbm[w];
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    const int rr = w / cw;
    const uint32_t off0 = (uint32_t)(rr * a.dom_z + (w - rr * cw) * 32);   // G*dom_z < 2^31 (checked)
    int64_t* out = out_tile + segoff[s];
    // stage index of code i is i + h with h = (out / 8) % 2, so that stage
    // quads [4q, 4q+4) map to 16-byte aligned output slots out + 4q - h
    const int h = (int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1);
    // MSB-first: FLO gives the bit, the lane's run is filled from its end
    int k = incl - 1 + h;
    while (word) {
      const int b = 31 - __clz(word);
      stage[stage_slot(k)] = off0 + (uint32_t)b;
      --k;
      word ^= 1u << b;
    }
    __syncwarp();
    const int endk = tot + h;                       // staged indices [h, endk)
    if (lane >= h && lane < 4 && lane < endk) st_stream(out + lane - h, tbase_code + stage[stage_slot(lane)]);
    const int nq = endk >> 2;
    for (int q = 1 + lane; q < nq; q += 32) {
      const uint4 v = *reinterpret_cast<const uint4*>(&stage[stage_slot(4 * q)]);
      int64_t* o = out + 4 * q - h;
      st_stream_v2(o, tbase_code + v.x, tbase_code + v.y);
      st_stream_v2(o + 2, tbase_code + v.z, tbase_code + v.w);
    }
    const int tail = max(4, nq << 2);
    if (tail + lane < endk) st_stream(out + tail + lane - h, tbase_code + stage[stage_slot(tail + lane)]);
    __syncwarp();
  }
}

}  // namespace

size_t row_emit_smem(int64_t /*G*/, int64_t /*wpr*/) { return 0; }   // static shared memory only

int row_light_emit(const uint32_t* heavy_bm, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z, int /*G_hint*/,
                   const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t d2,
                   const int32_t* hpos, const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr,
                   const int32_t* lz_idx, int64_t* codes, unsigned long long* status, int* /*ticket*/,
                   unsigned long long* witnesses, unsigned long long* total, cudaStream_t st) {
  if (rows <= 0) return MMJ_OK;
  if (wpr % 8 != 0 || wpr <= 0) {
    set_error("row_light_emit: wpr must be a positive multiple of 8");
    return MMJ_ERR_ARG;
  }
  RowEmitArgs a;
  a.heavy_bm = heavy_bm;
  a.x0 = x0;
  a.rows = rows;
  a.wpr = wpr;
  a.dom_z = dom_z;
  if (wpr <= TILE_WORDS) {
    a.G = (int)(TILE_WORDS / wpr);
    a.cb_words = (int)wpr;
    a.ncb = 1;
  } else {
    a.G = 1;
    a.cb_words = TILE_WORDS;
    a.ncb = (int)ceil_div(wpr, TILE_WORDS);
  }
  // tile offsets are stored as 32-bit deltas from the tile's first code
  if ((int64_t)a.G * dom_z >= (1ll << 31)) {
    set_error("row_light_emit: tile code span exceeds 32 bits");
    return MMJ_ERR_UNSUPPORTED;
  }
  a.ntiles = ceil_div(rows, a.G) * a.ncb;
  if (a.ntiles >= (1ll << 31)) {
    set_error("row_light_emit: too many tiles in one chunk");
    return MMJ_ERR_ARG;
  }
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
  a.witnesses = witnesses;
  a.total = total;
  k_row_light_emit<<<(unsigned)a.ntiles, RE_THREADS, 0, st>>>(a);
  MMJ_CHECK_LAUNCH("k_row_light_emit");
  return MMJ_OK;
}

int64_t row_emit_tiles(int64_t rows, int64_t wpr) {
  if (wpr <= TILE_WORDS) return ceil_div(rows, TILE_WORDS / wpr);
  return rows * ceil_div(wpr, TILE_WORDS);
}

}  // namespace mmj
