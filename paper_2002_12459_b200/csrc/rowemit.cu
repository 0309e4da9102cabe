// Light expansion merged into the heavy bitmap, then emission of sorted codes.
//
// Replaces, for the projection (no counts) two-path path, the light passes
// (joinproject.py:183-203) and the np.unique merge (joinproject.py:220-225).
// The chunk's output space (rows x dom_z cells, bitmap rows padded to whole
// 1024-bit segments) is processed in two kernels:
//
//   k_tile_merge  one CTA per tile of <= 2^19 cells (whole rows up to 64 KB
//                 of bitmap, several when dom_z is small, otherwise one row and
//                 a 16384-word column block): the heavy product's bitmap tile
//                 is staged in shared
//                 memory, every light witness (x, z) of the tile -- R tuples
//                 of its rows, each expanding its z-sorted S-side list (so a
//                 column block is a contiguous slice) exactly as the
//                 reference's three witness-disjoint passes do -- is OR-ed in
//                 with shared-memory atomics (no global atomics, no
//                 materialised keys), the merged tile is written back and the
//                 popcount of every 32-word segment is recorded;
//   (exclusive scan of the segment counts, scan.cu)
//   k_emit_pf16   one warp per segment (the CTA's 32 segments of bitmap words and
//                 offsets prefetched into shared memory first): prefix of the 32 word popcounts, the
//                 lane's set bits staged as 32-bit cell offsets in a swizzled
//                 shared buffer, then coalesced 16-byte streaming stores of
//                 the int64 codes x*dom_z + z.
// The bitmap is read twice and written once (1/64 of the code bytes each);
// every code is written once: emission is bound by the HBM write of the
// sorted output (8 B per distinct (x, z)).
#include <cub/block/block_scan.cuh>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "mmj_common.cuh"

namespace mmj {
namespace {

constexpr int TM_THREADS = 256;
constexpr int TUP_BATCH = TM_THREADS;   // light tuples staged per round
constexpr int TILE_WORDS = 16384;       // up to 64 KB of bitmap per tile (whole rows up to 524288 cells)
constexpr int SHORT_LIST = 96;          // lists up to this length are filtered, longer ones bisected
// (the emission kernel has no minimum-CTA bound: forcing 6 or 8 resident CTAs
// per SM (40 / 32 registers) measured 1-4% slower than ptxas's 48 registers)
constexpr int MERGE_ILP = 8;            // witness slots per thread per step of the merge
constexpr int EM_WARPS = 8;
constexpr int EM_SEGS = 32;             // segments per emission CTA (4 per warp)

__device__ __forceinline__ void st_cs2(int64_t* p, int64_t a, int64_t b) {
  asm volatile("st.global.cs.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_cs(int64_t* p, int64_t a) {
  asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}

// 32-byte store (sm_100: st.global.v4.b64)
__device__ __forceinline__ void st_v4(int64_t* p, int64_t a, int64_t b, int64_t c, int64_t d) {
  asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 1-D bulk async copies (TMA engine) between global memory and shared memory
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bar_wait0(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ int lower_bound_i32(const int32_t* __restrict__ v, int n, int32_t key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (v[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Emission of one 1024-cell segment (32 bitmap words) by one warp in output
// order without shared-memory staging: step i takes word i, lane l owns its
// bit l (cell 32 i + l) and, when set, writes the code to out[excl_i +
// popc(word_i & lanemask_lt)] -- the active lanes of each store cover one
// contiguous run, so every store is a single coalesced request.  `pw` is the
// warp's 32-entry (word, exclusive code prefix) table, filled by the caller
// (broadcast LDS.128 reads: two words per load).  ~7.5 instructions per word
// against ~19 for the staged 16-bit offset path (ncu r2b source page).
// Returns false when the segment's low code word could carry (the caller
// takes the 64-bit path): code = seg_base + cell with seg_base's low 32 bits
// <= 2^32 - 1025.
__device__ __forceinline__ bool emit_segment_rr(const uint2* __restrict__ pw, int64_t* out, int64_t seg_base,
                                                int lane) {
  if ((uint32_t)seg_base > 0xFFFFFFFFu - 1024u) return false;
  const uint32_t bit = 1u << lane, lt = bit - 1u;
  const uint32_t lo0 = (uint32_t)seg_base + (uint32_t)lane;
  const uint32_t hi = (uint32_t)((uint64_t)seg_base >> 32);
  int64_t* ob;
  asm("mov.b64 %0, %1;" : "=l"(ob) : "l"(out));   // opaque base: one IMAD.WIDE per address
#pragma unroll 4
  for (int i = 0; i < 32; i += 2) {
    const uint4 q = *reinterpret_cast<const uint4*>(pw + i);
    int64_t* p0 = ob + (q.y + __popc(q.x & lt));
    int64_t* p1 = ob + (q.w + __popc(q.z & lt));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %1, 0;\n\t@p st.global.cs.v2.b32 [%0], {%2, %3};\n\t}" ::"l"(p0),
                 "r"(q.x & bit), "r"(lo0 + 32u * i), "r"(hi)
                 : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %1, 0;\n\t@p st.global.cs.v2.b32 [%0], {%2, %3};\n\t}" ::"l"(p1),
                 "r"(q.z & bit), "r"(lo0 + 32u * (i + 1)), "r"(hi)
                 : "memory");
  }
  return true;
}

// segments with fewer codes than this take the staged sparse path
constexpr int RR_MIN_CODES = 128;

// has_heavy: 0 = no heavy part; 1 = the chunk's heavy bitmap (the tcgen05
// product's output) is in bm; 2 = the heavy part is computed by the tile
// itself from the heavy-y bit rows `hbits` (heavy_or_rows)
struct TileArgs {
  uint32_t* bm;               // rows x wpr words (in: heavy bits if has_heavy == 1; out: merged)
  int has_heavy;
  int64_t x0, rows, wpr, dom_z;
  int G, cb_words, ncb;
  const int32_t* fwd_ptr;
  const int32_t* fwd_idx;
  const int32_t* rdeg_x;
  int64_t d2;
  const int32_t* hpos;        // nullptr: FULL_JOIN (every y light)
  const int32_t* s_rev_ptr;
  const int32_t* s_rev_idx;
  const int32_t* lz_ptr;
  const int32_t* lz_idx;
  int32_t* segcnt;            // popcount per 32-word segment of the chunk
  unsigned long long* witnesses;
  // optional (dom_y x (ncb+1)) absolute list positions of the column-block
  // boundaries (full S.rev lists / light-z lists): replaces per-tile bisection
  const int32_t* split_full = nullptr;
  const int32_t* split_lz = nullptr;
  // has_heavy == 2: K x wpr bit rows of S_h (bit z of row hpos[y] set iff z
  // heavy and (z, y) in S) and the heavy_pairs counter
  const uint32_t* hbits = nullptr;
  unsigned long long* heavy_nnz = nullptr;
};

// Heavy part of a tile's rows [xa, xa + nrow), columns [c0w, c0w + cw) words,
// as a sparse boolean product (joinproject.py:208-216, nonzero(M1 @ M2)):
// word i of heavy row x = OR over the heavy y of R[x] of hbits[hpos[y]][c0w+i]
// (light x rows are zero, as in M1).  Each row's heavy positions are
// compacted NT at a time into s_list, then every thread ORs its 16-byte word
// groups over them (the bit rows are L2-resident: K x wpr x 4 B).  Writes
// every word of the tile; returns this thread's popcount of the heavy bits
// (the heavy_pairs statistic).  Block-uniform control flow.
template <int NT>
__device__ unsigned long long heavy_or_rows(const TileArgs& a, uint32_t* sbm, int64_t xa, int nrow, int cw,
                                            int64_t c0w, typename cub::BlockScan<int, NT>::TempStorage& scan_tmp,
                                            int* s_list) {
  const int tid = threadIdx.x;
  const int q4 = cw >> 2;
  unsigned long long pc = 0;
  for (int rr = 0; rr < nrow; ++rr) {
    const int64_t x = xa + rr;
    uint4* dst = reinterpret_cast<uint4*>(sbm + (int64_t)rr * cw);
    const bool heavy_x = a.rdeg_x[x] > a.d2;
    const int64_t tb0 = heavy_x ? a.fwd_ptr[x] : 0, te = heavy_x ? a.fwd_ptr[x + 1] : 0;
    if (tb0 >= te) {
      for (int q = tid; q < q4; q += NT) dst[q] = make_uint4(0u, 0u, 0u, 0u);
      continue;
    }
    for (int64_t tb = tb0; tb < te; tb += NT) {
      const int64_t t = tb + tid;
      const int h = t < te ? a.hpos[a.fwd_idx[t]] : -1;
      int pos, cnt;
      cub::BlockScan<int, NT>(scan_tmp).ExclusiveSum(h >= 0 ? 1 : 0, pos, cnt);
      MMJ_DCHECK(pos <= NT, "heavy list position");
      if (h >= 0) s_list[pos] = h;
      __syncthreads();
      const bool last = tb + NT >= te;
      for (int q = tid; q < q4; q += NT) {
        uint4 v = tb == tb0 ? make_uint4(0u, 0u, 0u, 0u) : dst[q];
        int j = 0;
        for (; j + 2 <= cnt; j += 2) {   // two independent L2 loads in flight
          const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(a.hbits + (int64_t)s_list[j] * a.wpr + c0w) + q);
          const uint4 w1 = __ldg(reinterpret_cast<const uint4*>(a.hbits + (int64_t)s_list[j + 1] * a.wpr + c0w) + q);
          v.x |= w0.x | w1.x;
          v.y |= w0.y | w1.y;
          v.z |= w0.z | w1.z;
          v.w |= w0.w | w1.w;
        }
        if (j < cnt) {
          const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(a.hbits + (int64_t)s_list[j] * a.wpr + c0w) + q);
          v.x |= w0.x;
          v.y |= w0.y;
          v.z |= w0.z;
          v.w |= w0.w;
        }
        dst[q] = v;
        if (last) pc += __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
      }
      __syncthreads();   // s_list / scan storage reused by the next batch
    }
  }
  return pc;
}

// Light witnesses of one tile OR-ed into its shared-memory bitmap (rows
// [xa, xb), columns [zlo, zhi), cw words per row): R tuples are staged NT at a
// time, each expanding its z-sorted S-side list -- the full S.rev(y) when y
// is light or x is light, the light-z part otherwise (joinproject.py:183-203
// restated from the x side) -- with MERGE_ILP list loads in flight per thread
// before the shared-memory atomics.  Returns this thread's witness count.
template <int NT>
__device__ __forceinline__ unsigned long long merge_light(
    const TileArgs& a, uint32_t* sbm, int64_t xa, int64_t xb, int64_t t_begin, int64_t t_end, int32_t zlo,
    int32_t zhi, int cw, int cbi, typename cub::BlockScan<int, NT>::TempStorage& scan_tmp, int* s_tb_len,
    const int32_t** s_tb_base, int* s_tb_row, int* s_tb_filt, int* s_touched) {
  const int tid = threadIdx.x;
  unsigned long long my_w = 0;
  for (int64_t tb = t_begin; tb < t_end; tb += NT) {
    const int64_t t = tb + tid;
    int len = 0, row = 0, filt = 0;
    const int32_t* base = nullptr;
    if (t < t_end) {
      int64_t lo = xa, hi = xb;   // row of tuple t: last x with fwd_ptr[x] <= t
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (a.fwd_ptr[mid] <= t) lo = mid;
        else hi = mid;
      }
      row = (int)(lo - xa);
      const int32_t y = a.fwd_idx[t];
      // joinproject.py:183-203: y light or x light -> S.rev(y); else light z only
      const bool full = (a.hpos == nullptr) || (a.hpos[y] < 0) || (a.rdeg_x[lo] <= a.d2);
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
        const int32_t* sp = full ? a.split_full : a.split_lz;
        if (sp != nullptr) {
          // precomputed column-block boundaries of the list (mmj_list_splits)
          const int32_t* q = sp + (int64_t)y * (a.ncb + 1) + cbi;
          const int32_t lb = q[0], ub = q[1];
          base += lb - b;
          len = ub - lb;
        } else if (len > SHORT_LIST) {
          const int lb = lower_bound_i32(base, len, zlo);
          const int ub = lb + lower_bound_i32(base + lb, len - lb, zhi);
          base += lb;
          len = ub - lb;
        } else {
          filt = 1;
        }
      }
    }
    int excl, tot;
    cub::BlockScan<int, NT>(scan_tmp).ExclusiveSum(len, excl, tot);
    s_tb_len[tid] = excl;
    s_tb_base[tid] = base;
    s_tb_row[tid] = row;
    s_tb_filt[tid] = filt;
    if (tid == 0) s_tb_len[NT] = tot;
    __syncthreads();
    const int nt = (int)min((int64_t)NT, t_end - tb);
    int kept = 0;
    int ti = 0;   // tuple of the current slot; slots grow, so the cursor only moves forward
    // MERGE_ILP slots per thread per step: their list loads are issued
    // together before the shared-memory atomics (the loads are the latency)
    for (int s0 = tid; s0 < tot; s0 += MERGE_ILP * NT) {
      int32_t zv[MERGE_ILP];
      int rowv[MERGE_ILP];
      bool ok[MERGE_ILP];
#pragma unroll
      for (int u = 0; u < MERGE_ILP; ++u) {
        const int s = s0 + u * NT;
        ok[u] = s < tot;
        rowv[u] = 0;
        zv[u] = 0;
        if (ok[u]) {
          while (ti + 1 < nt && s_tb_len[ti + 1] <= s) ++ti;
          zv[u] = __ldg(s_tb_base[ti] + (s - s_tb_len[ti]));
          rowv[u] = s_tb_row[ti] | (s_tb_filt[ti] << 30);
        }
      }
#pragma unroll
      for (int u = 0; u < MERGE_ILP; ++u) {
        if (!ok[u]) continue;
        const int32_t z = zv[u];
        if ((rowv[u] >> 30) && (z < zlo || z >= zhi)) continue;
        MMJ_DCHECK(z >= zlo && z < zhi && (rowv[u] & 0x3FFFFFFF) < (int)(xb - xa), "light witness outside the tile");
        atomicOr(&sbm[(rowv[u] & 0x3FFFFFFF) * cw + ((z - zlo) >> 5)], 1u << (z & 31));
        ++kept;
      }
    }
    my_w += kept;
    if (tot > 0 && tid == 0) *s_touched = 1;
    __syncthreads();
  }
  return my_w;
}

__global__ void __launch_bounds__(TM_THREADS) k_tile_merge(const TileArgs a) {
  using BScan = cub::BlockScan<int, TM_THREADS>;
  __shared__ typename BScan::TempStorage scan_tmp;
  extern __shared__ __align__(16) uint32_t sbm[];     // tile words (dynamic)
  __shared__ int s_tb_len[TUP_BATCH + 1];
  __shared__ const int32_t* s_tb_base[TUP_BATCH];
  __shared__ int s_tb_row[TUP_BATCH];
  __shared__ int s_tb_filt[TUP_BATCH];
  __shared__ int s_touched;
  __shared__ __align__(8) uint64_t s_bar;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t tile = blockIdx.x;
  const int64_t rg = tile / a.ncb;
  const int cbi = (int)(tile - rg * a.ncb);
  const int64_t r0 = rg * a.G;
  const int64_t r1 = min(r0 + (int64_t)a.G, a.rows);
  const int64_t c0w = (int64_t)cbi * a.cb_words;
  const int cw = (int)min((int64_t)a.cb_words, a.wpr - c0w);   // multiple of 32
  const int nrow = (int)(r1 - r0);
  const int words = nrow * cw;
  const int32_t zlo = (int32_t)(c0w * 32);
  const int32_t zhi = (int32_t)min((c0w + cw) * 32, a.dom_z);
  const int q4 = cw >> 2;

  // the tile is one contiguous range of the chunk bitmap: several whole rows
  // (ncb == 1) or one row piece (G == 1)
  uint32_t* gtile = a.bm + r0 * a.wpr + c0w;
  const uint32_t tile_bytes = (uint32_t)words * 4u;
  if (a.has_heavy == 1) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      bulk_g2s(sbm, gtile, tile_bytes, &s_bar);
    }
  } else if (a.has_heavy == 0) {
    for (int i = tid; i < words; i += TM_THREADS) sbm[i] = 0;
  }
  if (tid == 0) s_touched = 0;

  const int64_t xa = a.x0 + r0, xb = a.x0 + r1;
  const int64_t t_begin = a.fwd_ptr[xa], t_end = a.fwd_ptr[xb];
  unsigned long long my_w = 0;
  if (a.has_heavy == 2) {
    unsigned long long pc = heavy_or_rows<TM_THREADS>(a, sbm, xa, nrow, cw, c0w, scan_tmp, s_tb_len);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
    if (lane == 0 && pc) atomicAdd(a.heavy_nnz, pc);
  }
  __syncthreads();
  if (a.has_heavy == 1) bar_wait0(&s_bar);   // tile bytes landed (all threads observe the phase)
  my_w = merge_light<TM_THREADS>(a, sbm, xa, xb, t_begin, t_end, zlo, zhi, cw, cbi, scan_tmp, s_tb_len, s_tb_base,
                                 s_tb_row, s_tb_filt, &s_touched);
  {
    unsigned long long w = my_w;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0 && w) atomicAdd(a.witnesses, w);
  }
  // write back the merged tile (skipped when the heavy bits are unchanged)
  __syncthreads();
  if ((s_touched || a.has_heavy != 1) && tid == 0) bulk_s2g(gtile, sbm, tile_bytes);
  // segment popcounts (segments never straddle rows: wpr % 32 == 0): a warp
  // takes 32 segments, lane l reads word l of each (conflict-free LDS) and
  // REDUX sums the 32 popcounts; lane j keeps the total of segment j
  const int nseg = words >> 5;
  const int segs_per_piece = cw >> 5;
  for (int sb = warp * 32; sb < nseg; sb += TM_THREADS) {
    int mine = 0;
    const int ns = min(32, nseg - sb);
    for (int j = 0; j < ns; ++j) {
      const int c = __reduce_add_sync(0xffffffffu, __popc(sbm[(sb + j) * 32 + lane]));
      if (lane == j) mine = c;
    }
    if (lane < ns) {
      const int sg = sb + lane;
      const int rr = sg / segs_per_piece, sc = sg - rr * segs_per_piece;
      a.segcnt[((r0 + rr) * a.wpr + c0w) / 32 + sc] = mine;
    }
  }
}

// --------------------------------------------------------------- emission
// Emission of the three-kernel tail: the CTA's SEGS segments (bitmap words
// and offsets) are prefetched into shared memory, then one warp per segment
// stages its cells as 16-bit offsets (cell offsets < 1024) -- a branch-free
// bit slice for dense words, an ffs loop for sparse ones -- and writes the
// codes with 16-byte streaming stores (8 CTAs, 64 warps, per SM).  Element
// i is staged at slot i + h (h = the output's 16-B misalignment) so every
// stored pair is one aligned 32-bit shared load.
template <int SEGS>
__global__ void __launch_bounds__(EM_WARPS * 32) k_emit_pf16(const uint32_t* __restrict__ bm,
                                                             const int64_t* __restrict__ segoff, int64_t nseg,
                                                             int64_t segs_per_row, int64_t x0, int64_t dom_z,
                                                             int64_t* __restrict__ codes) {
  __shared__ __align__(16) uint16_t stage_all[EM_WARPS][1024 + 8];
  __shared__ __align__(16) uint32_t sbits[SEGS * 32];
  __shared__ int64_t soff[SEGS + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint16_t* stage = stage_all[warp];
  // slot of element k: XOR bits 1-5 with bits 5-9 so the 32 lanes' runs (one
  // per 32-cell word, up to 32 long) fall in 32 different banks even when the
  // words are full; bit 0 is kept, so an even/odd pair shares one 32-bit word
  auto sl = [](int k) { return k ^ (((k >> 5) & 31) << 1); };
  const int64_t s0 = (int64_t)blockIdx.x * SEGS;
  const int64_t nhere = min((int64_t)SEGS, nseg - s0);
  {
    const uint4* src = reinterpret_cast<const uint4*>(bm + s0 * 32);
    uint4* dst = reinterpret_cast<uint4*>(sbits);
    const int nq = (int)(nhere * 8);
#pragma unroll 2
    for (int i = threadIdx.x; i < nq; i += EM_WARPS * 32) dst[i] = __ldcs(src + i);
    for (int i = threadIdx.x; i <= nhere; i += EM_WARPS * 32) soff[i] = segoff[s0 + i];
  }
  __syncthreads();
  for (int si = warp; si < nhere; si += EM_WARPS) {
    const int64_t s = s0 + si;
    uint32_t word = sbits[si * 32 + lane];
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    const int64_t row = s / segs_per_row;
    const int64_t base = (x0 + row) * dom_z + (s - row * segs_per_row) * 1024;
    int64_t* out = codes + soff[si];
    const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), tot);
    const uint32_t off0 = lane * 32;
    int k = h + (incl - c);
    // dense words (the warp's fullest lane >= 10 bits): the branch-free bit
    // slice; sparse ones: the ffs loop (warp-uniform choice)
    if (__reduce_max_sync(0xffffffffu, (unsigned)c) >= 10u) {
      // branch-free: 32 predicated 16-bit stores, independent of the density
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        if (word & (1u << b)) {
          stage[sl(k)] = (uint16_t)(off0 + b);
          ++k;
        }
      }
    } else {
      while (word) {
        const int b = __ffs(word) - 1;
        stage[sl(k)] = (uint16_t)(off0 + b);
        ++k;
        word &= word - 1;
      }
    }
    __syncwarp();
    if (lane < h) st_cs(out, base + stage[sl(h)]);
    const int np = (tot - h) >> 1;
    for (int p = lane; p < np; p += 32) {
      const uint32_t two = *reinterpret_cast<const uint32_t*>(stage + sl(2 * h + 2 * p));
      st_cs2(out + h + 2 * p, base + (two & 0xFFFFu), base + (two >> 16));
    }
    const int done = h + 2 * np;
    if (lane < tot - done) st_cs(out + done + lane, base + stage[sl(h + done + lane)]);
    __syncwarp();
  }
}


// ---------------------------------------------------------------------------
// Fused light merge + emission (one kernel per chunk, no bitmap write-back,
// no separate segment scan).  Tiles are taken in ticket order; each tile
//   1. stages its heavy bitmap words (TMA bulk copy) or zeros in shared memory,
//   2. ORs in its light witnesses (merge_light, as k_tile_merge),
//   3. popcounts and scans its 32-word segments in shared memory,
//   4. publishes its code count and obtains the codes of all earlier tiles by
//      a decoupled look-back over the per-tile status words (flag in bits
//      62-63: 1 = tile aggregate, 2 = inclusive prefix),
//   5. emits its sorted codes x*dom_z + z exactly as k_emit_pf16.
// Tickets make the look-back deadlock-free: a tile only waits on tiles whose
// CTAs were scheduled before it.
struct FuseArgs {
  TileArgs t;
  int64_t ntiles;
  unsigned int* ticket;
  unsigned long long* status;
  int64_t* total;           // chunk code count (written by the last tile)
  int64_t* codes;
  unsigned long long* tdbg;  // MMJ_DEBUG_TIMING: per-tile phase timestamps (8 per tile)
};

#ifndef MMJ_LOOKBACK_SLEEP_NS
#define MMJ_LOOKBACK_SLEEP_NS 128
#endif

constexpr unsigned long long ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int NT>
struct FuseSmem {
  typename cub::BlockScan<int, NT>::TempStorage scan_tmp;
  union __align__(16) {
    struct {
      int tb_len[NT + 1];
      const int32_t* tb_base[NT];
      int tb_row[NT];
      int tb_filt[NT];
    } m;
    uint16_t stage[NT / 32][1024 + 8];
  } u;
  int touched;
  int next_seg;
  unsigned int tile;
  long long prefix;
  __align__(8) uint64_t bar;
};

template <int TW, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_merge_emit(const FuseArgs f) {
  constexpr int NWARP = NT / 32;
  constexpr int MAXSEG = TW / 32;
  __shared__ FuseSmem<NT> sm;
  __shared__ int s_segoff[MAXSEG];
  extern __shared__ __align__(16) uint32_t sbm[];
  const TileArgs& a = f.t;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    sm.tile = atomicAdd(f.ticket, 1u);
    sm.touched = 0;
  }
  __syncthreads();

#ifdef MMJ_DEBUG_TIMING
  if (tid == 0 && f.tdbg) f.tdbg[(int64_t)sm.tile * 8 + 0] = gtimer();
#endif
  const int64_t tile = sm.tile;
  const int64_t rg = tile / a.ncb;
  const int cbi = (int)(tile - rg * a.ncb);
  const int64_t r0 = rg * a.G;
  const int64_t r1 = min(r0 + (int64_t)a.G, a.rows);
  const int64_t c0w = (int64_t)cbi * a.cb_words;
  const int cw = (int)min((int64_t)a.cb_words, a.wpr - c0w);
  const int nrow = (int)(r1 - r0);
  const int words = nrow * cw;
  const int32_t zlo = (int32_t)(c0w * 32);
  const int32_t zhi = (int32_t)min((c0w + cw) * 32, a.dom_z);
  const uint32_t* gtile = a.bm + r0 * a.wpr + c0w;
  if (a.has_heavy == 1) {
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      bulk_g2s(sbm, gtile, (uint32_t)words * 4u, &sm.bar);
    }
  } else if (a.has_heavy == 0) {
    for (int i = tid; i < words; i += NT) sbm[i] = 0;
  }
  const int64_t xa = a.x0 + r0, xb = a.x0 + r1;
  // fwd_ptr == nullptr: the bitmap is already complete (no light witnesses to merge)
  const int64_t t_begin = a.fwd_ptr ? a.fwd_ptr[xa] : 0, t_end = a.fwd_ptr ? a.fwd_ptr[xb] : 0;
  if (a.has_heavy == 2) {
    // the heavy part computed in place: no tcgen05 product, no bitmap in HBM
    unsigned long long pc = heavy_or_rows<NT>(a, sbm, xa, nrow, cw, c0w, sm.scan_tmp, sm.u.m.tb_len);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
    if (lane == 0 && pc) atomicAdd(a.heavy_nnz, pc);
  }
  __syncthreads();
  if (a.has_heavy == 1) bar_wait0(&sm.bar);

#ifdef MMJ_DEBUG_TIMING
  if (tid == 0 && f.tdbg) f.tdbg[(int64_t)sm.tile * 8 + 1] = gtimer();
#endif
  unsigned long long my_w = merge_light<NT>(a, sbm, xa, xb, t_begin, t_end, zlo, zhi, cw, cbi, sm.scan_tmp, sm.u.m.tb_len,
                                            sm.u.m.tb_base, sm.u.m.tb_row, sm.u.m.tb_filt, &sm.touched);
  {
    unsigned long long w = my_w;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    if (lane == 0 && w) atomicAdd(a.witnesses, w);
  }
  __syncthreads();   // merged tile complete

#ifdef MMJ_DEBUG_TIMING
  if (tid == 0 && f.tdbg) f.tdbg[(int64_t)sm.tile * 8 + 2] = gtimer();
#endif
  // segment popcounts (REDUX over the 32 words of a segment, one warp per 32 segments)
  const int nseg = words >> 5;
  for (int sb = warp * 32; sb < nseg; sb += NT) {
    int mine = 0;
    const int ns = min(32, nseg - sb);
    for (int j = 0; j < ns; ++j) {
      const int c = __reduce_add_sync(0xffffffffu, __popc(sbm[(sb + j) * 32 + lane]));
      if (lane == j) mine = c;
    }
    if (lane < ns) s_segoff[sb + lane] = mine;
  }
  __syncthreads();
  // exclusive scan of the segment counts (MAXSEG / NT items per thread)
  constexpr int IPT = (MAXSEG + NT - 1) / NT;
  int v[IPT];
  int loc = 0;
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int sg = tid * IPT + i;
    v[i] = sg < nseg ? s_segoff[sg] : 0;
    loc += v[i];
  }
  int excl, agg;
  cub::BlockScan<int, NT>(sm.scan_tmp).ExclusiveSum(loc, excl, agg);
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int sg = tid * IPT + i;
    if (sg < nseg) s_segoff[sg] = excl;
    excl += v[i];
  }

#ifdef MMJ_DEBUG_TIMING
  if (tid == 0 && f.tdbg) f.tdbg[(int64_t)sm.tile * 8 + 3] = gtimer();
#endif
  // decoupled look-back (warp 0)
  if (warp == 0) {
    long long prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_status(f.status, ST_INC | (unsigned long long)agg);
    } else {
      if (lane == 0) st_status(f.status + tile, ST_AGG | (unsigned long long)agg);
      int64_t pos = tile - 1;
      while (true) {
        const int64_t idx = pos - lane;
        MMJ_DCHECK(idx < f.ntiles, "look-back status index");
        unsigned long long st = idx >= 0 ? ld_status(f.status + idx) : ST_INC;
        while (__any_sync(0xffffffffu, (st >> 62) == 0)) {
          // back off between polls: the spinning warp otherwise takes issue
          // slots from the SM's emitting warps (4% of the kernel's instructions)
          if (MMJ_LOOKBACK_SLEEP_NS > 0) __nanosleep(MMJ_LOOKBACK_SLEEP_NS);
          if ((st >> 62) == 0) st = ld_status(f.status + idx);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        const int stop = inc ? __ffs(inc) - 1 : 31;
        long long val = lane <= stop ? (long long)(st & ST_VAL) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        prefix += val;
        if (inc) break;
        pos -= 32;
      }
      if (lane == 0) st_status(f.status + tile, ST_INC | (unsigned long long)(prefix + agg));
    }
    if (lane == 0) {
      sm.prefix = prefix;
      sm.next_seg = NWARP;
      if (tile == f.ntiles - 1) *f.total = prefix + agg;
    }
  }
  __syncthreads();
#ifdef MMJ_DEBUG_TIMING
  if (tid == 0 && f.tdbg) f.tdbg[(int64_t)sm.tile * 8 + 4] = gtimer();
#endif
  // emission: one warp per 1024-cell segment -- round robin over its words
  // straight to global memory (emit_segment_rr); full segments as one
  // 16-byte store run; sparse segments (< RR_MIN_CODES codes) through the
  // 16-bit shared staging of k_emit_pf16.  (Measured and not adopted, r2h /
  // r2i: TMA bulk stores of ~1.7 KB staged pieces 224 vs 175 ms; moving
  // segment boundaries to 128-byte lines so one warp writes each line 206 ms.)
  uint16_t* stage = sm.u.stage[warp];
  auto sl = [](int k) { return k ^ (((k >> 5) & 31) << 1); };
  const int segs_per_piece = cw >> 5;
  int64_t* const codes = f.codes + sm.prefix;
  // segments are handed out dynamically (segment densities vary: a static
  // round robin left warps idle at the CTA's exit waiting for the slowest)
  for (int si = warp; si < nseg;) {
    uint32_t word = sbm[si * 32 + lane];
    const int c = __popc(word);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int vv = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += vv;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    const int cur = si;
    {
      int nx = 0;
      if (lane == 0) nx = atomicAdd(&sm.next_seg, 1);
      si = __shfl_sync(0xffffffffu, nx, 0);
    }
    if (tot == 0) continue;
    const int rr = cur / segs_per_piece;
    const int64_t base = (a.x0 + r0 + rr) * a.dom_z + (c0w + (int64_t)(cur - rr * segs_per_piece) * 32) * 32;
    int64_t* out = codes + s_segoff[cur];
    MMJ_DCHECK(s_segoff[cur] >= 0 && s_segoff[cur] + tot <= agg, "segment codes outside the tile's output range");
    if (tot == 1024) {
      // full segment: codes base .. base + 1023, 16-byte stores
      const int hh = (int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1);
      if (lane == 0 && hh) st_cs(out, base);
      for (int p = hh + 2 * lane; p + 1 < 1024; p += 64) st_cs2(out + p, base + p, base + p + 1);
      if (lane == 0 && hh) st_cs(out + 1023, base + 1023);
      continue;
    }
    if (tot >= RR_MIN_CODES) {
      uint2* pw = reinterpret_cast<uint2*>(stage);
      pw[lane] = make_uint2(word, (uint32_t)(incl - c));
      __syncwarp();
      const bool done_rr = emit_segment_rr(pw, out, base, lane);
      __syncwarp();
      if (done_rr) continue;
    }
    const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), tot);
    const uint32_t off0 = lane * 32;
    int k = h + (incl - c);
    if (__reduce_max_sync(0xffffffffu, (unsigned)c) >= 10u) {
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        if (word & (1u << b)) {
          stage[sl(k)] = (uint16_t)(off0 + b);
          ++k;
        }
      }
    } else {
      while (word) {
        const int b = __ffs(word) - 1;
        stage[sl(k)] = (uint16_t)(off0 + b);
        ++k;
        word &= word - 1;
      }
    }
    __syncwarp();
    if (lane < h) st_cs(out, base + stage[sl(h)]);
    const int np = (tot - h) >> 1;
    for (int p = lane; p < np; p += 32) {
      const uint32_t two = *reinterpret_cast<const uint32_t*>(stage + sl(2 * h + 2 * p));
      st_cs2(out + h + 2 * p, base + (two & 0xFFFFu), base + (two >> 16));
    }
    const int done = h + 2 * np;
    if (lane < tot - done) st_cs(out + done + lane, base + stage[sl(h + done + lane)]);
    __syncwarp();
  }
#ifdef MMJ_DEBUG_TIMING
  __syncthreads();
  if (tid == 0 && f.tdbg) f.tdbg[(int64_t)sm.tile * 8 + 5] = gtimer();
#endif
}


// ---------------------------------------------------------------------------
// split[y*(ncb+1) + j] = absolute position in idx of the first entry of list
// y (ptr[y] .. ptr[y+1], sorted) that is >= j * cb_cells
__global__ void k_list_splits(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx, int64_t dom_y,
                              int ncb, int64_t cb_cells, int32_t* __restrict__ split) {
  const int64_t n = dom_y * (ncb + 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = i / (ncb + 1);
    const int j = (int)(i - y * (ncb + 1));
    const int32_t b = ptr[y], e = ptr[y + 1];
    int32_t pos;
    if (j == 0) pos = b;
    else if (j == ncb) pos = e;
    else {
      const int64_t key = (int64_t)j * cb_cells;
      int lo = b, hi = e;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)idx[mid] < key) lo = mid + 1;
        else hi = mid;
      }
      pos = lo;
    }
    split[i] = pos;
  }
}

void tile_geometry(int64_t wpr, int& G, int& cb, int& ncb, int64_t tile_words = TILE_WORDS) {
  if (wpr <= tile_words) {
    G = (int)(tile_words / wpr);
    cb = (int)wpr;
    ncb = 1;
  } else {
    G = 1;
    cb = (int)tile_words;
    ncb = (int)ceil_div(wpr, tile_words);
  }
}

// 32 KB of bitmap per tile (2048 / 4096 / 16384 measured slower: r2f 198 / 179 / - vs 175 ms)
constexpr int FUSE_TILE_WORDS = 8192;

// 9 warps x 4 CTAs = 36 warps per SM (171.8 vs 173.1 ms per cfg2 step for 8
// warps: more warps hide the look-back wait; 576 x 2 / 448 x 2 CTAs with the
// round-robin emission: 188 / 184 vs 170 ms, r2l)
constexpr int FUSE_THREADS = 288;
constexpr int FUSE_MIN_CTAS = 4;

int launch_merge_emit(const FuseArgs& f, cudaStream_t st) {
  auto kern = k_merge_emit<FUSE_TILE_WORDS, FUSE_THREADS, FUSE_MIN_CTAS>;
  MMJ_TRY(set_max_dynamic_smem((const void*)kern, FUSE_TILE_WORDS * 4, "k_merge_emit"));
  const size_t smem = (size_t)f.t.G * f.t.cb_words * 4;
  kern<<<(unsigned)f.ntiles, FUSE_THREADS, smem, st>>>(f);
  MMJ_CHECK_LAUNCH("k_merge_emit");
  return MMJ_OK;
}

}  // namespace

int merge_emit_col_blocks(int64_t wpr) {
  int G, cb, ncb;
  tile_geometry(wpr, G, cb, ncb, FUSE_TILE_WORDS);
  return ncb;
}

int list_splits(const int32_t* ptr, const int32_t* idx, int64_t dom_y, int64_t wpr, int32_t* split, cudaStream_t st) {
  int G, cb, ncb;
  tile_geometry(wpr, G, cb, ncb, FUSE_TILE_WORDS);
  const int64_t n = dom_y * (ncb + 1);
  if (n == 0) return MMJ_OK;
  const int64_t g = std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 16);
  k_list_splits<<<(unsigned)g, 256, 0, st>>>(ptr, idx, dom_y, ncb, (int64_t)cb * 32, split);
  MMJ_CHECK_LAUNCH("k_list_splits");
  return MMJ_OK;
}

int64_t merge_emit_tiles(int64_t rows, int64_t wpr) {
  int G, cb, ncb;
  tile_geometry(wpr, G, cb, ncb, FUSE_TILE_WORDS);
  return ceil_div(rows, G) * ncb;
}

size_t merge_emit_ws_bytes(int64_t rows, int64_t wpr) {
  return 16 + (size_t)merge_emit_tiles(rows, wpr) * 8;
}

unsigned long long* tdbg_buffer = nullptr;   // MMJ_DEBUG_TIMING builds: set by mmj_debug_timing_buffer

int merge_emit(const uint32_t* bm, int has_heavy, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z,
               const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t d2, const int32_t* hpos,
               const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr, const int32_t* lz_idx,
               const int32_t* split_full, const int32_t* split_lz, unsigned long long* witnesses,
               unsigned long long* heavy_pairs, int64_t* codes, int64_t* total, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  if (wpr <= 0 || wpr % 32 != 0) {
    set_error("merge_emit: bitmap pitch must be a positive multiple of 32 words");
    return MMJ_ERR_ARG;
  }
  if (has_heavy < 0 || has_heavy > 2 ||
      (has_heavy == 2 && (hpos == nullptr || fwd_ptr == nullptr || heavy_pairs == nullptr))) {
    set_error("merge_emit: has_heavy must be 0, 1 or 2 (2 needs hpos, the R CSR and a heavy_pairs counter)");
    return MMJ_ERR_ARG;
  }
  if (rows <= 0) return cuda_status(cudaMemsetAsync(total, 0, sizeof(int64_t), st), "merge_emit: total");
  FuseArgs f;
  TileArgs& a = f.t;
  a.bm = const_cast<uint32_t*>(bm);
  a.has_heavy = has_heavy;
  a.x0 = x0;
  a.rows = rows;
  a.wpr = wpr;
  a.dom_z = dom_z;
  tile_geometry(wpr, a.G, a.cb_words, a.ncb, FUSE_TILE_WORDS);
  f.ntiles = ceil_div(rows, a.G) * a.ncb;
  if (f.ntiles >= (1ll << 31)) {
    set_error("merge_emit: too many tiles in one chunk");
    return MMJ_ERR_ARG;
  }
  const size_t need = 16 + (size_t)f.ntiles * 8;
  if (ws == nullptr || ws_bytes < need) {
    set_error("merge_emit: workspace of %zu bytes needed (got %zu)", need, ws_bytes);
    return MMJ_ERR_CAPACITY;
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
  a.segcnt = nullptr;
  a.witnesses = witnesses;
  a.split_full = split_full;
  a.split_lz = split_lz;
  if (has_heavy == 2) {
    a.hbits = bm;
    a.heavy_nnz = heavy_pairs;
  }
  f.ticket = static_cast<unsigned int*>(ws);
  f.status = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 16);
  f.total = total;
  f.codes = codes;
  f.tdbg = tdbg_buffer;
  MMJ_TRY(cuda_status(cudaMemsetAsync(ws, 0, need, st), "merge_emit: workspace reset"));
  return launch_merge_emit(f, st);
}

int64_t row_emit_tiles(int64_t rows, int64_t wpr) {
  int G, cb, ncb;
  tile_geometry(wpr, G, cb, ncb);
  return ceil_div(rows, G) * ncb;
}

int tile_merge(uint32_t* bm, int has_heavy, int64_t x0, int64_t rows, int64_t wpr, int64_t dom_z,
               const int32_t* fwd_ptr, const int32_t* fwd_idx, const int32_t* rdeg_x, int64_t d2, const int32_t* hpos,
               const int32_t* s_rev_ptr, const int32_t* s_rev_idx, const int32_t* lz_ptr, const int32_t* lz_idx,
               const uint32_t* hbits, unsigned long long* heavy_pairs, int32_t* segcnt, unsigned long long* witnesses,
               cudaStream_t st) {
  if (rows <= 0) return MMJ_OK;
  if (wpr <= 0 || wpr % 32 != 0) {
    set_error("tile_merge: bitmap pitch must be a positive multiple of 32 words");
    return MMJ_ERR_ARG;
  }
  if (has_heavy < 0 || has_heavy > 2 ||
      (has_heavy == 2 && (hbits == nullptr || hpos == nullptr || heavy_pairs == nullptr))) {
    set_error("tile_merge: has_heavy must be 0, 1 or 2 (2 needs the heavy-y bit rows, hpos and a counter)");
    return MMJ_ERR_ARG;
  }
  TileArgs a;
  a.bm = bm;
  a.has_heavy = has_heavy;
  a.x0 = x0;
  a.rows = rows;
  a.wpr = wpr;
  a.dom_z = dom_z;
  tile_geometry(wpr, a.G, a.cb_words, a.ncb);
  const int64_t ntiles = ceil_div(rows, a.G) * a.ncb;
  if (ntiles >= (1ll << 31)) {
    set_error("tile_merge: too many tiles in one chunk");
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
  a.segcnt = segcnt;
  a.witnesses = witnesses;
  a.hbits = hbits;
  a.heavy_nnz = heavy_pairs;
  const size_t smem = (size_t)a.G * a.cb_words * 4;
  MMJ_TRY(set_max_dynamic_smem((const void*)k_tile_merge, TILE_WORDS * 4, "k_tile_merge"));
  k_tile_merge<<<(unsigned)ntiles, TM_THREADS, smem, st>>>(a);
  MMJ_CHECK_LAUNCH("k_tile_merge");
  return MMJ_OK;
}

int emit_codes(const uint32_t* bm, const int64_t* segoff, int64_t rows, int64_t wpr, int64_t x0, int64_t dom_z,
               int64_t* codes, cudaStream_t st) {
  if (wpr <= 0 || wpr % 32 != 0) {
    set_error("emit: bitmap pitch must be a positive multiple of 32 words");
    return MMJ_ERR_ARG;
  }
  const int64_t nseg = rows * wpr / 32;
  if (nseg == 0) return MMJ_OK;
  k_emit_pf16<EM_SEGS><<<(unsigned)ceil_div(nseg, EM_SEGS), EM_WARPS * 32, 0, st>>>(bm, segoff, nseg, wpr / 32, x0,
                                                                                 dom_z, codes);
  MMJ_CHECK_LAUNCH("k_emit_pf16");
  return MMJ_OK;
}

}  // namespace mmj
