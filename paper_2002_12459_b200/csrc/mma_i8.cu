// Heavy-part contraction on the 5th-generation tensor cores.
//
// Replaces the reference's dense heavy product
//   joinproject.py:208-216  (multiply_counts(M1, M2) -> nonzero)
//   matmul/core.py:95-123   (float64 BLAS / int64 Cython kernel, _kernel_cy.pyx:14-47)
// with a persistent, warp-specialised tcgen05 kernel:
//   * operands: uint8 matrices A[rows][Kp] and B[cols][Kp], both K-major
//     (B is "S_h transposed": one row per z), staged by TMA into 128B-swizzled
//     shared-memory tiles through a 4-deep mbarrier ring;
//   * math: tcgen05.mma.cta_group::1.kind::i8, M=128 N=256 K=32 per
//     instruction, unsigned 8-bit inputs, exact s32 accumulators in TMEM
//     (two 256-column accumulator stages so tile i's epilogue overlaps
//     tile i+1's MMAs);
//   * epilogue (4 warps, TMEM -> registers via tcgen05.ld):
//       BITMAP : nonzero test, 32 cells -> one 32-bit word, 32 B per row/tile
//                (the projection / intersection output);
//       COUNT32: exact int32 counts (witness counts / set overlaps);
//       COUNT16: the same as uint16 when every count is < 2^16 (half the bytes);
//       ACC64  : out[i][j] += count << shift  (int64 digit recombination for
//                the generic multiply_counts backend);
//       BITMAP_PAIR: B rows are z pairs weighted (1, 128) (mmj_build_operand_pairs),
//                one accumulator = two cells: half the MMAs and half the TMEM
//                read-out per output bit, 64 B per row/tile (a z-triple
//                form, three 7-bit fields per accumulator, measured slower:
//                35.1 vs 26.5 ms on cfg2, its packing is ALU-bound).
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator,
// w3 idle, w4..w11 epilogue (warp w owns TMEM lanes 32*(w%4) .. +31 and the
// 128-column half (w-4)/4 of the accumulator).  The ring depth is chosen per
// launch (2 stages when a tile has <= 2 K blocks).

#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdlib.h>

#include "mmj_common.cuh"

namespace mmj {
namespace mma {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 128;                 // bytes (= uint8 elements) of K per stage
constexpr int UMMA_K = 32;              // K per tcgen05.mma for kind::i8
constexpr int STAGES = 4;                // maximum ring depth (the launch picks 2..4)
constexpr int A_BYTES = BM * BK;        // 16 KB
constexpr int B_BYTES = BN * BK;        // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int ACC_STAGES = 2;
constexpr int TMEM_COLS = 512;          // 2 x 256 s32 accumulator columns
// 8 epilogue warps (128 columns each); 16 (64 columns, 640 threads) measured
// no faster: the epilogue is bound by the TMEM read-out (128 rows x 256
// columns x 4 B per tile at ~64 B/clk), not by its instruction latency
#ifndef MMJ_EPI_WARPS
#define MMJ_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = MMJ_EPI_WARPS;  // 4 x EPI_GROUPS: one warp per (TMEM lane quadrant, column group)
constexpr int EPI_GROUPS = EPI_WARPS / 4;
constexpr int CW = 256 / EPI_GROUPS;      // accumulator columns per epilogue warp
constexpr int NUM_THREADS = 128 + 32 * EPI_WARPS;
static_assert(CW == 64 || CW == 128, "epilogue column split");
constexpr int EPI_PITCH = 36;           // COUNT32 staging: words per row (16-B aligned, conflict-free v4)
constexpr int EPI_STAGE_BYTES = EPI_WARPS * 32 * EPI_PITCH * 4;
constexpr int smem_bytes_for(int stages, bool staged) {
  return stages * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + (staged ? EPI_STAGE_BYTES : 0);
}
constexpr int SMEM_MAX = smem_bytes_for(3, true) > smem_bytes_for(STAGES, false) ? smem_bytes_for(3, true)
                                                                                  : smem_bytes_for(STAGES, false);
static_assert(SMEM_MAX <= 227 * 1024, "shared memory budget");
constexpr int GROUP_M = 16;             // raster: sweep N for a band of 16 M blocks

enum Mode : int { BITMAP = 0, COUNT32 = 1, ACC64 = 2, BITMAP_U8 = 3, BITMAP_PAIR = 4, COUNT16 = 5, MODE_UPPER = 16 };

struct Params {
  int64_t m_begin;      // first A row of this launch (multiple of BM not required)
  int upper;            // skip tiles strictly below the x = z diagonal
  int backoff;          // producer / MMA issuer sleep between barrier polls
  int64_t m_rows;       // rows of A processed / rows of the output
  int64_t n_cols;       // columns of the product (= rows of B)
  int num_kb;           // Kp / BK
  int stages;           // smem ring depth (2..STAGES)
  int alt;              // BITMAP_PAIR: alternating epilogue warp groups
  int small_counts;     // BITMAP: every product entry < 256 (K window <= 255 nonzero columns)
  int mode;
  int shift;            // ACC64 only
  void* out;            // BITMAP: uint32 words, COUNT32: int32, ACC64: int64
  int64_t ld_out;       // row pitch of out in elements (words / int32 / int64)
  unsigned long long* nnz;   // BITMAP/COUNT32: nonzero cells found (may be null)
};

// ---------------------------------------------------------------- PTX wraps
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Same wait with a short sleep between polls: used by the single-thread TMA
// producer and MMA issuer so their spinning does not take issue slots from
// the epilogue warps sharing their SM sub-partitions.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  while (!ok) {
    __nanosleep(32);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// K-major operand tile, 128-byte rows, 128B swizzle, 8-row core groups 1 KB apart.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);   // start address
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                    // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

// kind::i8 instruction descriptor: D=s32, A=B=u8, both K-major, M=128, N=256.
__host__ __device__ constexpr uint32_t idesc_u8_s32(int m, int n) {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

#define TMEM_LD_32x32b_X32(taddr, r)                                                            \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"   \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"         \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),     \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),           \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),           \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])            \
      : "r"(taddr))

// 32 lanes x 64 columns, adjacent column pairs packed into one register as
// two 16-bit halves (low half = even column).  The accumulators are exact
// counts < 2^16 here (K windows <= 32768 with 0/1 operands in BITMAP mode).
#define TMEM_LD_32x32b_X32_PACK16(taddr, r)                                                     \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"  \
      "%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),     \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),           \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),           \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])            \
      : "r"(taddr))

// 16 pack::16b registers (32 columns, counts < 256) -> 32-bit nonzero mask
__device__ __forceinline__ uint32_t pack_bits_u8(const uint32_t* r) {
  uint32_t w = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t p = __byte_perm(r[2 * j], r[2 * j + 1], 0x6420);          // [c3 c2 c1 c0]
    const uint32_t nz = (((p & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | p) & 0x80808080u;   // byte MSB = (c != 0)
    w |= ((nz * 0x00204081u) >> 28) << (4 * j);                                // bits 7,15,23,31 -> 4 bits
  }
  return w;
}

// 16 pack::16b registers (32 columns, counts < 2^16) -> 32-bit nonzero mask
__device__ __forceinline__ uint32_t pack_bits_u16(const uint32_t* r) {
  uint32_t w = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t nz = (((r[i] & 0x7FFF7FFFu) + 0x7FFF7FFFu) | r[i]) & 0x80008000u;
    w |= ((nz * 0x8001u) >> 30) << (2 * i);                                     // bits 15,31 -> 2 bits
  }
  return w;
}

// BITMAP_PAIR: every B row holds two z cells weighted (1, 128), so an
// accumulator is c0 + 128*c1 with c0, c1 < 128 (the caller guarantees a side
// whose heavy degrees are <= 127).  The operand builder places z = 32G + b
// (b = k + 8j, k < 8, j < 4) in accumulator column 16G + 2k + (j >> 1), slot
// j & 1, so that after the per-register flag test (flags at bits 7, 15, 23,
// 31) a right-shift-and-or chain lands every flag on its own bit:
// 8 pack::16b registers = 16 accumulator columns = one 32-bit word.
__device__ __forceinline__ uint32_t pair_flags(uint32_t r) {
  const uint32_t lo = (r & 0x007F007Fu) + 0x007F007Fu;   // c0 != 0 -> bits 7, 23 (no bits above 7 per half)
  const uint32_t hi = r + 0x7F807F80u;                   // v >= 128 (c1 != 0) -> bits 15, 31; no carry
                                                         // out of the low half since v < 2^14
  return (lo & 0x00800080u) | (hi & 0x80008000u);
}

__device__ __forceinline__ uint32_t pack_bits_pair(const uint32_t* r) {
  uint32_t w = pair_flags(r[0]);
#pragma unroll
  for (int k = 1; k < 8; ++k) w = (w >> 1) + pair_flags(r[k]);   // disjoint bits: + == |
  return w;   // register k's flags now sit at bits k, 8+k, 16+k, 24+k
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct TileCoord {
  int m_blk, n_blk;
};

__device__ __forceinline__ TileCoord tile_of(int64_t t, int mt, int nt) {
  // bands of GROUP_M M-blocks; inside a band walk N, cycling M fastest so the
  // B tile just loaded is reused by the band from L2.  32-bit arithmetic when
  // the tile count allows (the 64-bit divide is a ~40-instruction sequence).
  TileCoord c;
  const uint32_t band_tiles = (uint32_t)GROUP_M * (uint32_t)nt;
  if ((uint64_t)mt * (uint64_t)nt < (1ull << 31)) {
    const uint32_t tt = (uint32_t)t;
    const uint32_t band = tt / band_tiles;
    const uint32_t r = tt - band * band_tiles;
    const int first_m = (int)band * GROUP_M;
    const uint32_t gsz = (uint32_t)min(GROUP_M, mt - first_m);
    const uint32_t nb = r / gsz;
    c.m_blk = first_m + (int)(r - nb * gsz);
    c.n_blk = (int)nb;
  } else {
    const int64_t bt = (int64_t)GROUP_M * nt;
    const int band = (int)(t / bt);
    const int64_t r = t - (int64_t)band * bt;
    const int first_m = band * GROUP_M;
    const int gsz = min(GROUP_M, mt - first_m);
    c.m_blk = first_m + (int)(r % gsz);
    c.n_blk = (int)(r / gsz);
  }
  return c;
}

// Self-join consumers that keep only z > x (SSJ's a < b filter) skip tiles
// whose every column is <= every row: A row m_begin + i is x, B row j is z.
__device__ __forceinline__ bool below_diagonal(const Params& p, TileCoord c) {
  return p.upper && (int64_t)c.n_blk * BN + BN - 1 <= p.m_begin + (int64_t)c.m_blk * BM;
}

// ----------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(NUM_THREADS, 1)
    heavy_mma_kernel(const __grid_constant__ CUtensorMap tmap_a,
                     const __grid_constant__ CUtensorMap tmap_b, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NST = p.stages;
  uint8_t* smem_a = smem;                                   // NST x A_BYTES
  uint8_t* smem_b = smem + NST * A_BYTES;                   // NST x B_BYTES
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE_BYTES);
  uint64_t* full = bars;                                    // [STAGES]
  uint64_t* empty = bars + STAGES;                          // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;                      // [ACC_STAGES]
  uint64_t* tempty = bars + 2 * STAGES + ACC_STAGES;        // [ACC_STAGES]
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2 * ACC_STAGES);
  // COUNT32 int32 blocks (after the barriers)
  uint32_t* epi_stage = reinterpret_cast<uint32_t*>(smem + NST * STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int mt = (int)((p.m_rows + BM - 1) / BM);
  const int nt = (int)((p.n_cols + BN - 1) / BN);
  const int64_t num_tiles = (int64_t)mt * nt;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap_b)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < ACC_STAGES; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], p.alt ? 4 : EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_base_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  if (warp == 0) {
    // ------------------------------------------------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        TileCoord c = tile_of(t, mt, nt);
        if (below_diagonal(p, c)) continue;
        const int32_t arow = (int32_t)(p.m_begin + (int64_t)c.m_blk * BM);
        const int32_t brow = c.n_blk * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          if (p.backoff) mbar_wait_backoff(&empty[s], ph ^ 1); else mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(smem_a + s * A_BYTES, &tmap_a, &full[s], kb * BK, arow);
          tma_load_2d(smem_b + s * B_BYTES, &tmap_b, &full[s], kb * BK, brow);
          if (++s == NST) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_u8_s32(BM, BN);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        if (below_diagonal(p, tile_of(t, mt, nt))) continue;
        if (p.backoff) mbar_wait_backoff(&tempty[acc], acc_ph ^ 1); else mbar_wait(&tempty[acc], acc_ph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem_a + s * A_BYTES);
          const uint32_t b0 = smem_u32(smem_b + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            tc_mma_i8(d_tmem, smem_desc_sw128(a0 + k * UMMA_K), smem_desc_sw128(b0 + k * UMMA_K), idesc,
                      (kb > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[s]);          // smem slot free once these MMAs retire
          if (++s == NST) { s = 0; ph ^= 1; }
        }
        tc_commit(&tfull[acc]);          // accumulator ready for the epilogue
        if (++acc == ACC_STAGES) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else if (warp >= 4 && p.alt) {
    // ------------------------------------------------------- epilogue, alternating groups
    // Warps 4-7 (group 0) take the CTA's even tiles (accumulator stage 0),
    // warps 8-11 (group 1) the odd ones (stage 1), each warp all 256 columns
    // of its TMEM lane quadrant.  The groups run half a tile apart, so one
    // group's packing overlaps the other's TMEM read-out (with both groups on
    // every tile, all warps load, then all pack, and the SM's TMEM read
    // port idles during the packing).
    const int q = warp & 3;
    const int grp = (warp - 4) >> 2;
    uint32_t acc_ph = 0;
    unsigned long long my_nnz = 0;
    int64_t li = 0;
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      TileCoord c = tile_of(t, mt, nt);
      if (below_diagonal(p, c)) continue;
      if ((int)(li++ & 1) != grp) continue;
      const int acc = grp;
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const int64_t row = (int64_t)c.m_blk * BM + q * 32 + lane;
      const bool row_ok = row < p.m_rows;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      {   // BITMAP_PAIR
        constexpr int NW = BN / 16;        // 16 words
        uint32_t w[NW];
        {
#pragma unroll
          for (int j = 0; j < BN / 128; ++j) {
            uint32_t r[64];
            uint32_t* r1 = r + 32;
            TMEM_LD_32x32b_X32_PACK16(taddr + 128 * j, r);
            TMEM_LD_32x32b_X32_PACK16(taddr + 128 * j + 64, r1);
            tmem_wait_ld();
            if (j == BN / 128 - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[acc]);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) w[8 * j + k] = pack_bits_pair(r + 8 * k);
          }
        }
        if (row_ok) {
          uint32_t* dst = reinterpret_cast<uint32_t*>(p.out) + row * p.ld_out + (int64_t)c.n_blk * NW;
#pragma unroll
          for (int k = 0; k < NW; k += 4) {
            *reinterpret_cast<uint4*>(dst + k) = make_uint4(w[k], w[k + 1], w[k + 2], w[k + 3]);
            my_nnz += __popc(w[k]) + __popc(w[k + 1]) + __popc(w[k + 2]) + __popc(w[k + 3]);
          }
        }
      }
      acc_ph ^= 1;
    }
    if (p.nnz != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) my_nnz += __shfl_xor_sync(0xffffffffu, my_nnz, o);
      if (lane == 0 && my_nnz) atomicAdd(p.nnz, my_nnz);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------- epilogue
    const int q = warp & 3;              // TMEM lane quadrant
    const int grp = (warp - 4) >> 2;     // CW-column group of the 256-column tile
    int acc = 0;
    uint32_t acc_ph = 0;
    unsigned long long my_nnz = 0;
    for (int64_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      TileCoord c = tile_of(t, mt, nt);
      if (below_diagonal(p, c)) continue;
      mbar_wait(&tfull[acc], acc_ph);
      tc_fence_after();
      const int64_t row = (int64_t)c.m_blk * BM + q * 32 + lane;   // local output row
      const bool row_ok = row < p.m_rows;
      const int64_t col0 = (int64_t)c.n_blk * BN + grp * CW;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + grp * CW;
      if (p.mode == BITMAP || p.mode == BITMAP_PAIR) {
        constexpr int NR = CW / 2;                   // pack::16b registers (2 columns each)
        uint32_t r[NR];
#pragma unroll
        for (int h = 0; h < NR / 32; ++h) {
          uint32_t* rh = r + 32 * h;
          TMEM_LD_32x32b_X32_PACK16(taddr + 64 * h, rh);
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        // BITMAP: CW columns -> CW/32 words; BITMAP_PAIR: CW accumulators = 2*CW z -> CW/16 words
        const bool pair = (p.mode == BITMAP_PAIR);
        constexpr int NW = CW / 16;
        uint32_t w[NW];
        if (pair) {
#pragma unroll
          for (int k = 0; k < NW; ++k) w[k] = pack_bits_pair(r + 8 * k);
        } else {
#pragma unroll
          for (int k = 0; k < NW / 2; ++k) {
            if (p.small_counts) w[k] = pack_bits_u8(r + 16 * k);    // counts < 256: PRMT + SWAR
            else w[k] = pack_bits_u16(r + 16 * k);
          }
#pragma unroll
          for (int k = NW / 2; k < NW; ++k) w[k] = 0;
        }
        if (row_ok) {
          uint32_t* dst = reinterpret_cast<uint32_t*>(p.out) + row * p.ld_out +
                          (pair ? (int64_t)c.n_blk * 16 + grp * NW : (int64_t)c.n_blk * 8 + grp * (NW / 2));
          if (pair) {
#pragma unroll
            for (int k = 0; k < NW; k += 4)
              *reinterpret_cast<uint4*>(dst + k) = make_uint4(w[k], w[k + 1], w[k + 2], w[k + 3]);
          } else if (NW / 2 >= 4) {
#pragma unroll
            for (int k = 0; k < NW / 2; k += 4)
              *reinterpret_cast<uint4*>(dst + k) = make_uint4(w[k], w[k + 1], w[k + 2], w[k + 3]);
          } else {
            *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
          }
#pragma unroll
          for (int k = 0; k < NW; ++k) my_nnz += __popc(w[k]);
        }
      } else if (p.mode == COUNT16) {
        // counts < 2^16 (caller's guarantee): pack::16b registers hold two
        // cells each; 32 rows x 32 words (64 cells) per block, staged and
        // stored 4 rows (128 B each) per instruction as in COUNT32
        uint32_t* stg = epi_stage + (warp - 4) * 32 * EPI_PITCH;
        const int64_t row_base = (int64_t)c.m_blk * BM + q * 32;
        const int sub_r = lane >> 3, sub_c = (lane & 7) * 4;
        const int64_t ldw = p.ld_out >> 1;                 // words per row
#pragma unroll 1
        for (int j = 0; j < CW / 64; ++j) {
          uint32_t r[32];
          TMEM_LD_32x32b_X32_PACK16(taddr + j * 64, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<uint4*>(stg + lane * EPI_PITCH + i) = make_uint4(r[i], r[i + 1], r[i + 2], r[i + 3]);
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int64_t cc = col0 + j * 64 + 2 * i;
              my_nnz += ((r[i] & 0xFFFFu) != 0u && cc < p.n_cols) + ((r[i] >> 16) != 0u && cc + 1 < p.n_cols);
            }
          }
          __syncwarp();
          const int64_t wcol = ((col0 + j * 64) >> 1) + sub_c;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = sub_r + 4 * i;
            const int64_t orow = row_base + rr;
            const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * EPI_PITCH + sub_c);
            if (orow < p.m_rows && wcol + 4 <= ldw)
              *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(p.out) + orow * ldw + wcol) = v;
          }
          __syncwarp();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else if (p.mode == COUNT32) {
        // 32x32 blocks: lane (= row) stages its 32 counts in shared memory,
        // then the warp stores 4 full rows (128 B each) per instruction.
        uint32_t* stg = epi_stage + (warp - 4) * 32 * EPI_PITCH;
        const int64_t row_base = (int64_t)c.m_blk * BM + q * 32;
        const int sub_r = lane >> 3, sub_c = (lane & 7) * 4;
#pragma unroll 1
        for (int j = 0; j < CW / 32; ++j) {
          uint32_t r[32];
          TMEM_LD_32x32b_X32(taddr + j * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<uint4*>(stg + lane * EPI_PITCH + i) = make_uint4(r[i], r[i + 1], r[i + 2], r[i + 3]);
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i) my_nnz += (r[i] != 0u && col0 + j * 32 + i < p.n_cols);
          }
          __syncwarp();
          const int64_t col = col0 + j * 32 + sub_c;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = sub_r + 4 * i;
            const int64_t orow = row_base + rr;
            const uint4 v = *reinterpret_cast<const uint4*>(stg + rr * EPI_PITCH + sub_c);
            if (orow < p.m_rows && col + 4 <= p.ld_out)
              *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(p.out) + orow * p.ld_out + col) = v;
          }
          __syncwarp();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else {  // ACC64
        int64_t* dst = reinterpret_cast<int64_t*>(p.out) + row * p.ld_out + col0;
#pragma unroll 1
        for (int j = 0; j < CW / 32; ++j) {
          uint32_t r[32];
          TMEM_LD_32x32b_X32(taddr + j * 32, r);
          tmem_wait_ld();
          if (row_ok) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int64_t col = col0 + j * 32 + i;
              if (col < p.n_cols && r[i] != 0u) dst[j * 32 + i] += ((int64_t)r[i]) << p.shift;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      }
      if (++acc == ACC_STAGES) { acc = 0; acc_ph ^= 1; }
    }
    if (p.nnz != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) my_nnz += __shfl_xor_sync(0xffffffffu, my_nnz, o);
      if (lane == 0 && my_nnz) atomicAdd(p.nnz, my_nnz);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ----------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t klen, int64_t pitch, int box_rows) {
  auto enc = get_encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return MMJ_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)klen, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)pitch};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld k=%lld pitch=%lld", (int)r, (long long)rows,
              (long long)klen, (long long)pitch);
    return MMJ_ERR_CUDA;
  }
  return MMJ_OK;
}

int launch_heavy_mma(const uint8_t* a, int64_t a_rows, const uint8_t* b, int64_t b_rows, int64_t kpad,
                     int64_t k_off, int64_t k_len, int64_t m_begin, int64_t m_rows, int mode, int shift, void* out,
                     int64_t ld_out, unsigned long long* nnz, int max_ctas, cudaStream_t st) {
  const int upper = (mode & MODE_UPPER) ? 1 : 0;
  mode &= ~MODE_UPPER;
  if (kpad <= 0 || kpad % BK != 0 || k_off < 0 || k_len <= 0 || k_off % BK != 0 || k_len % BK != 0 ||
      k_off + k_len > kpad) {
    set_error("heavy_mma: K window [%lld,+%lld) of pitch %lld must be multiples of %d", (long long)k_off,
              (long long)k_len, (long long)kpad, BK);
    return MMJ_ERR_ARG;
  }
  if (m_begin < 0 || m_rows < 0 || m_begin + m_rows > a_rows) {
    set_error("heavy_mma: row range [%lld,+%lld) outside A (%lld rows)", (long long)m_begin,
              (long long)m_rows, (long long)a_rows);
    return MMJ_ERR_ARG;
  }
  if (a_rows >= (1ll << 31) || b_rows >= (1ll << 31)) {
    set_error("heavy_mma: operand rows must be < 2^31");
    return MMJ_ERR_ARG;
  }
  if ((mode == BITMAP || mode == BITMAP_U8) && (ld_out % 8 != 0 || ld_out * 32 < round_up(b_rows, BN))) {
    set_error("heavy_mma: bitmap pitch %lld words too small / unaligned", (long long)ld_out);
    return MMJ_ERR_ARG;
  }
  if (mode == BITMAP_PAIR && (ld_out % 8 != 0 || ld_out * 16 < round_up(b_rows, BN))) {
    set_error("heavy_mma: pair-bitmap pitch %lld words too small / unaligned", (long long)ld_out);
    return MMJ_ERR_ARG;
  }
  if (mode == COUNT32 && ld_out % 4 != 0) {
    set_error("heavy_mma: count pitch must be a multiple of 4");
    return MMJ_ERR_ARG;
  }
  if (mode == COUNT16 && ld_out % 8 != 0) {
    set_error("heavy_mma: uint16 count pitch must be a multiple of 8");
    return MMJ_ERR_ARG;
  }
  if (mode < 0 || mode > COUNT16) {
    set_error("heavy_mma: unknown mode %d", mode);
    return MMJ_ERR_ARG;
  }
  if ((mode == BITMAP || mode == BITMAP_U8 || mode == BITMAP_PAIR) && k_len > 65535) {
    set_error("heavy_mma: BITMAP mode packs 16-bit counts; K window must be < 65536");
    return MMJ_ERR_ARG;
  }
  if (m_rows == 0 || b_rows == 0) return MMJ_OK;
  CUtensorMap ma, mb;
  MMJ_TRY(make_map(&ma, a + k_off, a_rows, k_len, kpad, BM));
  MMJ_TRY(make_map(&mb, b + k_off, b_rows, k_len, kpad, BN));

  Params p;
  p.m_begin = m_begin;
  p.upper = upper;
  p.m_rows = m_rows;
  p.n_cols = b_rows;
  p.num_kb = (int)(k_len / BK);
  p.stages = p.num_kb <= 2 ? 2 : STAGES;
  const bool staged = (mode == COUNT32 || mode == COUNT16);
  if (staged && p.stages > 3) p.stages = 3;   // room for the epilogue staging buffers
  p.small_counts = (mode == BITMAP_U8 || k_len <= 255) ? 1 : 0;
  // alternating epilogue groups for the z-pair bitmap (one group packs while
  // the other drains TMEM); the single-thread producer / issuer back off
  // between barrier polls so they do not take issue slots from the epilogue
  p.alt = mode == BITMAP_PAIR ? 1 : 0;
  p.backoff = 1;
  p.mode = mode == BITMAP_U8 ? BITMAP : mode;
  p.shift = shift;
  p.out = out;
  p.ld_out = ld_out;
  p.nnz = nnz;
  MMJ_TRY(set_max_dynamic_smem((const void*)heavy_mma_kernel, SMEM_MAX, "heavy_mma_kernel"));
  const int64_t tiles = ceil_div(m_rows, BM) * ceil_div(b_rows, BN);
  int grid = sm_count();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (tiles < grid) grid = (int)tiles;
  heavy_mma_kernel<<<grid, NUM_THREADS, smem_bytes_for(p.stages, staged), st>>>(ma, mb, p);
  MMJ_CHECK_LAUNCH("heavy_mma_kernel");
  return MMJ_OK;
}

}  // namespace mma
}  // namespace mmj
