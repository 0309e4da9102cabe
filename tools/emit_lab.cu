// Emission micro-lab: bitmap -> sorted int64 codes, several inner-loop
// variants on a synthetic bitmap, timed with CUDA events.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o emit_lab tools/emit_lab.cu && ./emit_lab
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int WARPS = 8;
constexpr int SEGS_PER_CTA = 64;     // 2048 words = one 8 KB tile

__device__ __forceinline__ void st_cs2(int64_t* p, int64_t a, int64_t b) {
  asm volatile("st.global.cs.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st_cs(int64_t* p, int64_t a) {
  asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ void st_wb2(int64_t* p, int64_t a, int64_t b) {
  asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void st_cs4(int64_t* p, int64_t a, int64_t b, int64_t c, int64_t d) {
  asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st_wb4(int64_t* p, int64_t a, int64_t b, int64_t c, int64_t d) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st_na4(int64_t* p, int64_t a, int64_t b, int64_t c, int64_t d) {
  asm volatile("st.global.L1::no_allocate.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

__device__ __forceinline__ int warp_incl(int c, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, c, o);
    if (lane >= o) c += v;
  }
  return c;
}

// V: variant id
template <int V, int SEGS = SEGS_PER_CTA, int ORDER = 0>
__global__ void __launch_bounds__(WARPS * 32) k_emit(const uint32_t* __restrict__ bm, const int64_t* __restrict__ segoff,
                                                     int64_t nseg, int64_t* __restrict__ out_all) {
  __shared__ __align__(16) uint32_t stage_all[WARPS][1024 + 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* stage = stage_all[warp];
  const int64_t s0 = (int64_t)blockIdx.x * SEGS;
  for (int j = 0; j < SEGS / WARPS; ++j) {
    const int si = ORDER == 0 ? warp + j * WARPS : warp * (SEGS / WARPS) + j;
    const int64_t s = s0 + si;
    if (s >= nseg) break;
    uint32_t word = bm[s * 32 + lane];
    const int c = __popc(word);
    const int incl = warp_incl(c, lane);
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    int64_t* out = out_all + segoff[s];
    const int64_t base = s * 1024;        // code = base + lane*32 + bit
    const uint32_t off0 = lane * 32;
    if (V == 0) {  // LSB ffs, xor5 swizzle, pairs
      int k = incl - c;
      while (word) {
        const int b = __ffs(word) - 1;
        const int kk = k ^ ((k >> 5) & 31);
        stage[kk] = off0 + b;
        ++k;
        word &= word - 1;
      }
      __syncwarp();
      const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), tot);
      auto sl = [](int q) { return q ^ ((q >> 5) & 31); };
      if (lane < h) st_cs(out + lane, base + stage[sl(lane)]);
      const int np = (tot - h) >> 1;
      for (int p = lane; p < np; p += 32) {
        const int i = h + 2 * p;
        st_cs2(out + i, base + stage[sl(i)], base + stage[sl(i + 1)]);
      }
      const int done = h + 2 * np;
      if (lane < tot - done) st_cs(out + done + lane, base + stage[sl(done + lane)]);
    } else if (V == 1 || V == 2 || V == 3) {  // quad swizzle + LDS.128; V1 MSB, V2 LSB, V3 = V2 with write-back stores
      const int h = (int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1);
      auto sl = [](int q) { return q ^ ((q >> 3) & 0x1C); };
      if (V == 1) {
        int k = incl - 1 + h;
        while (word) {
          const int b = 31 - __clz(word);
          stage[sl(k)] = off0 + b;
          --k;
          word ^= 1u << b;
        }
      } else {
        int k = incl - c + h;
        while (word) {
          const int b = __ffs(word) - 1;
          stage[sl(k)] = off0 + b;
          ++k;
          word &= word - 1;
        }
      }
      __syncwarp();
      const int endk = tot + h;
      if (lane >= h && lane < 4 && lane < endk) st_cs(out + lane - h, base + stage[sl(lane)]);
      const int nq = endk >> 2;
      for (int q = 1 + lane; q < nq; q += 32) {
        const uint4 v = *reinterpret_cast<const uint4*>(&stage[sl(4 * q)]);
        int64_t* o = out + 4 * q - h;
        if (V == 3) {
          st_wb2(o, base + v.x, base + v.y);
          st_wb2(o + 2, base + v.z, base + v.w);
        } else {
          st_cs2(o, base + v.x, base + v.y);
          st_cs2(o + 2, base + v.z, base + v.w);
        }
      }
      const int tail = max(4, nq << 2);
      if (tail + lane < endk) st_cs(out + tail + lane - h, base + stage[sl(tail + lane)]);
    } else if (V == 8) {  // V0 staging (lsb, xor5) + 32 B quad stores
      int k = incl - c;
      while (word) {
        const int b = __ffs(word) - 1;
        stage[k ^ ((k >> 5) & 31)] = off0 + b;
        ++k;
        word &= word - 1;
      }
      __syncwarp();
      auto sl = [](int q) { return q ^ ((q >> 5) & 31); };
      const int h = min((int)((4 - ((reinterpret_cast<uintptr_t>(out) >> 3) & 3)) & 3), tot);
      if (lane < h) st_cs(out + lane, base + stage[sl(lane)]);
      const int nq = (tot - h) >> 2;
      for (int q = lane; q < nq; q += 32) {
        const int i = h + 4 * q;
        st_wb4(out + i, base + stage[sl(i)], base + stage[sl(i + 1)], base + stage[sl(i + 2)], base + stage[sl(i + 3)]);
      }
      const int done = h + 4 * nq;
      if (lane < tot - done) st_cs(out + done + lane, base + stage[sl(done + lane)]);
    } else if (V == 9) {  // two bits per iteration
      int k = incl - c;
      while (word) {
        const int b0 = __ffs(word) - 1;
        word &= word - 1;
        const int b1 = __ffs(word) - 1;   // -1 when exhausted
        word &= word - 1;
        stage[k ^ ((k >> 5) & 31)] = off0 + b0;
        if (b1 >= 0) stage[(k + 1) ^ (((k + 1) >> 5) & 31)] = off0 + b1;
        k += 2;
      }
      __syncwarp();
      const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), tot);
      auto sl = [](int q) { return q ^ ((q >> 5) & 31); };
      if (lane < h) st_cs(out + lane, base + stage[sl(lane)]);
      const int np = (tot - h) >> 1;
      for (int p = lane; p < np; p += 32) {
        const int i = h + 2 * p;
        st_cs2(out + i, base + stage[sl(i)], base + stage[sl(i + 1)]);
      }
      const int done = h + 2 * np;
      if (lane < tot - done) st_cs(out + done + lane, base + stage[sl(done + lane)]);
    } else if (V == 10) {  // 16-bit offsets, two per 32-bit store; reader takes 32-bit pairs
      uint16_t* st16 = reinterpret_cast<uint16_t*>(stage);
      auto sl32 = [](int q) { return q ^ ((q >> 5) & 31); };   // swizzle on 32-bit word index
      int k = incl - c;
      if ((k & 1) && word) {          // odd start: one 16-bit store to align
        const int b = __ffs(word) - 1;
        word &= word - 1;
        st16[2 * sl32(k >> 1) + 1] = (uint16_t)(off0 + b);
        ++k;
      }
      while (word) {
        const int b0 = __ffs(word) - 1;
        word &= word - 1;
        if (word) {
          const int b1 = __ffs(word) - 1;
          word &= word - 1;
          stage[sl32(k >> 1)] = (off0 + b0) | ((off0 + b1) << 16);
          k += 2;
        } else {
          st16[2 * sl32(k >> 1)] = (uint16_t)(off0 + b0);
          ++k;
        }
      }
      __syncwarp();
      const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), tot);
      if (lane < h) st_cs(out + lane, base + st16[2 * sl32(0)]);
      const int np = (tot - h) >> 1;
      for (int p = lane; p < np; p += 32) {
        const int i = h + 2 * p;
        uint32_t lo, hi;
        if ((i & 1) == 0) {
          const uint32_t w2 = stage[sl32(i >> 1)];
          lo = w2 & 0xFFFFu;
          hi = w2 >> 16;
        } else {
          lo = st16[2 * sl32(i >> 1) + 1];
          hi = st16[2 * sl32((i + 1) >> 1)];
        }
        st_cs2(out + i, base + lo, base + hi);
      }
      const int done = h + 2 * np;
      if (lane < tot - done) {
        const int i = done + lane;
        st_cs(out + i, base + st16[2 * sl32(i >> 1) + (i & 1)]);
      }
    } else if (V == 13 || V == 14) {  // round robin, no staging: word i's codes by all lanes (lane = bit)
      __shared__ __align__(16) uint2 pairs_all[WARPS][32];
      uint2* pairs = pairs_all[warp];
      pairs[lane] = make_uint2(word, (uint32_t)(incl - c));
      __syncwarp();
      const uint32_t bit = 1u << lane, lt = bit - 1u;
      const int64_t cv = base + lane;
      const uint32_t lo0 = (uint32_t)cv, hi = (uint32_t)((uint64_t)cv >> 32);
      if (V == 13 && (uint32_t)base <= 0xFFFFFFFFu - 1024u) {
        // no carry out of the low word inside the segment: 32-bit code arithmetic
        int64_t* ob;
        asm("mov.b64 %0, %1;" : "=l"(ob) : "l"(out));   // opaque base: one IMAD.WIDE per address
#pragma unroll 4
        for (int i = 0; i < 32; i += 2) {
          const uint4 q = *reinterpret_cast<const uint4*>(pairs + i);
          int64_t* p0 = ob + (q.y + __popc(q.x & lt));
          int64_t* p1 = ob + (q.w + __popc(q.z & lt));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %1, 0;\n\t@p st.global.cs.v2.b32 [%0], {%2, %3};\n\t}"
                       ::"l"(p0), "r"(q.x & bit), "r"(lo0 + 32u * i), "r"(hi) : "memory");
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %1, 0;\n\t@p st.global.cs.v2.b32 [%0], {%2, %3};\n\t}"
                       ::"l"(p1), "r"(q.z & bit), "r"(lo0 + 32u * (i + 1)), "r"(hi) : "memory");
        }
      } else
#pragma unroll 4
      for (int i = 0; i < 32; i += 2) {
        const uint4 q = *reinterpret_cast<const uint4*>(pairs + i);
        if ((q.x | q.z) == 0) continue;
        if (V == 13) {
          if (q.x & bit) st_cs(out + q.y + __popc(q.x & lt), cv + 32 * i);
          if (q.z & bit) st_cs(out + q.w + __popc(q.z & lt), cv + 32 * (i + 1));
        } else {
          if (q.x & bit) out[q.y + __popc(q.x & lt)] = cv + 32 * i;
          if (q.z & bit) out[q.w + __popc(q.z & lt)] = cv + 32 * (i + 1);
        }
      }
    } else if (V == 4) {  // no staging: each lane writes its own run (uncoalesced)
      int k = incl - c;
      while (word) {
        const int b = __ffs(word) - 1;
        st_cs(out + k, base + off0 + b);
        ++k;
        word &= word - 1;
      }
    } else if (V == 5) {  // store ceiling: write tot codes from registers, no expansion
      const int h = (int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1);
      for (int i = h + 2 * lane; i + 1 < tot; i += 64) st_cs2(out + i, base + i, base + i + 1);
    } else if (V == 6) {  // unstaged pairs: no swizzle (conflicts) LSB
      int k = incl - c;
      while (word) {
        const int b = __ffs(word) - 1;
        stage[k] = off0 + b;
        ++k;
        word &= word - 1;
      }
      __syncwarp();
      const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), tot);
      if (lane < h) st_cs(out + lane, base + stage[lane]);
      const int np = (tot - h) >> 1;
      for (int p = lane; p < np; p += 32) {
        const int i = h + 2 * p;
        st_cs2(out + i, base + stage[i], base + stage[i + 1]);
      }
      const int done = h + 2 * np;
      if (lane < tot - done) st_cs(out + done + lane, base + stage[done + lane]);
    } else if (V == 7) {  // byte-parallel: lane handles 8 bits x 4 bytes with per-byte prefix (shared LUT-free)
      // each lane walks its word in two 16-bit halves interleaved to shorten the dependency chain
      int k0 = incl - c;
      uint32_t lo = word & 0xFFFFu, hi = word >> 16;
      int k1 = k0 + __popc(lo);
      while (lo | hi) {
        if (lo) {
          const int b = __ffs(lo) - 1;
          stage[k0 ^ ((k0 >> 5) & 31)] = off0 + b;
          ++k0;
          lo &= lo - 1;
        }
        if (hi) {
          const int b = __ffs(hi) + 15;
          stage[k1 ^ ((k1 >> 5) & 31)] = off0 + b;
          ++k1;
          hi &= hi - 1;
        }
      }
      __syncwarp();
      const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), tot);
      auto sl = [](int q) { return q ^ ((q >> 5) & 31); };
      if (lane < h) st_cs(out + lane, base + stage[sl(lane)]);
      const int np = (tot - h) >> 1;
      for (int p = lane; p < np; p += 32) {
        const int i = h + 2 * p;
        st_cs2(out + i, base + stage[sl(i)], base + stage[sl(i + 1)]);
      }
      const int done = h + 2 * np;
      if (lane < tot - done) st_cs(out + done + lane, base + stage[sl(done + lane)]);
    }
    __syncwarp();
  }
}

// V12: CTA of 8 warps stages its 8 segments' int64 codes contiguously in
// shared memory, then all 256 threads write the CTA range with 16 B stores
__global__ void __launch_bounds__(256) k_emit_cta(const uint32_t* __restrict__ bm, const int64_t* __restrict__ segoff,
                                                  int64_t nseg, int64_t* __restrict__ out_all) {
  extern __shared__ __align__(16) int64_t cstage[];      // 8192 codes worst case
  __shared__ int s_cnt[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t s = (int64_t)blockIdx.x * 8 + warp;
  uint32_t word = s < nseg ? bm[s * 32 + lane] : 0u;
  const int c = __popc(word);
  const int incl = warp_incl(c, lane);
  if (lane == 31) s_cnt[warp] = incl;
  __syncthreads();
  int wbase = 0, total = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const int v = s_cnt[w];
    if (w < warp) wbase += v;
    total += v;
  }
  const int64_t base = s * 1024;
  const uint32_t off0 = lane * 32;
  int k = wbase + incl - c;
  while (word) {
    const int b = __ffs(word) - 1;
    cstage[k ^ (((k >> 4) & 7) << 1)] = base + off0 + b;   // keep pairs, spread lanes over banks
    ++k;
    word &= word - 1;
  }
  __syncthreads();
  const int64_t s0 = (int64_t)blockIdx.x * 8;
  int64_t* out = out_all + segoff[s0];
  const int h = min((int)((reinterpret_cast<uintptr_t>(out) >> 3) & 1), total);
  auto sl = [](int q) { return q ^ (((q >> 4) & 7) << 1); };
  if (threadIdx.x < h) st_cs(out, cstage[sl(0)]);
  const int np = (total - h) >> 1;
  for (int p = threadIdx.x; p < np; p += 256) {
    const int i = h + 2 * p;
    st_cs2(out + i, cstage[sl(i)], cstage[sl(i + 1)]);
  }
  const int done = h + 2 * np;
  if (threadIdx.x < total - done) st_cs(out + done + threadIdx.x, cstage[sl(done + threadIdx.x)]);
}

// pure store kernels: the HBM write ceiling for different store shapes
template <int W>
__global__ void __launch_bounds__(256) k_store(int64_t* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i * 2 * W < n; i += stride) {
    int64_t* p = out + i * 2 * W;
    if (W == 1) {
      st_cs2(p, i, i + 1);
    } else if (W == 2) {   // 32 B per thread, two 16 B stores
      st_cs2(p, i, i + 1);
      st_cs2(p + 2, i + 2, i + 3);
    } else if (W == 3) {
      st_wb2(p, i, i + 1);
    }
  }
}

template <int W>
__global__ void __launch_bounds__(256) k_store4(int64_t* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i * 4 < n; i += stride) {
    int64_t* p = out + i * 4;
    if (W == 0) st_cs4(p, i, i + 1, i + 2, i + 3);
    else if (W == 1) st_wb4(p, i, i + 1, i + 2, i + 3);
    else st_na4(p, i, i + 1, i + 2, i + 3);
  }
}

// block-contiguous: CTA b writes [b*CH, (b+1)*CH) with 32 B per thread per step
template <int CH_ELEMS>
__global__ void __launch_bounds__(256) k_store_blk(int64_t* __restrict__ out, int64_t n) {
  const int64_t base = (int64_t)blockIdx.x * CH_ELEMS;
#pragma unroll 4
  for (int j = threadIdx.x * 4; j < CH_ELEMS; j += 256 * 4) {
    const int64_t i = base + j;
    if (i + 3 < n) st_wb4(out + i, i, i + 1, i + 2, i + 3);
  }
}

template <int CH>
float run_blk(int64_t* out, int64_t n) {
  const int grid = (int)((n + CH - 1) / CH);
  k_store_blk<CH><<<grid, 256>>>(out, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_store_blk<CH><<<grid, 256>>>(out, n);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

template <int W>
float run_store4(int64_t* out, int64_t n) {
  const int grid = 148 * 8;
  k_store4<W><<<grid, 256>>>(out, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_store4<W><<<grid, 256>>>(out, n);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

template <int W>
float run_store(int64_t* out, int64_t n) {
  const int grid = 148 * 8;
  k_store<W><<<grid, 256>>>(out, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_store<W><<<grid, 256>>>(out, n);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

template <int V, int SEGS = SEGS_PER_CTA, int ORDER = 0>
float run(const uint32_t* bm, const int64_t* segoff, int64_t nseg, int64_t* out) {
  const int grid = (int)((nseg + SEGS - 1) / SEGS);
  k_emit<V, SEGS, ORDER><<<grid, WARPS * 32>>>(bm, segoff, nseg, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_emit<V, SEGS, ORDER><<<grid, WARPS * 32>>>(bm, segoff, nseg, out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const double density = argc > 1 ? atof(argv[1]) : 0.49;
  const int64_t nwords = 1ll << 27;   // 4.3e9 cells, ~2.1e9 codes at 49%
  const int64_t nseg = nwords / 32;
  std::vector<uint32_t> h(nwords);
  std::vector<int64_t> so(nseg + 1);
  uint64_t st = 88172645463325252ull;
  int64_t acc = 0;
  for (int64_t s = 0; s < nseg; ++s) {
    so[s] = acc;
    for (int l = 0; l < 32; ++l) {
      uint32_t w = 0;
      for (int b = 0; b < 32; ++b) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        if ((double)(st >> 11) * (1.0 / 9007199254740992.0) < density) w |= 1u << b;
      }
      h[s * 32 + l] = w;
      acc += __builtin_popcount(w);
    }
  }
  so[nseg] = acc;
  uint32_t* dbm;
  int64_t *dso, *dout;
  CK(cudaMalloc(&dbm, nwords * 4));
  CK(cudaMalloc(&dso, (nseg + 1) * 8));
  CK(cudaMalloc(&dout, acc * 8 + 64));
  CK(cudaMemcpy(dbm, h.data(), nwords * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dso, so.data(), (nseg + 1) * 8, cudaMemcpyHostToDevice));
  const double bytes = acc * 8.0;
  printf("density %.2f codes %lld (%.1f GB)\n", density, (long long)acc, bytes / 1e9);
  {
    float a = run<0, 8>(dbm, dso, nseg, dout), b = run<0, 16>(dbm, dso, nseg, dout), c = run<0, 256>(dbm, dso, nseg, dout);
    float d = run<0, 64, 1>(dbm, dso, nseg, dout), e = run<0, 256, 1>(dbm, dso, nseg, dout), f = run<0, 1024, 1>(dbm, dso, nseg, dout);
    printf("V0 segs 8 / 16 / 256 (interleaved): %.1f %.1f %.1f GB/s\n", bytes / (a * 1e-3) / 1e9, bytes / (b * 1e-3) / 1e9, bytes / (c * 1e-3) / 1e9);
    printf("V0 segs 64 / 256 / 1024 (contiguous per warp): %.1f %.1f %.1f GB/s\n", bytes / (d * 1e-3) / 1e9, bytes / (e * 1e-3) / 1e9, bytes / (f * 1e-3) / 1e9);
  }
  {
    cudaFuncSetAttribute(k_emit_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const int grid = (int)((nseg + 7) / 8);
    k_emit_cta<<<grid, 256, 65536>>>(dbm, dso, nseg, dout);
    CK(cudaDeviceSynchronize());
    cudaEvent_t ea, eb;
    cudaEventCreate(&ea);
    cudaEventCreate(&eb);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(ea);
      k_emit_cta<<<grid, 256, 65536>>>(dbm, dso, nseg, dout);
      cudaEventRecord(eb);
      CK(cudaEventSynchronize(eb));
      float ms;
      cudaEventElapsedTime(&ms, ea, eb);
      if (ms < best) best = ms;
    }
    printf("%-24s %8.3f ms  %7.1f GB/s\n", "V12 CTA-staged int64", best, bytes / (best * 1e-3) / 1e9);
  }
  {
    const float r0 = run<13>(dbm, dso, nseg, dout), r1 = run<14>(dbm, dso, nseg, dout);
    const float r2 = run<13, 8>(dbm, dso, nseg, dout), r3 = run<0, 8>(dbm, dso, nseg, dout);
    const float r4 = run<13, 256, 1>(dbm, dso, nseg, dout);
    printf("%-24s %8.3f ms  %7.1f GB/s\n", "V13 round robin cs", r0, bytes / (r0 * 1e-3) / 1e9);
    printf("%-24s %8.3f ms  %7.1f GB/s\n", "V14 round robin wb", r1, bytes / (r1 * 1e-3) / 1e9);
    printf("%-24s %8.3f ms  %7.1f GB/s\n", "V13 segs 8", r2, bytes / (r2 * 1e-3) / 1e9);
    printf("%-24s %8.3f ms  %7.1f GB/s\n", "V0 segs 8", r3, bytes / (r3 * 1e-3) / 1e9);
    printf("%-24s %8.3f ms  %7.1f GB/s\n", "V13 256 contiguous/warp", r4, bytes / (r4 * 1e-3) / 1e9);
    // parity of V13 vs V0
    std::vector<int64_t> o0(acc), o1(acc);
    run<0>(dbm, dso, nseg, dout);
    CK(cudaMemcpy(o0.data(), dout, acc * 8, cudaMemcpyDeviceToHost));
    run<13>(dbm, dso, nseg, dout);
    CK(cudaMemcpy(o1.data(), dout, acc * 8, cudaMemcpyDeviceToHost));
    printf("V13 == V0: %s\n", o0 == o1 ? "yes" : "NO");
  }
  const float t8 = run<8>(dbm, dso, nseg, dout);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "V8 xor5 + 32B quads", t8, bytes / (t8 * 1e-3) / 1e9);
  const float t9 = run<9>(dbm, dso, nseg, dout);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "V9 2 bits/iter", t9, bytes / (t9 * 1e-3) / 1e9);
  const float t10 = run<10>(dbm, dso, nseg, dout);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "V10 16-bit staging", t10, bytes / (t10 * 1e-3) / 1e9);
  const char* names[] = {"V0 lsb xor5 pairs", "V1 msb quad LDS128", "V2 lsb quad LDS128", "V3 V2 + wb stores",
                         "V4 unstaged lane runs", "V5 store ceiling", "V6 unswizzled pairs", "V7 2-chain xor5"};
  float t[8];
  t[0] = run<0>(dbm, dso, nseg, dout);
  t[1] = run<1>(dbm, dso, nseg, dout);
  t[2] = run<2>(dbm, dso, nseg, dout);
  t[3] = run<3>(dbm, dso, nseg, dout);
  t[4] = run<4>(dbm, dso, nseg, dout);
  t[5] = run<5>(dbm, dso, nseg, dout);
  t[6] = run<6>(dbm, dso, nseg, dout);
  t[7] = run<7>(dbm, dso, nseg, dout);
  for (int v = 0; v < 8; ++v) printf("%-24s %8.3f ms  %7.1f GB/s\n", names[v], t[v], bytes / (t[v] * 1e-3) / 1e9);
  const float s1 = run_store<1>(dout, acc), s2 = run_store<2>(dout, acc), s3 = run_store<3>(dout, acc);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "store 16B cs", s1, bytes / (s1 * 1e-3) / 1e9);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "store 2x16B cs", s2, bytes / (s2 * 1e-3) / 1e9);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "store 16B wb", s3, bytes / (s3 * 1e-3) / 1e9);
  const float q0 = run_store4<0>(dout, acc), q1 = run_store4<1>(dout, acc), q2 = run_store4<2>(dout, acc);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "store 32B cs", q0, bytes / (q0 * 1e-3) / 1e9);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "store 32B wb", q1, bytes / (q1 * 1e-3) / 1e9);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "store 32B L1::no_alloc", q2, bytes / (q2 * 1e-3) / 1e9);
  const float b1 = run_blk<4096>(dout, acc), b2 = run_blk<16384>(dout, acc), b3 = run_blk<65536>(dout, acc);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "blk 32KB", b1, bytes / (b1 * 1e-3) / 1e9);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "blk 128KB", b2, bytes / (b2 * 1e-3) / 1e9);
  printf("%-24s %8.3f ms  %7.1f GB/s\n", "blk 512KB", b3, bytes / (b3 * 1e-3) / 1e9);
  return 0;
}
