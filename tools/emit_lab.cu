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

__device__ __forceinline__ int warp_incl(int c, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, c, o);
    if (lane >= o) c += v;
  }
  return c;
}

// V: variant id
template <int V>
__global__ void __launch_bounds__(WARPS * 32) k_emit(const uint32_t* __restrict__ bm, const int64_t* __restrict__ segoff,
                                                     int64_t nseg, int64_t* __restrict__ out_all) {
  __shared__ __align__(16) uint32_t stage_all[WARPS][1024 + 8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* stage = stage_all[warp];
  const int64_t s0 = (int64_t)blockIdx.x * SEGS_PER_CTA;
  for (int si = warp; si < SEGS_PER_CTA; si += WARPS) {
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

template <int V>
float run(const uint32_t* bm, const int64_t* segoff, int64_t nseg, int64_t* out) {
  const int grid = (int)((nseg + SEGS_PER_CTA - 1) / SEGS_PER_CTA);
  k_emit<V><<<grid, WARPS * 32>>>(bm, segoff, nseg, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_emit<V><<<grid, WARPS * 32>>>(bm, segoff, nseg, out);
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
  return 0;
}
