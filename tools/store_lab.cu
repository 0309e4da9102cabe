// HBM write-pattern lab: which property of a store stream decides whether it
// reaches the ~7.5 TB/s block-contiguous ceiling or the ~6.0-6.4 TB/s of the
// per-warp segment runs the emission kernels produce?  Pure stores, no
// expansion work.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_lab tools/store_lab.cu && ./tools/store_lab
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ void st1(int64_t* p, int64_t a, bool cs) {
  if (cs) asm volatile("st.global.cs.b64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
  else asm volatile("st.global.b64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ void st2(int64_t* p, int64_t a, int64_t b, bool cs) {
  if (cs) asm volatile("st.global.cs.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
  else asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void st4(int64_t* p, int64_t a, int64_t b, int64_t c, int64_t d, bool cs) {
  if (cs) asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
  else asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// A CTA owns `run` consecutive elements starting at run * blockIdx.x + shift
// (shift in elements: 0 = 32-B aligned ranges).  MODE:
//   0  all threads stream the CTA range together, W elements per lane per store
//   1  warp w writes the w-th of NT/32 consecutive sub-runs (per-warp segments)
//   2  as 1, but sub-runs are taken in round-robin order by the warps, like the
//      emission kernels' dynamic segment hand-out over a whole tile
template <int MODE, int W, bool CS>
__global__ void __launch_bounds__(256) k_pat(int64_t* __restrict__ out, int64_t n, int run, int seg, int shift) {
  const int64_t r0 = (int64_t)blockIdx.x * run + shift;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (MODE == 0) {
    // head to W-element alignment
    int64_t b = r0, e = min(r0 + run, n);
    const int64_t ab = (b + W - 1) / W * W;
    if (threadIdx.x < ab - b && b + threadIdx.x < e) st1(out + b + threadIdx.x, b + threadIdx.x, CS);
    for (int64_t i = ab + (int64_t)threadIdx.x * W; i + W <= e; i += 256 * W) {
      if (W == 4) st4(out + i, i, i + 1, i + 2, i + 3, CS);
      else if (W == 2) st2(out + i, i, i + 1, CS);
      else st1(out + i, i, CS);
    }
    const int64_t tail = ab + (e - ab) / W * W;
    if (tail + threadIdx.x < e) st1(out + tail + threadIdx.x, tail + threadIdx.x, CS);
  } else {
    const int nseg = run / seg;
    for (int s = warp; s < nseg; s += 8) {
      const int64_t b = r0 + (int64_t)s * seg, e = min(b + seg, n);
      if (b >= n) break;
      const int64_t ab = (b + W - 1) / W * W;
      if (lane < ab - b && b + lane < e) st1(out + b + lane, b + lane, CS);
      for (int64_t i = ab + (int64_t)lane * W; i + W <= e; i += 32 * W) {
        if (W == 4) st4(out + i, i, i + 1, i + 2, i + 3, CS);
        else if (W == 2) st2(out + i, i, i + 1, CS);
        else st1(out + i, i, CS);
      }
      const int64_t tail = ab + (e - ab) / W * W;
      if (tail + lane < e) st1(out + tail + lane, tail + lane, CS);
    }
  }
}

// TMA bulk stores: each warp owns consecutive runs of `seg` elements (the
// CTA range as MODE 1); it writes a run's codes into a shared-memory staging
// buffer (8-byte stores, lane = element) in pieces of CH elements and hands
// each piece's 16-B aligned middle to the TMA engine (cp.async.bulk global <-
// shared), head/tail elements with plain stores.  NB staging buffers per warp.
template <int CH, int NB>
__global__ void __launch_bounds__(256) k_tma(int64_t* __restrict__ out, int64_t n, int run, int seg, int shift) {
  extern __shared__ __align__(128) int64_t stg_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t* stg = stg_all + (int64_t)warp * NB * (CH + 2);
  const int64_t r0 = (int64_t)blockIdx.x * run + shift;
  const int nseg = run / seg;
  int buf = 0;
  for (int s = warp; s < nseg; s += 8) {
    const int64_t b = r0 + (int64_t)s * seg, e = min(b + seg, n);
    for (int64_t p0 = b; p0 < e; p0 += CH) {
      const int64_t p1 = min(p0 + CH, e);
      int64_t* sb = stg + buf * (CH + 2);
      // reuse: the bulk copy that read this buffer NB pieces ago has finished reading
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 1) : "memory");
      __syncwarp();
      const int a = (int)(p0 & 1);               // 16-B phase of the piece's first element
      for (int64_t i = p0 + lane; i < p1; i += 32) sb[a + (i - p0)] = i;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        int64_t m0 = p0 + a, m1 = p1 - ((p1 - m0) & 1);   // aligned middle [m0, m1)
        if (a) out[p0] = sb[a];
        if (m1 < p1) out[m1] = sb[a + (m1 - p0)];
        if (m1 > m0) {
          const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(sb + a + (m0 - p0));
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + m0), "r"(saddr),
                       "r"((uint32_t)((m1 - m0) * 8))
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      buf = (buf + 1) % NB;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int CH, int NB>
float run_tma(int64_t* out, int64_t n, int run, int seg, int shift) {
  const int64_t grid = (n - shift) / run;
  const int smem = 8 * NB * (CH + 2) * 8;
  CK(cudaFuncSetAttribute(k_tma<CH, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_tma<CH, NB><<<(unsigned)grid, 256, smem>>>(out, n, run, seg, shift);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_tma<CH, NB><<<(unsigned)grid, 256, smem>>>(out, n, run, seg, shift);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  // check a prefix
  static int64_t h[4096];
  CK(cudaMemcpy(h, out + shift, sizeof(h), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 4096; ++i)
    if (h[i] != shift + i) { printf("TMA MISMATCH at %d\n", i); break; }
  return (float)((double)grid * run * 8.0 / (best * 1e-3) / 1e9);
}

template <int MODE, int W, bool CS>
float run_pat(int64_t* out, int64_t n, int run, int seg, int shift) {
  const int64_t grid = (n - shift) / run;
  k_pat<MODE, W, CS><<<(unsigned)grid, 256>>>(out, n, run, seg, shift);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_pat<MODE, W, CS><<<(unsigned)grid, 256>>>(out, n, run, seg, shift);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return (float)((double)grid * run * 8.0 / (best * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
  const int64_t n = 1ll << 31;   // 16 GB of int64
  int64_t* out;
  CK(cudaMalloc(&out, n * 8 + 4096));
  const bool sweep = argc > 1;
  printf("GB/s (best of 5), 16 GB of int64 stores\n");
  if (!sweep) {
  printf("blk 32KB  W4 cs aligned      %7.1f\n", run_pat<0, 4, true>(out, n, 4096, 0, 0));
  printf("blk 32KB  W2 cs aligned      %7.1f\n", run_pat<0, 2, true>(out, n, 4096, 0, 0));
  printf("blk 32KB  W2 cs shift 1      %7.1f\n", run_pat<0, 2, true>(out, n, 4096, 0, 1));
  printf("seg 512 (4KB) W2 cs aligned, CTA 32KB   %7.1f\n", run_pat<1, 2, true>(out, n, 4096, 512, 0));
  printf("seg 525 W2 cs misaligned, CTA 33.6KB    %7.1f\n", run_pat<1, 2, true>(out, n, 4200, 525, 0));
  printf("seg 525 W2 cs, CTA 1MB (256 segs)       %7.1f\n", run_pat<1, 2, true>(out, n, 525 * 256, 525, 0));
  printf("seg 1024 W2 cs, CTA 1MB (128 segs)      %7.1f\n", run_pat<1, 2, true>(out, n, 1024 * 128, 1024, 0));
  }
  // window sweep: misaligned 525-element segments, CTA runs of 8 .. 512 segments
  for (int segs : {8, 16, 32, 64, 128, 256, 512})
    printf("seg 525 W2 cs, CTA %4d segs (%6.0f KB)  %7.1f\n", segs, segs * 525 * 8 / 1024.0,
           run_pat<1, 2, true>(out, n, 525 * segs, 525, 0));
  for (int segs : {8, 64, 256})
    printf("seg 512 W2 cs aligned, CTA %4d segs     %7.1f\n", segs, run_pat<1, 2, true>(out, n, 512 * segs, 512, 0));
  CK(cudaMemset(out, 0, n * 8));
  // TMA op size x buffers, misaligned 525 segments in 1 MB CTAs
  printf("tma piece 128 x1 (1 KB ops)             %7.1f\n", run_tma<128, 1>(out, n, 525 * 256, 525, 0));
  printf("tma piece 128 x2                        %7.1f\n", run_tma<128, 2>(out, n, 525 * 256, 525, 0));
  printf("tma piece 256 x1 (2 KB ops)             %7.1f\n", run_tma<256, 1>(out, n, 525 * 256, 525, 0));
  printf("tma piece 256 x2                        %7.1f\n", run_tma<256, 2>(out, n, 525 * 256, 525, 0));
  printf("tma piece 512 x1 (4 KB ops)             %7.1f\n", run_tma<512, 1>(out, n, 525 * 256, 525, 0));
  printf("tma piece 1024 x1 (whole segment)       %7.1f\n", run_tma<1024, 1>(out, n, 525 * 256, 525, 0));
  printf("tma piece 256 x1, CTA 33.6KB            %7.1f\n", run_tma<256, 1>(out, n, 525 * 8, 525, 0));
  printf("tma piece 1024 x1, CTA 33.6KB           %7.1f\n", run_tma<1024, 1>(out, n, 525 * 8, 525, 0));
  return 0;
}
