// Device-wide exclusive prefix sums (reduce-then-scan, recursive on the block
// totals).  Used for every variable-size step of the path: heavy-y position
// maps, light-z CSR compaction, per-tuple expansion offsets (the witness
// balance of the light passes) and per-segment output offsets of the merge.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <stdarg.h>

#include <algorithm>
#include <mutex>
#include <tuple>
#include <vector>

#include "mmj_common.cuh"

namespace mmj {

static thread_local char g_err[1024];

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

static long long g_launches = 0;
void count_launch() { __atomic_add_fetch(&g_launches, 1, __ATOMIC_RELAXED); }
long long launch_count() { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

int sm_count() {
  int dev = 0;
  cudaGetDevice(&dev);
  static int cached[64] = {0};
  if (dev < 64 && cached[dev]) return cached[dev];
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cached[dev] = n;
  return n;
}

int set_max_dynamic_smem(const void* func, int bytes, const char* where) {
  static std::mutex mu;
  static std::vector<std::tuple<int, const void*, int>> done;   // (device, function, bytes)
  int dev = 0;
  MMJ_TRY(cuda_status(cudaGetDevice(&dev), where));
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (std::get<0>(d) == dev && std::get<1>(d) == func && std::get<2>(d) >= bytes) return MMJ_OK;
  MMJ_TRY(cuda_status(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), where));
  done.emplace_back(dev, func, bytes);
  return MMJ_OK;
}

namespace {

constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;   // 4096 items per block

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(SCAN_THREADS) tile_reduce(const TIn* __restrict__ in, int64_t n,
                                                            TOut* __restrict__ partial) {
  using BR = cub::BlockReduce<TOut, SCAN_THREADS>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  TOut acc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t j = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
    if (j < n) acc += (TOut)in[j];
  }
  TOut tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <typename TIn, typename TOut>
__global__ void __launch_bounds__(SCAN_THREADS) tile_scan(const TIn* __restrict__ in, int64_t n,
                                                          const TOut* __restrict__ offsets,
                                                          TOut* __restrict__ out, bool write_total) {
  using BS = cub::BlockScan<TOut, SCAN_THREADS>;
  __shared__ typename BS::TempStorage tmp;
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  TOut v[SCAN_ITEMS];
  // blocked arrangement: thread t owns items [t*ITEMS, t*ITEMS+ITEMS)
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    v[i] = j < n ? (TOut)in[j] : (TOut)0;
  }
  TOut agg;
  BS(tmp).ExclusiveSum(v, v, agg);
  const TOut off = offsets ? offsets[blockIdx.x] : (TOut)0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    int64_t j = base + (int64_t)threadIdx.x * SCAN_ITEMS + i;
    if (j < n) out[j] = v[i] + off;
  }
  if (write_total && threadIdx.x == 0 && base + SCAN_TILE >= n) out[n] = off + agg;
}

inline int64_t nblocks(int64_t n) { return ceil_div(n, SCAN_TILE); }

// workspace: for each recursion level, partial sums (nb) + their scan (nb+1)
size_t ws_levels(int64_t n, size_t elem) {
  size_t total = 0;
  while (n > SCAN_TILE) {
    int64_t nb = nblocks(n);
    total += (size_t)(2 * nb + 1) * elem + 256;
    n = nb;
  }
  return total + 256;
}

template <typename TIn, typename TOut>
int scan_impl(const TIn* in, TOut* out, int64_t n, void* ws, cudaStream_t st) {
  if (n < 0) {
    set_error("scan: negative length");
    return MMJ_ERR_ARG;
  }
  if (n == 0) {
    return cuda_status(cudaMemsetAsync(out, 0, sizeof(TOut), st), "scan memset");
  }
  if (n <= SCAN_TILE) {
    tile_scan<TIn, TOut><<<1, SCAN_THREADS, 0, st>>>(in, n, nullptr, out, true);
    MMJ_CHECK_LAUNCH("tile_scan");
    return MMJ_OK;
  }
  const int64_t nb = nblocks(n);
  TOut* partial = reinterpret_cast<TOut*>(ws);
  TOut* pscan = partial + nb;
  uint8_t* next_ws = reinterpret_cast<uint8_t*>(pscan + nb + 1);
  next_ws = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(next_ws) + 255) & ~uintptr_t(255));
  tile_reduce<TIn, TOut><<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, n, partial);
  MMJ_CHECK_LAUNCH("tile_reduce");
  MMJ_TRY((scan_impl<TOut, TOut>(partial, pscan, nb, next_ws, st)));
  tile_scan<TIn, TOut><<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, n, pscan, out, true);
  MMJ_CHECK_LAUNCH("tile_scan");
  return MMJ_OK;
}

}  // namespace

size_t scan_ws_bytes(int64_t n) { return ws_levels(n, 8) + 256; }

int scan_i32_i64(const int32_t* in, int64_t* out, int64_t n, void* ws, cudaStream_t st) {
  return scan_impl<int32_t, int64_t>(in, out, n, ws, st);
}
int scan_u8_i32(const uint8_t* in, int32_t* out, int64_t n, void* ws, cudaStream_t st) {
  return scan_impl<uint8_t, int32_t>(in, out, n, ws, st);
}
int scan_i32_i32(const int32_t* in, int32_t* out, int64_t n, void* ws, cudaStream_t st) {
  return scan_impl<int32_t, int32_t>(in, out, n, ws, st);
}
int scan_i64_i64(const int64_t* in, int64_t* out, int64_t n, void* ws, cudaStream_t st) {
  return scan_impl<int64_t, int64_t>(in, out, n, ws, st);
}

// ---- order-sensitive checksum of a sorted code run ---------------------------
// out[0] += sum(codes[i]), out[1] += sum((base + i + 1) * codes[i]), both
// mod 2^64: equal for two code arrays of one length only if (with
// overwhelming probability) they are equal element by element, and additive
// over consecutive chunks when `base` is the number of codes before the chunk.
namespace {
__global__ void k_code_checksum(const int64_t* __restrict__ codes, int64_t n, unsigned long long base,
                                unsigned long long* __restrict__ out) {
  unsigned long long s = 0, w = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + stride < n; i += 2 * stride) {   // two streaming loads in flight per thread
    const unsigned long long c0 = (unsigned long long)__ldcs(codes + i);
    const unsigned long long c1 = (unsigned long long)__ldcs(codes + i + stride);
    s += c0 + c1;
    w += (base + (unsigned long long)i + 1ull) * c0 + (base + (unsigned long long)(i + stride) + 1ull) * c1;
  }
  if (i < n) {
    const unsigned long long c = (unsigned long long)__ldcs(codes + i);
    s += c;
    w += (base + (unsigned long long)i + 1ull) * c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    w += __shfl_xor_sync(0xffffffffu, w, o);
  }
  if ((threadIdx.x & 31) == 0 && (s | w)) {
    atomicAdd(out, s);
    atomicAdd(out + 1, w);
  }
}
}  // namespace

int code_checksum(const int64_t* codes, int64_t n, int64_t base, unsigned long long* out, cudaStream_t st) {
  if (n < 0 || base < 0) {
    set_error("code_checksum: negative length / base");
    return MMJ_ERR_ARG;
  }
  if (n == 0) return MMJ_OK;
  const int64_t g = std::min<int64_t>(ceil_div(n, 512), (int64_t)sm_count() * 8);
  k_code_checksum<<<(unsigned)g, 256, 0, st>>>(codes, n, (unsigned long long)base, out);
  MMJ_CHECK_LAUNCH("k_code_checksum");
  return MMJ_OK;
}

}  // namespace mmj
