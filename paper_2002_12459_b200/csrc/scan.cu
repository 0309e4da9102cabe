// Device-wide exclusive prefix sums (reduce-then-scan, recursive on the block
// totals).  Used for every variable-size step of the path: heavy-y position
// maps, light-z CSR compaction, per-tuple expansion offsets (the witness
// balance of the light passes) and per-segment output offsets of the merge.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <stdarg.h>

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

}  // namespace mmj
