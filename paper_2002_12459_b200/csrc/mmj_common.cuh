// Shared helpers for the mmjoin B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define MMJ_OK 0
#define MMJ_ERR_ARG 1
#define MMJ_ERR_CUDA 2
#define MMJ_ERR_OVERFLOW 3
#define MMJ_ERR_UNSUPPORTED 4
#define MMJ_ERR_CAPACITY 5

namespace mmj {

// thread-local last error message (exposed through mmj_last_error()).
void set_error(const char* fmt, ...);
const char* last_error();

inline int cuda_status(cudaError_t e, const char* where) {
  if (e != cudaSuccess) {
    set_error("%s: %s", where, cudaGetErrorString(e));
    return MMJ_ERR_CUDA;
  }
  return MMJ_OK;
}

// every kernel launch of the library goes through MMJ_CHECK_LAUNCH, which
// also counts it (mmj_launch_count(): the bench's gpu_launches evidence).
void count_launch();
long long launch_count();

#define MMJ_CHECK_LAUNCH(where)                                   \
  do {                                                            \
    ::mmj::count_launch();                                        \
    int _st = ::mmj::cuda_status(cudaGetLastError(), where);      \
    if (_st) return _st;                                          \
  } while (0)

#define MMJ_TRY(expr)            \
  do {                           \
    int _st = (expr);            \
    if (_st) return _st;         \
  } while (0)

// Device-side bounds checks, compiled in only for the checked library
// variant (libmmjoin_b200_check.so, -DMMJ_DEBUG_CHECKS; build.py): a failed
// check prints the site and traps, so a bad index surfaces as a launch error
// instead of a silent out-of-bounds access.  The stand-in for
// compute-sanitizer, which this GPU pool does not run.
#ifdef MMJ_DEBUG_CHECKS
#define MMJ_DCHECK(cond, what)                                                                         \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("MMJ_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,          \
             (int)blockIdx.x, (int)threadIdx.x);                                                      \
      __trap();                                                                                       \
    }                                                                                                 \
  } while (0)
#else
#define MMJ_DCHECK(cond, what) \
  do {                         \
  } while (0)
#endif

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

int sm_count();

// cudaFuncAttributeMaxDynamicSharedMemorySize for `func` on the CURRENT
// device, set once per (device, function): the attribute is per device, so
// a process driving several GPUs must set it on each (scan.cu).
int set_max_dynamic_smem(const void* func, int bytes, const char* where);

// ---- exclusive scans (scan.cu) --------------------------------------------
// out[i] = sum(in[0..i)), out[n] = total.  `ws` must hold scan_ws_bytes(n).
size_t scan_ws_bytes(int64_t n);
int scan_i32_i64(const int32_t* in, int64_t* out, int64_t n, void* ws, cudaStream_t st);
int scan_u8_i32(const uint8_t* in, int32_t* out, int64_t n, void* ws, cudaStream_t st);
int scan_i64_i64(const int64_t* in, int64_t* out, int64_t n, void* ws, cudaStream_t st);
int scan_i32_i32(const int32_t* in, int32_t* out, int64_t n, void* ws, cudaStream_t st);
int code_checksum(const int64_t* codes, int64_t n, int64_t base, unsigned long long* out, cudaStream_t st);

// result text formats (format.cu): up to 4 code columns + the count column
constexpr int MMJ_FMT_COLS = 5;
struct FmtArgs {
  const int64_t* codes;           // n mixed-radix codes over dims[0 .. ncode)
  const int64_t* counts;          // n counts (the last column) or nullptr
  const int32_t* order;           // line -> tuple (nullptr = identity)
  int64_t n;
  int ncode;                      // code columns
  int64_t dims[MMJ_FMT_COLS];
  const int32_t* rank[MMJ_FMT_COLS];
  int64_t nrank[MMJ_FMT_COLS];    // table sizes (count column: max count + 1)
  const int64_t* soff[MMJ_FMT_COLS];  // string offsets into blob, nrank + 1 entries
  const uint8_t* blob[MMJ_FMT_COLS];
};

}  // namespace mmj

// ---- device helpers ----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
