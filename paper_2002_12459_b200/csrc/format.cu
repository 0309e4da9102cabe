// Result text formats of the reference CLI (cli.py:129-136, 154-161,
// 180-182, 205-206): one line per output tuple, "v0 v1 [... ] [count]",
// raw dictionary values separated by single spaces, lines sorted as Python
// sorts the strings, joined by "\n".
//
// Python's string order of such lines equals the lexicographic order of the
// tuple of its fields' strings whenever no field contains a character below
// ' ' (0x20): where one field is a proper prefix of another the shorter
// line continues with ' ' (or ends) while the longer continues with a
// character > ' '.  Dictionary values come from whitespace-split tokens
// (relation.py:100-111) or str() of numbers, so the order of a line is the
// order of (rank(v0), rank(v1), ..., rank(count)) with rank = position of
// the field's string among its column's sorted distinct strings (UTF-8
// byte order = code point order).  So the device builds one int64 key per
// tuple in that mixed radix, sorts the keys (the ingest radix sort), and
// writes the bytes: per-tuple line lengths, an exclusive scan, then each
// line copied from the columns' string blobs.
#include "mmj_common.cuh"

namespace mmj {

namespace {

constexpr int TPB = 256;

inline int grid_for(int64_t n) {
  int64_t g = ceil_div(n, TPB);
  const int64_t cap = (int64_t)sm_count() * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// column values of tuple t: codes decoded right to left (joinproject.py:58-63)
__device__ __forceinline__ int columns(const FmtArgs& f, int64_t t, int64_t* v) {
  int64_t rem = f.codes[t];
  for (int c = f.ncode - 1; c >= 0; --c) {
    v[c] = rem % f.dims[c];
    rem /= f.dims[c];
  }
  int nc = f.ncode;
  if (f.counts) v[nc++] = f.counts[t];
  return nc;
}

__global__ void k_fmt_keys(const FmtArgs f, int64_t* __restrict__ key, int* __restrict__ bad) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < f.n; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t v[MMJ_FMT_COLS];
    const int nc = columns(f, t, v);
    int64_t k = 0;
    for (int c = 0; c < nc; ++c) {
      if (v[c] < 0 || v[c] >= f.nrank[c]) {
        atomicExch(bad, 1);
        break;
      }
      k = k * f.nrank[c] + f.rank[c][v[c]];
    }
    key[t] = k;
  }
}

__global__ void k_fmt_lengths(const FmtArgs f, int32_t* __restrict__ len) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < f.n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = f.order ? f.order[p] : p;
    int64_t v[MMJ_FMT_COLS];
    const int nc = columns(f, t, v);
    int64_t l = nc - 1 + (p + 1 < f.n ? 1 : 0);   // separators + newline (none after the last line)
    for (int c = 0; c < nc; ++c) l += f.soff[c][v[c] + 1] - f.soff[c][v[c]];
    len[p] = (int32_t)l;
  }
}

__global__ void k_fmt_write(const FmtArgs f, const int64_t* __restrict__ line_off, uint8_t* __restrict__ out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < f.n; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = f.order ? f.order[p] : p;
    int64_t v[MMJ_FMT_COLS];
    const int nc = columns(f, t, v);
    uint8_t* o = out + line_off[p];
    for (int c = 0; c < nc; ++c) {
      if (c) *o++ = ' ';
      const int64_t b = f.soff[c][v[c]], e = f.soff[c][v[c] + 1];
      for (int64_t i = b; i < e; ++i) *o++ = f.blob[c][i];
    }
    if (p + 1 < f.n) *o = '\n';
  }
}

}  // namespace

int fmt_keys(const FmtArgs& f, int64_t* key, int* bad, cudaStream_t st) {
  if (f.n == 0) return MMJ_OK;
  MMJ_TRY(cuda_status(cudaMemsetAsync(bad, 0, sizeof(int), st), "memset fmt flag"));
  k_fmt_keys<<<grid_for(f.n), TPB, 0, st>>>(f, key, bad);
  MMJ_CHECK_LAUNCH("k_fmt_keys");
  return MMJ_OK;
}

int fmt_lengths(const FmtArgs& f, int32_t* len, cudaStream_t st) {
  if (f.n == 0) return MMJ_OK;
  k_fmt_lengths<<<grid_for(f.n), TPB, 0, st>>>(f, len);
  MMJ_CHECK_LAUNCH("k_fmt_lengths");
  return MMJ_OK;
}

int fmt_write(const FmtArgs& f, const int64_t* line_off, uint8_t* out, cudaStream_t st) {
  if (f.n == 0) return MMJ_OK;
  k_fmt_write<<<grid_for(f.n), TPB, 0, st>>>(f, line_off, out);
  MMJ_CHECK_LAUNCH("k_fmt_write");
  return MMJ_OK;
}

}  // namespace mmj
