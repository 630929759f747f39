// amr_octree.cu — linear octree build and 2:1 balance on the device
// (octree.py:249-330 of the reference).
//
// An octant is one 64-bit key: morton(anchor) << 6 | level, the Morton code
// taken at the finest depth (x is the lowest bit of each digit, as in
// SfcOrdering("morton"), octree.py:175-198).  Sorting keys as integers is the
// curve order with ancestors first.  A complete linear octree is a sorted key
// array whose octants tile the domain, so
//   * the leaf covering a finest cell is the last key <= (cell code << 6 | 63)
//     (one binary search; the reference probes a hash set level by level,
//     octree.py:279-286);
//   * replacing a leaf by its 2^dim children in child-code order keeps the
//     array sorted: refinement (construct) and the balance ripple never sort.
// construct: per level, the octants of that level the predicate marks are
// split (amr_oct_split).  balance_2to1: every leaf probes the finest cell
// diagonally outside each of its 3^dim - 1 directions (the reference's probe,
// octree.py:305-318) and marks the covering leaf when it is more than one
// level coarser (amr_oct_balance_mark); marked leaves are split; repeat until
// nothing is marked.  Every split is forced, so the fixed point is the
// reference's unique minimal balanced refinement.
// The exclusive prefix sum between mark and split is the caller's (torch.cumsum).
#include "amr_common.cuh"

namespace {

constexpr int kLevelBits = 6;

__host__ __device__ inline uint64_t interleave(const int32_t* a, int dim, int L) {
  uint64_t code = 0;
  for (int bit = 0; bit < L; ++bit)
    for (int d = 0; d < dim; ++d) code |= (uint64_t)((a[d] >> bit) & 1) << (bit * dim + d);
  return code;
}

__host__ __device__ inline void deinterleave(uint64_t code, int dim, int L, int32_t* a) {
  for (int d = 0; d < dim; ++d) a[d] = 0;
  for (int bit = 0; bit < L; ++bit)
    for (int d = 0; d < dim; ++d) a[d] |= (int32_t)((code >> (bit * dim + d)) & 1) << bit;
}

__global__ void keys_kernel(int dim, int L, int64_t n, const int32_t* __restrict__ anchors,
                            const int32_t* __restrict__ levels, uint64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t a[3] = {0, 0, 0};
  for (int d = 0; d < dim; ++d) a[d] = anchors[i * dim + d];
  keys[i] = (interleave(a, dim, L) << kLevelBits) | (uint64_t)levels[i];
}

__global__ void octants_kernel(int dim, int L, int64_t n, const uint64_t* __restrict__ keys,
                               int32_t* __restrict__ anchors, int32_t* __restrict__ levels) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  int32_t a[3];
  deinterleave(k >> kLevelBits, dim, L, a);
  for (int d = 0; d < dim; ++d) anchors[i * dim + d] = a[d];
  levels[i] = (int32_t)(k & ((1u << kLevelBits) - 1));
}

// out[off[i] ...] = the octant itself, or its 2^dim children in child-code order
__global__ void split_kernel(int dim, int L, int64_t n, const uint64_t* __restrict__ keys,
                             const int32_t* __restrict__ mark, const int64_t* __restrict__ off,
                             uint64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  const int64_t o = off[i];
  if (!mark[i]) {
    out[o] = k;
    return;
  }
  const int lvl = (int)(k & ((1u << kLevelBits) - 1));
  const uint64_t code = k >> kLevelBits;
  const int shift = dim * (L - lvl - 1);  // the child digit's position in the code
  for (int c = 0; c < (1 << dim); ++c)
    out[o + c] = ((code | ((uint64_t)c << shift)) << kLevelBits) | (uint64_t)(lvl + 1);
}

// one thread per (leaf, direction)
__global__ void balance_mark_kernel(int dim, int L, int64_t n, const uint64_t* __restrict__ keys,
                                    int32_t* __restrict__ mark) {
  const int ndir = (dim == 3) ? 27 : 9;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * ndir) return;
  const int64_t i = t / ndir;
  int dcode = (int)(t % ndir);
  const uint64_t k = keys[i];
  const int lvl = (int)(k & ((1u << kLevelBits) - 1));
  if (lvl < 2) return;  // nothing can be two levels coarser
  int32_t a[3];
  deinterleave(k >> kLevelBits, dim, L, a);
  const int32_t side = 1 << (L - lvl), top = 1 << L;
  int32_t cell[3] = {0, 0, 0};
  bool any = false;
  for (int d = 0; d < dim; ++d) {
    const int dv = dcode % 3 - 1;
    dcode /= 3;
    any |= dv != 0;
    const int32_t c = dv < 0 ? a[d] - 1 : (dv > 0 ? a[d] + side : a[d]);
    if (c < 0 || c >= top) return;
    cell[d] = c;
  }
  if (!any) return;
  // the leaf covering the probe cell: last key <= (cell code, deepest level)
  const uint64_t probe = (interleave(cell, dim, L) << kLevelBits) | ((1u << kLevelBits) - 1);
  int64_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (keys[mid] <= probe) lo = mid; else hi = mid - 1;
  }
  const int nl = (int)(keys[lo] & ((1u << kLevelBits) - 1));
  if (nl < lvl - 1) mark[lo] = 1;
}

int check(int dim, int L) {
  if (dim != 2 && dim != 3) {
    amr_set_error_internal("dimension must be 2 or 3");
    return AMR_EINVAL;
  }
  if (L < 0 || dim * L > 57 || L > 30) {
    amr_set_error_internal("max_depth too large for 64-bit Morton keys");
    return AMR_EINVAL;
  }
  return AMR_OK;
}

int done(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, what);
}

}  // namespace

extern "C" int amr_oct_keys(int dim, int max_depth, int64_t n, const int32_t* anchors, const int32_t* levels,
                            uint64_t* keys, void* stream) {
  if (int rc = check(dim, max_depth)) return rc;
  if (n <= 0) return AMR_OK;
  keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(dim, max_depth, n, anchors, levels, keys);
  return done("amr_oct_keys launch");
}

extern "C" int amr_oct_octants(int dim, int max_depth, int64_t n, const uint64_t* keys, int32_t* anchors,
                               int32_t* levels, void* stream) {
  if (int rc = check(dim, max_depth)) return rc;
  if (n <= 0) return AMR_OK;
  octants_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(dim, max_depth, n, keys, anchors,
                                                                                levels);
  return done("amr_oct_octants launch");
}

extern "C" int amr_oct_split(int dim, int max_depth, int64_t n, const uint64_t* keys, const int32_t* mark,
                             const int64_t* offsets, uint64_t* out, void* stream) {
  if (int rc = check(dim, max_depth)) return rc;
  if (n <= 0) return AMR_OK;
  split_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(dim, max_depth, n, keys, mark, offsets,
                                                                              out);
  return done("amr_oct_split launch");
}

extern "C" int amr_oct_balance_mark(int dim, int max_depth, int64_t n, const uint64_t* keys, int32_t* mark,
                                    void* stream) {
  if (int rc = check(dim, max_depth)) return rc;
  if (n <= 0) return AMR_OK;
  const int64_t total = n * (dim == 3 ? 27 : 9);
  balance_mark_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(dim, max_depth, n, keys, mark);
  return done("amr_oct_balance_mark launch");
}
