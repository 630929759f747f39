// amr_devmesh.cu — node registry, leaf-tile unzip tables and interpolation rows
// on the device (mesh.py:214-398 of the reference; the host statement of the
// same passes is amr_mesh_build in amr_mesh.cpp, and the two are compared bit
// for bit in tests/test_devmesh_gpu.py).
//
// Input: the balanced tree as sorted keys (amr_octree.cu) with its anchors and
// levels.  Lattice points are in units of a finest cell / (ppo-1) (mesh.py:8-11).
//   pass 1  ownership: every leaf lattice point is owned (first leaf of the
//           curve that holds it as a real node), shared, or hanging (off the
//           lattice of a coarser leaf that touches it) (mesh.py:214-245);
//   pass 2  gids: first-claim order = leaf start + rank among the leaf's owned
//           points; shared points take their owner's gid (mesh.py:246-277);
//   pass 3  tile table over the stencil cross: gid, -1 outside the domain, or a
//           hanging point (its lattice code goes to a compact list);
//   pass 4  after the caller's sort/unique of the codes: the interpolation row
//           of each hanging point — tensor-product 4-point Lagrange weights in
//           the coarsest touching leaf, taps resolved recursively while they
//           hang, merged in insertion order, sorted by gid (mesh.py:316-351,
//           391-393) — as a count pass and a fill pass.
// -fmad=false (build.py): the weights are the reference's bits.
#include "amr_common.cuh"

namespace {

constexpr int kLevelBits = 6;
constexpr int kRowCap = 128;   // taps per row (the tile encoding holds 124)
constexpr int kMaxDepth = 6;   // nesting of hanging taps

struct DM {
  int dim, L, ppo, pad, scale, P, E;
  int64_t n, top_nodes;
  const uint64_t* keys;    // sorted
  const int32_t* anchor;   // [n][dim]
  const int32_t* level;    // [n]
};

__device__ __forceinline__ uint64_t interleave(const int32_t* a, int dim, int L) {
  uint64_t code = 0;
  for (int bit = 0; bit < L; ++bit)
    for (int d = 0; d < dim; ++d) code |= (uint64_t)((a[d] >> bit) & 1) << (bit * dim + d);
  return code;
}

__device__ __forceinline__ int32_t find_leaf(const DM& m, const int32_t* cell) {
  const uint64_t probe = (interleave(cell, m.dim, m.L) << kLevelBits) | ((1u << kLevelBits) - 1);
  int64_t lo = 0, hi = m.n - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (m.keys[mid] <= probe) lo = mid; else hi = mid - 1;
  }
  return (int32_t)lo;
}

__device__ __forceinline__ int64_t spacing(const DM& m, int lvl) { return (int64_t)1 << (m.L - lvl); }

// leaves whose closed box holds lattice point p, ascending (mesh.py:293-314)
__device__ int containing(const DM& m, const int64_t* p, int32_t* out) {
  int n = 0;
  for (int sig = 0; sig < (1 << m.dim); ++sig) {
    int32_t cell[3] = {0, 0, 0};
    bool ok = true;
    for (int d = 0; d < m.dim; ++d) {
      const int64_t q = ((sig >> d) & 1) ? p[d] : p[d] - 1;
      if (q < 0 || q >= m.top_nodes) {
        ok = false;
        break;
      }
      cell[d] = (int32_t)(q / m.scale);
    }
    if (!ok) continue;
    const int32_t j = find_leaf(m, cell);
    bool dup = false;
    for (int k = 0; k < n; ++k) dup |= (out[k] == j);
    if (!dup) out[n++] = j;
  }
  for (int a = 1; a < n; ++a) {  // ascending
    const int32_t v = out[a];
    int b = a - 1;
    while (b >= 0 && out[b] > v) {
      out[b + 1] = out[b];
      --b;
    }
    out[b + 1] = v;
  }
  return n;
}

__device__ __forceinline__ bool on_lattice(const DM& m, int32_t leaf, const int64_t* p) {
  const int64_t s = spacing(m, m.level[leaf]);
  for (int d = 0; d < m.dim; ++d)
    if ((p[d] - (int64_t)m.anchor[(int64_t)leaf * m.dim + d] * m.scale) % s != 0) return false;
  return true;
}

__device__ __forceinline__ int local_index(const DM& m, int32_t leaf, const int64_t* p) {
  const int64_t s = spacing(m, m.level[leaf]);
  int idx = 0;
  for (int d = 0; d < m.dim; ++d)
    idx = idx * m.ppo + (int)((p[d] - (int64_t)m.anchor[(int64_t)leaf * m.dim + d] * m.scale) / s);
  return idx;
}

// owner leaf of a real node, -1 if p hangs, -2 if no leaf holds it
__device__ int32_t real_owner(const DM& m, const int64_t* p) {
  int32_t c[8];
  const int n = containing(m, p, c);
  if (n == 0) return -2;
  for (int k = 0; k < n; ++k)
    if (!on_lattice(m, c[k], p)) return -1;
  return c[0];
}

__device__ __forceinline__ int32_t gid_of(const DM& m, const int32_t* leaf_gids, const int64_t* p) {
  const int32_t o = real_owner(m, p);
  if (o < 0) return -1;
  return leaf_gids[(int64_t)o * m.P + local_index(m, o, p)];
}

__device__ __forceinline__ int64_t encode(const DM& m, const int64_t* p) {
  int64_t c = p[0];
  for (int d = 1; d < m.dim; ++d) c = c * (m.top_nodes + 1) + p[d];
  return c;
}

__device__ __forceinline__ void decode_point(const DM& m, int64_t code, int64_t* p) {
  for (int d = m.dim - 1; d >= 0; --d) {
    p[d] = code % (m.top_nodes + 1);
    code /= (m.top_nodes + 1);
  }
}

__device__ __forceinline__ void leaf_point(const DM& m, int64_t leaf, int k, int64_t* p, bool* interior) {
  const int64_t s = spacing(m, m.level[leaf]);
  bool in = true;
  int r = k;
  for (int d = m.dim - 1; d >= 0; --d) {
    const int loc = r % m.ppo;
    r /= m.ppo;
    in &= (loc > 0 && loc < m.ppo - 1);
    p[d] = (int64_t)m.anchor[leaf * m.dim + d] * m.scale + s * loc;
  }
  *interior = in;
}

// ---- pass 1: one CTA per leaf; status 1 owned, 0 shared, -1 hanging; owner leaf of shared points
__global__ void ownership_kernel(DM m, int8_t* __restrict__ status, int32_t* __restrict__ owner,
                                 int64_t* __restrict__ counts, int* __restrict__ err) {
  const int64_t leaf = blockIdx.x;
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int mine = 0;
  for (int k = threadIdx.x; k < m.P; k += blockDim.x) {
    int64_t p[3] = {0, 0, 0};
    bool interior;
    leaf_point(m, leaf, k, p, &interior);
    int8_t st = 1;
    int32_t ow = (int32_t)leaf;
    if (!interior) {
      int32_t c[8];
      const int n = containing(m, p, c);
      if (n == 0) {
        atomicOr(err, 1);
        st = -1;
      } else {
        bool real = true;
        for (int q = 0; q < n; ++q) real &= on_lattice(m, c[q], p);
        st = !real ? -1 : (c[0] == leaf ? 1 : 0);
        ow = real ? c[0] : -1;
      }
    }
    status[leaf * m.P + k] = st;
    owner[leaf * m.P + k] = ow;
    mine += (st == 1);
  }
  atomicAdd(&s_cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0) counts[leaf] = s_cnt;
}

// ---- pass 2a: owned gids = start + rank in the leaf's C-order enumeration (one warp per leaf)
__global__ void owned_gids_kernel(DM m, const int8_t* __restrict__ status, const int64_t* __restrict__ starts,
                                  int32_t* __restrict__ leaf_gids) {
  const int64_t leaf = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (leaf >= m.n) return;
  const int lane = threadIdx.x & 31;
  int base = (int)starts[leaf];
  for (int k0 = 0; k0 < m.P; k0 += 32) {
    const int k = k0 + lane;
    const bool own = k < m.P && status[leaf * m.P + k] == 1;
    const unsigned ball = __ballot_sync(0xffffffffu, own);
    if (k < m.P) leaf_gids[leaf * m.P + k] = own ? base + __popc(ball & ((1u << lane) - 1)) : -1;
    base += __popc(ball);
  }
}

// ---- pass 2b: shared points take their owner's gid
__global__ void shared_gids_kernel(DM m, const int8_t* __restrict__ status, const int32_t* __restrict__ owner,
                                   int32_t* __restrict__ leaf_gids) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m.n * m.P) return;
  if (status[t] != 0) return;
  const int64_t leaf = t / m.P;
  int64_t p[3] = {0, 0, 0};
  bool interior;
  leaf_point(m, leaf, (int)(t % m.P), p, &interior);
  const int32_t o = owner[t];
  leaf_gids[t] = leaf_gids[(int64_t)o * m.P + local_index(m, o, p)];  // an owned entry (pass 2a)
}

// cross enumeration shared with the kernels and tileprog.cross_cells: the
// ppo^dim interior in C order, then per axis the 2*pad layers below and above
__device__ __forceinline__ void cross_entry_local(const DM& m, int e, int* loc) {
  int NF = 1;
  for (int d = 1; d < m.dim; ++d) NF *= m.ppo;
  if (e < m.P) {
    int r = e;
    for (int d = m.dim - 1; d >= 0; --d) {
      loc[d] = m.pad + r % m.ppo;
      r /= m.ppo;
    }
    return;
  }
  int r = e - m.P;
  const int axis = r / (2 * m.pad * NF);
  r %= 2 * m.pad * NF;
  const int layer = r / NF;
  int within = r % NF;
  for (int d = m.dim - 1; d >= 0; --d) {
    if (d == axis) continue;
    loc[d] = m.pad + within % m.ppo;
    within /= m.ppo;
  }
  loc[axis] = layer < m.pad ? layer : m.ppo + layer;
}

__device__ __forceinline__ bool cross_point(const DM& m, int64_t leaf, int e, int64_t* p, int* idx_in_leaf) {
  int lp[3] = {0, 0, 0};
  cross_entry_local(m, e, lp);
  const int64_t s = spacing(m, m.level[leaf]);
  bool in_dom = true, in_leaf = true;
  int idx = 0;
  for (int d = 0; d < m.dim; ++d) {
    const int loc = lp[d] - m.pad;
    p[d] = (int64_t)m.anchor[leaf * m.dim + d] * m.scale + s * loc;
    in_dom &= (p[d] >= 0 && p[d] <= m.top_nodes);
    in_leaf &= (loc >= 0 && loc < m.ppo);
    idx = idx * m.ppo + loc;
  }
  *idx_in_leaf = in_leaf ? idx : -1;
  return in_dom;
}

// ---- pass 3: table entries; hanging entries get -2 and are counted per leaf
__global__ void table_kernel(DM m, const int32_t* __restrict__ leaf_gids, int32_t* __restrict__ table,
                             int32_t* __restrict__ n_hang) {
  const int64_t leaf = blockIdx.x;
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  int mine = 0;
  for (int e = threadIdx.x; e < m.E; e += blockDim.x) {
    int64_t p[3] = {0, 0, 0};
    int idx;
    int32_t ent;
    if (!cross_point(m, leaf, e, p, &idx)) {
      ent = -1;
    } else {
      ent = idx >= 0 ? leaf_gids[leaf * m.P + idx] : gid_of(m, leaf_gids, p);
      if (ent < 0) {
        ent = -2;
        ++mine;
      }
    }
    table[leaf * m.E + e] = ent;
  }
  atomicAdd(&s_cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0) n_hang[leaf] = s_cnt;
}

// ---- pass 3b: compact list of the hanging entries (table position, lattice code); one warp per leaf
__global__ void hang_list_kernel(DM m, const int32_t* __restrict__ table, const int64_t* __restrict__ hang_off,
                                 int64_t* __restrict__ pos_out, int64_t* __restrict__ code_out) {
  const int64_t leaf = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (leaf >= m.n) return;
  const int lane = threadIdx.x & 31;
  int64_t base = hang_off[leaf];
  for (int e0 = 0; e0 < m.E; e0 += 32) {
    const int e = e0 + lane;
    const bool h = e < m.E && table[leaf * m.E + e] == -2;
    const unsigned ball = __ballot_sync(0xffffffffu, h);
    if (h) {
      int64_t p[3] = {0, 0, 0};
      int idx;
      cross_point(m, leaf, e, p, &idx);
      const int64_t o = base + __popc(ball & ((1u << lane) - 1));
      pos_out[o] = leaf * m.E + e;
      code_out[o] = encode(m, p);
    }
    base += __popc(ball);
  }
}

// ---- pass 3c: table[pos] = -2 - (row of its code among the sorted unique codes)
__global__ void table_rows_kernel(int64_t n_hang, const int64_t* __restrict__ pos, const int64_t* __restrict__ code,
                                  int64_t n_rows, const int64_t* __restrict__ rows, int32_t* __restrict__ table) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_hang) return;
  const int64_t c = code[t];
  int64_t lo = 0, hi = n_rows - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (rows[mid] < c) lo = mid + 1; else hi = mid;
  }
  table[pos[t]] = -2 - (int32_t)lo;
}

// ---- pass 4: interpolation rows
struct Row {
  int n;
  int32_t g[kRowCap];
  double w[kRowCap];
};

// _lagrange_weights (mesh.py:138-150)
__device__ void lagrange(double xi, int n, int* w0_out, double* ws, int* npts_out) {
  const int npts = n < 4 ? n : 4;
  int w0 = (int)floor(xi) - 1;
  w0 = w0 < 0 ? 0 : (w0 > n - npts ? n - npts : w0);
  double xs[4];
  for (int a = 0; a < npts; ++a) xs[a] = (double)(w0 + a);
  for (int a = 0; a < npts; ++a) {
    ws[a] = 1.0;
    for (int b = 0; b < npts; ++b)
      if (a != b) ws[a] *= (xi - xs[b]) / (xs[a] - xs[b]);
  }
  *w0_out = w0;
  *npts_out = npts;
}

// _point_weights (mesh.py:316-351): insertion-ordered sparse row; err bits: 1 outside the
// domain, 2 row longer than kRowCap, 4 hanging taps nested deeper than kMaxDepth
template <int DEPTH>
__device__ void point_weights(const DM& m, const int32_t* leaf_gids, const int64_t* p, Row& acc, int* err) {
  acc.n = 0;
  int32_t c[8];
  const int n = containing(m, p, c);
  if (n == 0) {
    *err |= 1;
    return;
  }
  bool real = true;
  for (int k = 0; k < n; ++k) real &= on_lattice(m, c[k], p);
  if (real) {
    acc.n = 1;
    acc.g[0] = leaf_gids[(int64_t)c[0] * m.P + local_index(m, c[0], p)];
    acc.w[0] = 1.0;
    return;
  }
  if constexpr (DEPTH >= kMaxDepth) {
    *err |= 4;
    return;
  } else {
    int lvl = 1 << 30;
    for (int k = 0; k < n; ++k) lvl = min(lvl, m.level[c[k]]);
    int32_t leaf = -1;
    for (int k = 0; k < n; ++k)
      if (m.level[c[k]] == lvl) {
        leaf = c[k];
        break;
      }
    const int64_t s = spacing(m, lvl);
    int64_t org[3] = {0, 0, 0};
    int w0[3] = {0, 0, 0}, np[3] = {1, 1, 1};
    double ws[3][4];
    for (int d = 0; d < m.dim; ++d) {
      org[d] = (int64_t)m.anchor[(int64_t)leaf * m.dim + d] * m.scale;
      const double xi = (double)(p[d] - org[d]) / (double)s;
      lagrange(xi, m.ppo, &w0[d], ws[d], &np[d]);
    }
    int total = 1;
    for (int d = 0; d < m.dim; ++d) total *= np[d];
    Row sub;
    for (int combo = 0; combo < total; ++combo) {
      int cidx[3] = {0, 0, 0};
      int rem = combo;
      for (int d = m.dim - 1; d >= 0; --d) {
        cidx[d] = rem % np[d];
        rem /= np[d];
      }
      double w = 1.0;
      int64_t q[3] = {0, 0, 0};
      for (int d = 0; d < m.dim; ++d) {
        w *= ws[d][cidx[d]];
        q[d] = org[d] + (int64_t)(w0[d] + cidx[d]) * s;
      }
      if (w == 0.0) continue;
      point_weights<DEPTH + 1>(m, leaf_gids, q, sub, err);
      if (*err) return;
      for (int j = 0; j < sub.n; ++j) {
        bool found = false;
        for (int a = 0; a < acc.n; ++a)
          if (acc.g[a] == sub.g[j]) {
            acc.w[a] = acc.w[a] + w * sub.w[j];
            found = true;
            break;
          }
        if (!found) {
          if (acc.n >= kRowCap) {
            *err |= 2;
            return;
          }
          acc.g[acc.n] = sub.g[j];
          acc.w[acc.n] = 0.0 + w * sub.w[j];
          ++acc.n;
        }
      }
    }
  }
}

// count pass (row_ptr == NULL) or fill pass: one thread per hanging point
__global__ void rows_kernel(DM m, const int32_t* __restrict__ leaf_gids, int64_t n_rows,
                            const int64_t* __restrict__ codes, const int64_t* __restrict__ row_ptr,
                            int32_t* __restrict__ counts, int32_t* __restrict__ gid_out, double* __restrict__ w_out,
                            int* __restrict__ err) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  int64_t p[3] = {0, 0, 0};
  decode_point(m, codes[r], p);
  Row row;
  int e = 0;
  point_weights<0>(m, leaf_gids, p, row, &e);
  if (e) {
    atomicOr(err, e);
    return;
  }
  if (row_ptr == nullptr) {
    counts[r] = row.n;
    return;
  }
  // ascending gid (mesh.py:391-393); gids of a row are distinct
  for (int a = 1; a < row.n; ++a) {
    const int32_t g = row.g[a];
    const double w = row.w[a];
    int b = a - 1;
    while (b >= 0 && row.g[b] > g) {
      row.g[b + 1] = row.g[b];
      row.w[b + 1] = row.w[b];
      --b;
    }
    row.g[b + 1] = g;
    row.w[b + 1] = w;
  }
  const int64_t o = row_ptr[r];
  for (int a = 0; a < row.n; ++a) {
    gid_out[o + a] = row.g[a];
    w_out[o + a] = row.w[a];
  }
}

int make(DM& m, int dim, int L, int ppo, int pad, int64_t n, const uint64_t* keys, const int32_t* anchor,
         const int32_t* level) {
  if (dim != 2 && dim != 3) {
    amr_set_error_internal("dimension must be 2 or 3");
    return AMR_EINVAL;
  }
  if (ppo < 5 || ppo % 2 == 0 || pad != 2 || dim * L > 57) {
    amr_set_error_internal("device mesh: ppo must be odd >= 5, pad 2, dim * max_depth <= 57");
    return AMR_EINVAL;
  }
  m.dim = dim;
  m.L = L;
  m.ppo = ppo;
  m.pad = pad;
  m.scale = ppo - 1;
  m.P = 1;
  for (int d = 0; d < dim; ++d) m.P *= ppo;
  m.E = m.P + 2 * dim * pad * (m.P / ppo);
  m.n = n;
  m.top_nodes = (int64_t)m.scale << L;
  m.keys = keys;
  m.anchor = anchor;
  m.level = level;
  return AMR_OK;
}

int finish(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, what);
}

}  // namespace

extern "C" int amr_dm_ownership(int dim, int L, int ppo, int pad, int64_t n, const uint64_t* keys,
                                const int32_t* anchors, const int32_t* levels, int8_t* status, int32_t* owner,
                                int64_t* counts, int* err, void* stream) {
  DM m;
  if (int rc = make(m, dim, L, ppo, pad, n, keys, anchors, levels)) return rc;
  if (n <= 0) return AMR_OK;
  ownership_kernel<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(m, status, owner, counts, err);
  return finish("amr_dm_ownership launch");
}

extern "C" int amr_dm_gids(int dim, int L, int ppo, int pad, int64_t n, const uint64_t* keys, const int32_t* anchors,
                           const int32_t* levels, const int8_t* status, const int32_t* owner, const int64_t* starts,
                           int32_t* leaf_gids, void* stream) {
  DM m;
  if (int rc = make(m, dim, L, ppo, pad, n, keys, anchors, levels)) return rc;
  if (n <= 0) return AMR_OK;
  cudaStream_t st = (cudaStream_t)stream;
  owned_gids_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(m, status, starts, leaf_gids);
  const int64_t total = n * m.P;
  shared_gids_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(m, status, owner, leaf_gids);
  return finish("amr_dm_gids launch");
}

extern "C" int amr_dm_table(int dim, int L, int ppo, int pad, int64_t n, const uint64_t* keys, const int32_t* anchors,
                            const int32_t* levels, const int32_t* leaf_gids, int32_t* table, int32_t* n_hang,
                            void* stream) {
  DM m;
  if (int rc = make(m, dim, L, ppo, pad, n, keys, anchors, levels)) return rc;
  if (n <= 0) return AMR_OK;
  table_kernel<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(m, leaf_gids, table, n_hang);
  return finish("amr_dm_table launch");
}

extern "C" int amr_dm_hang_list(int dim, int L, int ppo, int pad, int64_t n, const uint64_t* keys,
                                const int32_t* anchors, const int32_t* levels, const int32_t* table,
                                const int64_t* hang_off, int64_t* pos, int64_t* code, void* stream) {
  DM m;
  if (int rc = make(m, dim, L, ppo, pad, n, keys, anchors, levels)) return rc;
  if (n <= 0) return AMR_OK;
  hang_list_kernel<<<(unsigned)((n + 7) / 8), 256, 0, (cudaStream_t)stream>>>(m, table, hang_off, pos, code);
  return finish("amr_dm_hang_list launch");
}

extern "C" int amr_dm_table_rows(int64_t n_hang, const int64_t* pos, const int64_t* code, int64_t n_rows,
                                 const int64_t* rows, int32_t* table, void* stream) {
  if (n_hang <= 0) return AMR_OK;
  table_rows_kernel<<<(unsigned)((n_hang + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n_hang, pos, code, n_rows,
                                                                                       rows, table);
  return finish("amr_dm_table_rows launch");
}

extern "C" int amr_dm_rows(int dim, int L, int ppo, int pad, int64_t n, const uint64_t* keys, const int32_t* anchors,
                           const int32_t* levels, const int32_t* leaf_gids, int64_t n_rows, const int64_t* codes,
                           const int64_t* row_ptr, int32_t* counts, int32_t* gid_out, double* w_out, int* err,
                           void* stream) {
  DM m;
  if (int rc = make(m, dim, L, ppo, pad, n, keys, anchors, levels)) return rc;
  if (n_rows <= 0) return AMR_OK;
  static bool stack_set = false;
  if (!stack_set) {  // Row buffers of the nested calls live on the thread stack
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitStackSize);
    if (cur < 24 * 1024) cudaDeviceSetLimit(cudaLimitStackSize, 24 * 1024);
    stack_set = true;
  }
  rows_kernel<<<(unsigned)((n_rows + 63) / 64), 64, 0, (cudaStream_t)stream>>>(m, leaf_gids, n_rows, codes, row_ptr,
                                                                              counts, gid_out, w_out, err);
  return finish("amr_dm_rows launch");
}
