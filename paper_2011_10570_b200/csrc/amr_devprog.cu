// amr_devprog.cu — the per-tile stage programs on the device: the passes of
// amr_programs.cpp (host) / tileprog.build_programs (numpy), one thread per
// tile over a fixed grid, with per-thread scratch in global memory.  The
// output is byte-identical to the host builder's (tests/test_devprog_gpu.py).
//
//   amr_dp_need    owned-cross mask of every tile (which cross entries the
//                  owned stencils read), the interpolation rows those entries
//                  use, and the number of LTS interface-pair candidates;
//   amr_dp_keys    the candidates (31 - reader cadence) << 32 | gid, at the
//                  caller's prefix offsets; the caller sorts/uniques them;
//   amr_dp_encode  head and tail of every tile: with heads == NULL the sizes
//                  (head bytes, tail bytes, slots, rows, cells), else the
//                  bytes at stride max_head / at tail_off.
// Layouts: tileprog.py's module docstring.
#include "amr_common.cuh"

namespace {

constexpr int HDR_WORDS = 16;
constexpr int RUN_MAX = 8;
constexpr int MAX_SLOTS = 1023;  // usable: < 1023
constexpr int MAX_ROWS = 1024;   // usable: < 1024

struct DP {
  int dim, L, ppo, lts, RS, NI, E, box_n, n_wtab, max_bases;
  int bs[3];
  int64_t n_leaves, n_tiles, n_iface;
  const int32_t* table;    // [n_leaves][E]
  const int64_t* starts;   // [n_leaves + 1]
  const int32_t* anchor;   // [n_leaves][dim]
  const int32_t* level;
  const int32_t* leaf_cad;
  const int32_t* tiles;    // launch order
  const int64_t* iptr;
  const int32_t* igid;
  const double* iw;
  const int32_t* cell;     // [E] box cell of a cross entry
  const int32_t* cell2e;   // [box_n] -> entry or -1
  const int16_t* pos;      // [NI][3] interior position
  const int64_t* ukeys;    // sorted unique pair keys
  const int64_t* grp_start;
  const double* wtab;      // sorted
};

__device__ __forceinline__ int64_t node_leaf(const DP& p, int64_t g) {  // owner leaf of zip node g
  int64_t lo = 0, hi = p.n_leaves;                                      // last i with starts[i] <= g
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (p.starts[mid] <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int tile_faces(const DP& p, int64_t leaf) {
  int faces = 0;
  const int64_t side = (int64_t)1 << (p.L - p.level[leaf]);
  for (int d = 0; d < p.dim; ++d) {
    const int64_t a = p.anchor[leaf * p.dim + d];
    if (a == 0) faces |= 1 << (2 * d);
    if (a + side == ((int64_t)1 << p.L)) faces |= 2 << (2 * d);
  }
  return faces;
}

__device__ __forceinline__ int64_t r16(int64_t b) { return (b + 15) / 16 * 16; }

// ---- need mask, used rows, candidate-key counts
__global__ void need_kernel(DP p, uint8_t* __restrict__ need_all, uint8_t* __restrict__ row_used,
                            int64_t* __restrict__ n_keys) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.n_tiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t leaf = p.tiles[t];
    const int32_t* row = p.table + leaf * p.E;
    uint8_t* need = need_all + t * p.E;
    const int64_t g0 = p.starts[leaf], g1 = p.starts[leaf + 1];
    const int faces = tile_faces(p, leaf);
    for (int e = 0; e < p.E; ++e) need[e] = 0;
    for (int e = 0; e < p.NI; ++e) {
      if (!(row[e] >= g0 && row[e] < g1)) continue;
      need[e] = 1;
      for (int d = 0; d < p.dim; ++d) {
        for (int o = -2; o <= 2; ++o) need[p.cell2e[p.cell[e] + o * p.bs[d]]] = 1;
        const int q = p.pos[e * 3 + d];
        const bool lo = (faces >> (2 * d)) & 1, hi = (faces >> (2 * d + 1)) & 1;
        if ((lo && q <= 1) || (hi && q >= p.ppo - 2))
          for (int o = -5; o <= 5; ++o) {
            if (q + o < 0 || q + o >= p.ppo) continue;
            need[p.cell2e[p.cell[e] + o * p.bs[d]]] = 1;
          }
      }
    }
    const int tc = p.leaf_cad[leaf];
    int64_t nk = 0;
    for (int e = 0; e < p.E; ++e) {
      if (!need[e]) continue;
      const int32_t v = row[e];
      if (v >= 0) {
        if (p.lts && p.leaf_cad[node_leaf(p, v)] != tc) ++nk;
      } else if (v <= -2) {
        const int64_t r = -(int64_t)v - 2;
        row_used[r] = 1;
        if (p.lts)
          for (int64_t k = p.iptr[r]; k < p.iptr[r + 1]; ++k)
            if (p.leaf_cad[node_leaf(p, p.igid[k])] != tc) ++nk;
      }
    }
    n_keys[t] = nk;
  }
}

__global__ void keys_kernel(DP p, const uint8_t* __restrict__ need_all, const int64_t* __restrict__ key_off,
                            int64_t* __restrict__ keys) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.n_tiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t leaf = p.tiles[t];
    const int32_t* row = p.table + leaf * p.E;
    const uint8_t* need = need_all + t * p.E;
    const int tc = p.leaf_cad[leaf];
    int64_t o = key_off[t];
    for (int e = 0; e < p.E; ++e) {
      if (!need[e]) continue;
      const int32_t v = row[e];
      if (v >= 0) {
        if (p.leaf_cad[node_leaf(p, v)] != tc) keys[o++] = ((int64_t)(31 - tc) << 32) | (uint32_t)v;
      } else if (v <= -2) {
        const int64_t r = -(int64_t)v - 2;
        for (int64_t k = p.iptr[r]; k < p.iptr[r + 1]; ++k)
          if (p.leaf_cad[node_leaf(p, p.igid[k])] != tc) keys[o++] = ((int64_t)(31 - tc) << 32) | (uint32_t)p.igid[k];
      }
    }
  }
}

// a source of the tile: (base value, offset)
__device__ __forceinline__ void src_of_gid(const DP& p, int tc, int64_t g, int64_t* base, int64_t* off) {
  const int64_t lf = node_leaf(p, g);
  if (p.lts && p.leaf_cad[lf] != tc) {
    const int64_t key = ((int64_t)(31 - tc) << 32) | (uint32_t)g;
    int64_t lo = 0, hi = p.n_iface - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (p.ukeys[mid] < key) lo = mid + 1; else hi = mid;
    }
    *base = -p.grp_start[lo] - 1;
    *off = lo - p.grp_start[lo];
  } else {
    *base = p.starts[lf];
    *off = g - *base;
  }
}

__device__ __forceinline__ int find_i64(const int64_t* a, int n, int64_t v) {  // lower_bound
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int find_i32(const int32_t* a, int n, int32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int widx_of(const DP& p, double w) {
  int lo = 0, hi = p.n_wtab;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p.wtab[mid] < w) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// sorted-unique insert; returns false when the array is full
template <class T>
__device__ __forceinline__ bool insert_unique(T* a, int* n, int cap, T v) {
  int lo = 0, hi = *n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  if (lo < *n && a[lo] == v) return true;
  if (*n >= cap) return false;
  for (int k = *n; k > lo; --k) a[k] = a[k - 1];
  a[lo] = v;
  ++*n;
  return true;
}

// per-thread scratch
struct Scratch {
  int32_t slots[MAX_SLOTS + 1];
  int64_t bases[64];
  int32_t hr_cnt[MAX_ROWS];
  int32_t hr_e[MAX_ROWS];
};

__global__ void encode_kernel(DP p, const uint8_t* __restrict__ need_all, Scratch* __restrict__ scratch,
                              int64_t* __restrict__ sizes /* [n_tiles][5] */, uint8_t* __restrict__ heads,
                              int64_t max_head, const int64_t* __restrict__ tail_off, uint16_t* __restrict__ tail,
                              int* __restrict__ err) {
  Scratch& S = scratch[(int64_t)blockIdx.x * blockDim.x + threadIdx.x];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < p.n_tiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t leaf = p.tiles[t];
    const int32_t* row = p.table + leaf * p.E;
    const uint8_t* need = need_all + t * p.E;
    const int64_t g0 = p.starts[leaf], g1 = p.starts[leaf + 1];
    const int tc = p.leaf_cad[leaf];
    const int faces = tile_faces(p, leaf);
    // hanging rows, (count desc, entry asc); cells
    int nrow = 0, e_bits = 0;
    int64_t ncells = 0;
    for (int e = 0; e < p.E; ++e) {
      if (!need[e]) continue;
      ++ncells;
      if (row[e] <= -2) {
        if (nrow >= MAX_ROWS - 1) {
          e_bits |= 8;
          break;
        }
        const int64_t r = -(int64_t)row[e] - 2;
        const int32_t cnt = (int32_t)(p.iptr[r + 1] - p.iptr[r]);
        int k = nrow - 1;  // insertion: entries arrive in ascending e, so equal counts keep e order
        while (k >= 0 && S.hr_cnt[k] < cnt) {
          S.hr_cnt[k + 1] = S.hr_cnt[k];
          S.hr_e[k + 1] = S.hr_e[k];
          --k;
        }
        S.hr_cnt[k + 1] = cnt;
        S.hr_e[k + 1] = e;
        ++nrow;
      }
    }
    // slots: unique tap gids, ascending
    int nslot = 0;
    for (int i = 0; i < nrow && !e_bits; ++i) {
      const int64_t r = -(int64_t)row[S.hr_e[i]] - 2;
      for (int64_t k = p.iptr[r]; k < p.iptr[r + 1]; ++k)
        if (!insert_unique<int32_t>(S.slots, &nslot, MAX_SLOTS - 1, p.igid[k])) {
          e_bits |= 1;
          break;
        }
    }
    // bases: unique source groups of copies and slots, ascending
    int nbase = 0;
    for (int e = 0; e < p.E && !e_bits; ++e) {
      if (!need[e] || row[e] < 0) continue;
      int64_t b, o;
      src_of_gid(p, tc, row[e], &b, &o);
      if (o >= 1024) e_bits |= 4;
      if (!insert_unique<int64_t>(S.bases, &nbase, 64, b)) e_bits |= 2;
    }
    for (int k = 0; k < nslot && !e_bits; ++k) {
      int64_t b, o;
      src_of_gid(p, tc, S.slots[k], &b, &o);
      if (o >= 1024) e_bits |= 4;
      if (!insert_unique<int64_t>(S.bases, &nbase, 64, b)) e_bits |= 2;
    }
    if (nbase > p.max_bases) e_bits |= 2;
    if (e_bits) {
      atomicOr(err, e_bits);
      if (!heads) {
        for (int k = 0; k < 5; ++k) sizes[t * 5 + k] = 0;
      }
      continue;
    }
    // runs, in box-cell order: counts per bucket first
    int bcnt[4] = {0, 0, 0, 0};
    int nrun = 0;
    {
      int len = 0;
      int64_t pc = -10, pcode = -10;
      for (int c = 0; c <= p.box_n; ++c) {
        const int e = c < p.box_n ? p.cell2e[c] : -1;
        const bool is_copy = e >= 0 && need[e] && row[e] >= 0;
        int64_t code = -1;
        if (is_copy) {
          int64_t b, o;
          src_of_gid(p, tc, row[e], &b, &o);
          code = ((int64_t)find_i64(S.bases, nbase, b) << 10) | o;
        }
        const bool cont = is_copy && len > 0 && len < RUN_MAX && c == pc + 1 && c % p.RS != 0 &&
                          (code >> 10) == (pcode >> 10) && (code & 1023) == (pcode & 1023) + 1;
        if (!cont) {
          if (len > 0) {
            ++bcnt[len > 4 ? 0 : len > 2 ? 1 : len > 1 ? 2 : 3];
            ++nrun;
          }
          len = is_copy ? 1 : 0;
        } else {
          ++len;
        }
        if (is_copy) {
          pc = c;
          pcode = code;
        }
      }
    }
    // taps
    int64_t ntap = 0;
    for (int i = 0; i < nrow; ++i) ntap += (S.hr_cnt[i] + 3) / 4 * 4;
    const int64_t off_base = 4 * HDR_WORDS;
    const int64_t off_run = off_base + r16(4 * nbase);
    const int64_t off_slot = off_run + r16(4 * nrun);
    const int64_t head_len = off_slot + r16(2 * nslot);
    const int64_t rows_b = r16(4 * nrow);
    const int64_t tail_len = rows_b + r16(2 * ntap);
    if (!heads) {
      sizes[t * 5 + 0] = head_len;
      sizes[t * 5 + 1] = tail_len;
      sizes[t * 5 + 2] = nslot;
      sizes[t * 5 + 3] = nrow;
      sizes[t * 5 + 4] = ncells;
      continue;
    }
    // ---- write the head
    uint32_t* h = reinterpret_cast<uint32_t*>(heads + t * max_head);
    for (int64_t k = 0; k < max_head / 4; ++k) h[k] = 0u;
    const int64_t lmeta = p.level[leaf] | ((int64_t)tc << 8) | ((int64_t)faces << 16);
    int32_t a3[3] = {0, 0, 0};
    for (int d = 0; d < p.dim; ++d) a3[d] = p.anchor[leaf * p.dim + d];
    const int64_t hdr[HDR_WORDS] = {g0, g1 - g0, lmeta, nrun, nslot, nrow, nbase, tail_len, a3[0], a3[1], a3[2],
                                    bcnt[0] | ((int64_t)bcnt[1] << 16), bcnt[2] | ((int64_t)bcnt[3] << 16), 0,
                                    tail_off[t] / 16, rows_b / 2};
    for (int k = 0; k < HDR_WORDS; ++k) h[k] = (uint32_t)hdr[k];
    for (int k = 0; k < nbase; ++k) h[off_base / 4 + k] = (uint32_t)(int32_t)S.bases[k];
    {  // runs placed by bucket, cell order inside a bucket
      int wpos[4] = {0, bcnt[0], bcnt[0] + bcnt[1], bcnt[0] + bcnt[1] + bcnt[2]};
      int len = 0;
      int64_t pc = -10, pcode = -10, c0 = 0, code0 = 0;
      for (int c = 0; c <= p.box_n; ++c) {
        const int e = c < p.box_n ? p.cell2e[c] : -1;
        const bool is_copy = e >= 0 && need[e] && row[e] >= 0;
        int64_t code = -1;
        if (is_copy) {
          int64_t b, o;
          src_of_gid(p, tc, row[e], &b, &o);
          code = ((int64_t)find_i64(S.bases, nbase, b) << 10) | o;
        }
        const bool cont = is_copy && len > 0 && len < RUN_MAX && c == pc + 1 && c % p.RS != 0 &&
                          (code >> 10) == (pcode >> 10) && (code & 1023) == (pcode & 1023) + 1;
        if (!cont) {
          if (len > 0) {
            const int b = len > 4 ? 0 : len > 2 ? 1 : len > 1 ? 2 : 3;
            h[off_run / 4 + wpos[b]++] = (uint32_t)(c0 | ((int64_t)(len - 1) << 12) | (code0 << 16));
          }
          len = is_copy ? 1 : 0;
          c0 = c;
          code0 = code;
        } else {
          ++len;
        }
        if (is_copy) {
          pc = c;
          pcode = code;
        }
      }
    }
    uint16_t* h16 = reinterpret_cast<uint16_t*>(h);
    for (int k = 0; k < nslot; ++k) {
      int64_t b, o;
      src_of_gid(p, tc, S.slots[k], &b, &o);
      h16[off_slot / 2 + k] = (uint16_t)(((int64_t)find_i64(S.bases, nbase, b) << 10) | o);
    }
    // ---- the tail: row words, then taps (rows padded to quads with the zero slot / zero weight)
    uint16_t* tl = tail + tail_off[t] / 2;
    for (int64_t k = 0; k < tail_len / 2; ++k) tl[k] = 0;
    uint32_t* rw = reinterpret_cast<uint32_t*>(tl);
    uint16_t* taps = tl + rows_b / 2;
    const int zero_w = widx_of(p, 0.0);
    int64_t nt = 0;
    for (int i = 0; i < nrow; ++i) {
      const int e = S.hr_e[i];
      const int64_t r = -(int64_t)row[e] - 2;
      const int64_t cnt = S.hr_cnt[i];
      const int64_t nq = (cnt + 3) / 4, qoff = nt / 4;
      if (nq > 31 || qoff >= (1 << 15) || p.cell[e] >= (1 << 12)) {
        atomicOr(err, 16);
        break;
      }
      rw[i] = (uint32_t)(p.cell[e] | (nq << 12) | (qoff << 17));
      for (int64_t k = p.iptr[r]; k < p.iptr[r + 1]; ++k)
        taps[nt++] = (uint16_t)((find_i32(S.slots, nslot, p.igid[k]) << 6) | widx_of(p, p.iw[k]));
      for (int64_t k = cnt; k < 4 * nq; ++k) taps[nt++] = (uint16_t)((nslot << 6) | zero_w);
    }
  }
}

int finish(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, what);
}

}  // namespace

// AmrDevProg: plain-pointer view of the builder's inputs (all device memory)
extern "C" int amr_dp_scratch_bytes(int threads_total, int64_t* bytes) {
  *bytes = (int64_t)threads_total * (int64_t)sizeof(Scratch);
  return AMR_OK;
}

static DP make_dp(const AmrDevProg* a) {
  DP p;
  p.dim = a->dim;
  p.L = a->max_depth;
  p.ppo = a->ppo;
  p.lts = a->lts;
  const int NP = a->ppo + 4;
  p.RS = a->row_stride > NP ? a->row_stride : NP;
  if (a->dim == 3) {
    p.bs[0] = NP * p.RS;
    p.bs[1] = p.RS;
    p.bs[2] = 1;
  } else {
    p.bs[0] = p.RS;
    p.bs[1] = 1;
    p.bs[2] = 0;
  }
  p.box_n = (a->dim == 3 ? NP : 1) * NP * p.RS;
  p.NI = 1;
  for (int d = 0; d < a->dim; ++d) p.NI *= a->ppo;
  p.E = p.NI + 2 * a->dim * 2 * (p.NI / a->ppo);
  p.n_wtab = a->n_wtab;
  p.max_bases = a->max_bases > 0 && a->max_bases < 63 ? a->max_bases : 63;
  p.n_leaves = a->n_leaves;
  p.n_tiles = a->n_tiles;
  p.n_iface = a->n_iface;
  p.table = a->table;
  p.starts = a->starts;
  p.anchor = a->anchors;
  p.level = a->levels;
  p.leaf_cad = a->leaf_cad;
  p.tiles = a->tiles;
  p.iptr = a->row_ptr;
  p.igid = a->gid;
  p.iw = a->w;
  p.cell = a->cell;
  p.cell2e = a->cell2e;
  p.pos = a->pos;
  p.ukeys = a->ukeys;
  p.grp_start = a->grp_start;
  p.wtab = a->wtab;
  return p;
}

extern "C" int amr_dp_need(const AmrDevProg* a, uint8_t* need, uint8_t* row_used, int64_t* n_keys, int blocks,
                           int threads, void* stream) {
  if (a->n_tiles <= 0) return AMR_OK;
  need_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(make_dp(a), need, row_used, n_keys);
  return finish("amr_dp_need launch");
}

extern "C" int amr_dp_keys(const AmrDevProg* a, const uint8_t* need, const int64_t* key_off, int64_t* keys,
                           int blocks, int threads, void* stream) {
  if (a->n_tiles <= 0) return AMR_OK;
  keys_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(make_dp(a), need, key_off, keys);
  return finish("amr_dp_keys launch");
}

extern "C" int amr_dp_encode(const AmrDevProg* a, const uint8_t* need, void* scratch, int64_t* sizes, uint8_t* heads,
                             int64_t max_head, const int64_t* tail_off, uint16_t* tail, int* err, int blocks,
                             int threads, void* stream) {
  if (a->n_tiles <= 0) return AMR_OK;
  encode_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(make_dp(a), need, (Scratch*)scratch, sizes, heads,
                                                              max_head, tail_off, tail, err);
  return finish("amr_dp_encode launch");
}
