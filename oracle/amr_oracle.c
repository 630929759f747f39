/*
 * amr_oracle.c — TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * `amrlts` algorithms (/root/reference/pkg/src/amrlts), used as the parity
 * checker by tests/, by __graft_entry__.smoke() and as bench.py's CPU
 * baseline ("port").  The product never links or calls this file.
 *
 * It follows the reference's *structure*, not the GPU design: maximal blocks
 * split at rank cuts, a sort-based node registry with coarse-neighbour
 * hanging detection, per-block CSR gathers, a zip-space stage source per
 * (level) group, padded-block RHS and record-based LTS time interpolation.
 * Pinned against goldens generated from the reference itself
 * (tests/golden/*.npz, tests/test_oracle.py).
 *
 * Cited reference code (file:line):
 *   octree.py:175-198 (Morton order), 279-330 (balance_2to1), 350-399 (neighbors)
 *   mesh.py:87-135 (decompose_blocks), 138-150 (_lagrange_weights),
 *   mesh.py:214-277 (_build_registry), 293-351 (_containing_leaves,
 *   _point_weights), 355-398 (_build_gathers)
 *   wave.py:57-201 (derivative_axis, wave_rhs, _radiative_faces)
 *   stepper.py:238-314 (_transfer, _virtual_state, _stage_source),
 *   stepper.py:370-456 (advance_slice)
 * The cubic source is the documented oracle extension of tests/golden/make_golden.py.
 *
 * Floating point: compiled with -ffp-contract=off; fma() only where the
 * reference goes through OpenBLAS dgemm (np.tensordot, stepper.py:264,305).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXP 4

static char g_err[512];
const char* ora_last_error(void) { return g_err; }
static int ora_fail(const char* m) {
  snprintf(g_err, sizeof g_err, "%s", m);
  return 1;
}

/* ------------------------------------------------------------ hash map -- */
typedef struct {
  uint64_t* keys;
  int64_t* vals;
  int64_t cap, n;
} HMap;

static uint64_t hmix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
static void hm_init(HMap* h, int64_t n) {
  int64_t cap = 16;
  while (cap < 2 * n + 16) cap <<= 1;
  h->cap = cap;
  h->n = 0;
  h->keys = (uint64_t*)malloc(cap * sizeof(uint64_t));
  h->vals = (int64_t*)malloc(cap * sizeof(int64_t));
  for (int64_t i = 0; i < cap; ++i) h->keys[i] = UINT64_MAX;
}
static void hm_free(HMap* h) {
  free(h->keys);
  free(h->vals);
  h->keys = NULL;
  h->vals = NULL;
}
static int64_t* hm_slot(HMap* h, uint64_t k, int create);
static void hm_grow(HMap* h) {
  HMap o = *h;
  hm_init(h, o.cap);
  for (int64_t i = 0; i < o.cap; ++i)
    if (o.keys[i] != UINT64_MAX) *hm_slot(h, o.keys[i], 1) = o.vals[i];
  hm_free(&o);
}
static int64_t* hm_slot(HMap* h, uint64_t k, int create) {
  if (create && 2 * (h->n + 1) > h->cap) hm_grow(h);
  int64_t i = (int64_t)(hmix(k) & (uint64_t)(h->cap - 1));
  for (;;) {
    if (h->keys[i] == k) return &h->vals[i];
    if (h->keys[i] == UINT64_MAX) {
      if (!create) return NULL;
      h->keys[i] = k;
      h->n++;
      return &h->vals[i];
    }
    i = (i + 1) & (h->cap - 1);
  }
}
static int64_t hm_get(const HMap* h, uint64_t k, int64_t dflt) {
  int64_t* s = hm_slot((HMap*)h, k, 0);
  return s ? *s : dflt;
}
static int hm_del(HMap* h, uint64_t k) {
  /* backward-shift deletion for linear probing */
  int64_t i = (int64_t)(hmix(k) & (uint64_t)(h->cap - 1));
  for (;;) {
    if (h->keys[i] == UINT64_MAX) return 0;
    if (h->keys[i] == k) break;
    i = (i + 1) & (h->cap - 1);
  }
  int64_t j = i;
  for (;;) {
    j = (j + 1) & (h->cap - 1);
    if (h->keys[j] == UINT64_MAX) break;
    int64_t home = (int64_t)(hmix(h->keys[j]) & (uint64_t)(h->cap - 1));
    int between = (i <= j) ? (i < home && home <= j) : (i < home || home <= j);
    if (between) continue;
    h->keys[i] = h->keys[j];
    h->vals[i] = h->vals[j];
    i = j;
  }
  h->keys[i] = UINT64_MAX;
  h->n--;
  return 1;
}

/* --------------------------------------------------------------- octree -- */
static uint64_t key_of(const int32_t* a, int dim, int level) {
  /* (anchor, level) packed; anchors < 2^20 */
  uint64_t k = (uint64_t)level;
  for (int d = 0; d < dim; ++d) k = (k << 20) | (uint64_t)a[d];
  return k;
}

/* Morton digit tuple comparison (octree.py:175-206) */
static int g_sort_dim, g_sort_L;
static const int32_t* g_sort_anchor;
static const int32_t* g_sort_level;
static int morton_cmp_idx(int64_t ia, int64_t ib) {
  const int dim = g_sort_dim, L = g_sort_L;
  const int32_t* a = g_sort_anchor + ia * dim;
  const int32_t* b = g_sort_anchor + ib * dim;
  int la = g_sort_level[ia], lb = g_sort_level[ib];
  int lm = la < lb ? la : lb;
  for (int depth = 1; depth <= lm; ++depth) {
    int sh = L - depth, ca = 0, cb = 0;
    for (int d = 0; d < dim; ++d) {
      ca |= ((a[d] >> sh) & 1) << d;
      cb |= ((b[d] >> sh) & 1) << d;
    }
    if (ca != cb) return ca < cb ? -1 : 1;
  }
  return la < lb ? -1 : (la > lb ? 1 : 0);
}
static int qs_cmp(const void* x, const void* y) {
  int c = morton_cmp_idx(*(const int64_t*)x, *(const int64_t*)y);
  if (c) return c;
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return a < b ? -1 : (a > b);
}
int ora_morton_sort(int dim, int L, int64_t n, const int32_t* anchors, const int32_t* levels, int64_t* perm) {
  g_sort_dim = dim;
  g_sort_L = L;
  g_sort_anchor = anchors;
  g_sort_level = levels;
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  qsort(perm, n, sizeof(int64_t), qs_cmp);
  return 0;
}

typedef struct {
  int dim, L;
  int64_t n;
  int32_t* anchors;
  int32_t* levels;
} OraTree;

static int leaf_containing_cell(const HMap* set, const int32_t* cell, int dim, int L, int32_t* anc) {
  for (int lvl = L; lvl >= 0; --lvl) {
    int sh = L - lvl;
    int32_t a[3];
    for (int d = 0; d < dim; ++d) a[d] = (cell[d] >> sh) << sh;
    if (hm_get(set, key_of(a, dim, lvl), -1) >= 0) {
      for (int d = 0; d < dim; ++d) anc[d] = a[d];
      return lvl;
    }
  }
  return -1;
}

/* balance_2to1 (octree.py:289-330): forced-split ripple, finest first */
OraTree* ora_balance(int dim, int L, int64_t n, const int32_t* anchors, const int32_t* levels, int64_t* n_out) {
  HMap set;
  hm_init(&set, n * 4);
  int64_t qcap = n * 8 + 64, qh = 0, qt = 0;
  int32_t* q = (int32_t*)malloc(qcap * 4 * sizeof(int32_t));
  /* sorted by -level (stable over input order) */
  for (int lv = L; lv >= 0; --lv)
    for (int64_t i = 0; i < n; ++i)
      if (levels[i] == lv) {
        for (int d = 0; d < dim; ++d) q[qt * 4 + d] = anchors[i * dim + d];
        q[qt * 4 + 3] = lv;
        ++qt;
      }
  for (int64_t i = 0; i < n; ++i) *hm_slot(&set, key_of(anchors + i * dim, dim, levels[i]), 1) = 1;
  const int32_t top = 1 << L;
  int ndir = dim == 3 ? 27 : 9;
  while (qh < qt) {
    int32_t anc[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) anc[d] = q[qh * 4 + d];
    int level = q[qh * 4 + 3];
    ++qh;
    if (hm_get(&set, key_of(anc, dim, level), -1) < 0) continue;
    int32_t side = 1 << (L - level);
    for (int di = 0; di < ndir; ++di) {
      int dv[3] = {di % 3 - 1, (di / 3) % 3 - 1, (di / 9) % 3 - 1};
      if (dim == 2) dv[2] = 0;
      if (!dv[0] && !dv[1] && !dv[2]) continue;
      int32_t cell[3];
      int ok = 1;
      for (int d = 0; d < dim; ++d) {
        int32_t c = dv[d] < 0 ? anc[d] - 1 : (dv[d] > 0 ? anc[d] + side : anc[d]);
        if (c < 0 || c >= top) ok = 0;
        cell[d] = c;
      }
      if (!ok) continue;
      int32_t nb[3];
      int nl = leaf_containing_cell(&set, cell, dim, L, nb);
      while (nl >= 0 && nl < level - 1) {
        hm_del(&set, key_of(nb, dim, nl));
        int32_t half = 1 << (L - nl - 1);
        for (int code = 0; code < (1 << dim); ++code) {
          int32_t ch[3];
          for (int d = 0; d < dim; ++d) ch[d] = nb[d] + (((code >> d) & 1) * half);
          *hm_slot(&set, key_of(ch, dim, nl + 1), 1) = 1;
          if (qt >= qcap) {
            qcap *= 2;
            q = (int32_t*)realloc(q, qcap * 4 * sizeof(int32_t));
          }
          for (int d = 0; d < dim; ++d) q[qt * 4 + d] = ch[d];
          q[qt * 4 + 3] = nl + 1;
          ++qt;
        }
        nl = leaf_containing_cell(&set, cell, dim, L, nb);
      }
    }
  }
  free(q);
  OraTree* t = (OraTree*)calloc(1, sizeof(OraTree));
  t->dim = dim;
  t->L = L;
  t->n = set.n;
  int32_t* an = (int32_t*)malloc(set.n * dim * sizeof(int32_t));
  int32_t* lv = (int32_t*)malloc(set.n * sizeof(int32_t));
  int64_t k = 0;
  for (int64_t i = 0; i < set.cap; ++i) {
    uint64_t key = set.keys[i];
    if (key == UINT64_MAX) continue;
    for (int d = dim - 1; d >= 0; --d) {
      an[k * dim + d] = (int32_t)(key & 0xFFFFF);
      key >>= 20;
    }
    lv[k] = (int32_t)key;
    ++k;
  }
  hm_free(&set);
  int64_t* perm = (int64_t*)malloc(t->n * sizeof(int64_t));
  ora_morton_sort(dim, L, t->n, an, lv, perm);
  t->anchors = (int32_t*)malloc(t->n * dim * sizeof(int32_t));
  t->levels = (int32_t*)malloc(t->n * sizeof(int32_t));
  for (int64_t i = 0; i < t->n; ++i) {
    for (int d = 0; d < dim; ++d) t->anchors[i * dim + d] = an[perm[i] * dim + d];
    t->levels[i] = lv[perm[i]];
  }
  free(perm);
  free(an);
  free(lv);
  *n_out = t->n;
  return t;
}
int ora_tree_fetch(const OraTree* t, int32_t* anchors, int32_t* levels) {
  memcpy(anchors, t->anchors, t->n * t->dim * sizeof(int32_t));
  memcpy(levels, t->levels, t->n * sizeof(int32_t));
  return 0;
}
void ora_tree_free(OraTree* t) {
  if (!t) return;
  free(t->anchors);
  free(t->levels);
  free(t);
}

/* ----------------------------------------------------------------- mesh -- */
typedef struct {
  int32_t anchor[3];
  int root_level, leaf_level, owner;
  int64_t a, b;
  int64_t n_int, n_pad; /* interior / padded points per axis */
  int64_t* g_ptr;       /* gather CSR over the padded grid */
  int64_t* g_col;
  double* g_val;
  int64_t* reads; /* read leaves (sorted) */
  int64_t n_reads;
  int faces; /* bit 2*axis+side */
} OraBlock;

typedef struct {
  int64_t n;
  int64_t* gid;
  double* w;
} Row;

typedef struct {
  int dim, L, ppo, pad, scale;
  int64_t top_nodes, n_leaves, n_nodes, per_leaf;
  int32_t* anchor; /* n*dim */
  int32_t* level;
  int32_t* owner;
  HMap leaf_index; /* key_of(anchor,level) -> leaf */
  int64_t* leaf_start; /* n+1 */
  int64_t* leaf_gids;  /* n*per_leaf, -1 hanging */
  int64_t* zip_pos;    /* per leaf owned points: flat position in its block's padded grid */
  int64_t* zip_ptr;    /* n+1 (== leaf_start) */
  int64_t* sorted_codes;
  int64_t* sorted_gids;
  int32_t* node_coords;
  OraBlock* blocks;
  int64_t n_blocks, blocks_cap;
  int64_t* leaf_block;
  double lo[3], hi[3];
  /* _point_weights memo: code -> row index */
  HMap memo;
  Row* rows;
  int64_t n_rows, rows_cap;
} OraMesh;

static int64_t enc(const OraMesh* m, const int64_t* p) {
  int64_t M = m->top_nodes + 1, c = p[0];
  for (int d = 1; d < m->dim; ++d) c = c * M + p[d];
  return c;
}
static int64_t spacing(const OraMesh* m, int lvl) { return (int64_t)1 << (m->L - lvl); }

static int64_t find_leaf(const OraMesh* m, const int32_t* a, int lvl) {
  return hm_get(&m->leaf_index, key_of(a, m->dim, lvl), -1);
}

/* neighbors(key, tree, scope="all") restricted to what the registry needs:
 * collect adjacent leaves (octree.py:350-399) */
static int neighbors_all(const OraMesh* m, int64_t leaf, int64_t* out) {
  const int dim = m->dim, L = m->L;
  const int32_t* an = m->anchor + leaf * dim;
  int level = m->level[leaf];
  int32_t side = 1 << (L - level), top = 1 << L;
  int nfound = 0;
  int ndir = dim == 3 ? 27 : 9;
  for (int di = 0; di < ndir; ++di) {
    int dv[3] = {di % 3 - 1, (di / 3) % 3 - 1, (di / 9) % 3 - 1};
    if (dim == 2) dv[2] = 0;
    if (!dv[0] && !dv[1] && !dv[2]) continue;
    if (dim == 2 && di >= 9) continue;
    int32_t cand[3];
    int ok = 1;
    for (int d = 0; d < dim; ++d) {
      cand[d] = an[d] + dv[d] * side;
      if (cand[d] < 0 || cand[d] >= top) ok = 0;
    }
    if (!ok) continue;
    int64_t hits[8];
    int nh = 0;
    int64_t j = find_leaf(m, cand, level);
    if (j >= 0) {
      hits[nh++] = j;
    } else {
      int32_t par[3];
      int64_t pj = -1;
      if (level > 0) {
        int32_t ps = side << 1;
        for (int d = 0; d < dim; ++d) par[d] = (cand[d] / ps) * ps;
        pj = find_leaf(m, par, level - 1);
      }
      if (pj >= 0) {
        hits[nh++] = pj;
      } else if (level < L) {
        int32_t half = side >> 1;
        int nchoice[3], choice[3][2];
        for (int d = 0; d < dim; ++d) {
          if (dv[d] > 0) {
            nchoice[d] = 1;
            choice[d][0] = 0;
          } else if (dv[d] < 0) {
            nchoice[d] = 1;
            choice[d][0] = half;
          } else {
            nchoice[d] = 2;
            choice[d][0] = 0;
            choice[d][1] = half;
          }
        }
        int tot = 1;
        for (int d = 0; d < dim; ++d) tot *= nchoice[d];
        for (int c = 0; c < tot; ++c) {
          int r = c;
          int32_t ch[3];
          for (int d = dim - 1; d >= 0; --d) {
            ch[d] = cand[d] + choice[d][r % nchoice[d]];
            r /= nchoice[d];
          }
          int64_t cj = find_leaf(m, ch, level + 1);
          if (cj >= 0) hits[nh++] = cj;
        }
      }
    }
    for (int h = 0; h < nh; ++h) {
      int dup = 0;
      for (int k = 0; k < nfound; ++k) dup |= out[k] == hits[h];
      if (!dup) out[nfound++] = hits[h];
    }
  }
  return nfound;
}

static void emit_block(OraMesh* m, const int32_t* node, int nlevel, int64_t a, int64_t b) {
  if (m->n_blocks == m->blocks_cap) {
    m->blocks_cap = m->blocks_cap ? 2 * m->blocks_cap : 64;
    m->blocks = (OraBlock*)realloc(m->blocks, m->blocks_cap * sizeof(OraBlock));
  }
  OraBlock* blk = &m->blocks[m->n_blocks++];
  memset(blk, 0, sizeof *blk);
  for (int d = 0; d < m->dim; ++d) blk->anchor[d] = node[d];
  blk->root_level = nlevel;
  blk->leaf_level = m->level[a];
  blk->owner = m->owner[a];
  blk->a = a;
  blk->b = b;
  blk->n_int = (int64_t)(m->ppo - 1) * ((int64_t)1 << (blk->leaf_level - nlevel)) + 1;
  blk->n_pad = blk->n_int + 2 * m->pad;
  int32_t side = 1 << (m->L - nlevel);
  for (int d = 0; d < m->dim; ++d) {
    if (node[d] == 0) blk->faces |= 1 << (2 * d);
    if (node[d] + side == (1 << m->L)) blk->faces |= 2 << (2 * d);
  }
}

/* decompose_blocks recursion (mesh.py:115-131).  Children are taken in the
 * tree's SFC order: leaves of one child are contiguous along any SFC, so the
 * children are the maximal runs of leaves sharing the child digit. */
static void decompose(OraMesh* m, const int32_t* node, int nlevel, int64_t a, int64_t b) {
  int lvl = m->level[a], uniform = 1;
  for (int64_t i = a; i < b; ++i)
    if (m->level[i] != lvl) uniform = 0;
  if (uniform && m->owner[a] == m->owner[b - 1]) {
    emit_block(m, node, nlevel, a, b);
    return;
  }
  int sh = m->L - (nlevel + 1);
  int64_t pos = a;
  while (pos < b) {
    int32_t ch[3];
    for (int d = 0; d < m->dim; ++d) ch[d] = (m->anchor[pos * m->dim + d] >> sh) << sh;
    int64_t end = pos;
    while (end < b) {
      int inside = 1;
      for (int d = 0; d < m->dim; ++d) inside &= ((m->anchor[end * m->dim + d] >> sh) << sh) == ch[d];
      if (!inside) break;
      ++end;
    }
    decompose(m, ch, nlevel + 1, pos, end);
    pos = end;
  }
}

static int64_t* g_codes_sort;
static int cmp_by_code(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  int64_t ca = g_codes_sort[a], cb = g_codes_sort[b];
  if (ca != cb) return ca < cb ? -1 : 1;
  return a < b ? -1 : (a > b);
}
static int cmp_i64(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return a < b ? -1 : (a > b);
}

static void leaf_point(const OraMesh* m, int64_t leaf, int64_t k, int64_t* p) {
  int64_t s = spacing(m, m->level[leaf]);
  int64_t r = k;
  int64_t loc[3];
  for (int d = m->dim - 1; d >= 0; --d) {
    loc[d] = r % m->ppo;
    r /= m->ppo;
  }
  for (int d = 0; d < m->dim; ++d) p[d] = (int64_t)m->anchor[leaf * m->dim + d] * m->scale + s * loc[d];
}

/* _build_registry (mesh.py:214-277) */
static int build_registry(OraMesh* m) {
  const int64_t n = m->n_leaves, P = m->per_leaf, N = n * P;
  const int dim = m->dim;
  int64_t* codes = (int64_t*)malloc(N * sizeof(int64_t));
  char* hanging = (char*)calloc(N, 1);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i) {
    int64_t nb[64];
    int nn = neighbors_all(m, i, nb);
    int lvl = m->level[i];
    int64_t coarse[64];
    int nc = 0;
    for (int k = 0; k < nn; ++k)
      if (m->level[nb[k]] == lvl - 1) coarse[nc++] = nb[k];
    int64_t s2 = lvl > 0 ? spacing(m, lvl - 1) : 1;
    for (int64_t k = 0; k < P; ++k) {
      int64_t p[3];
      leaf_point(m, i, k, p);
      codes[i * P + k] = enc(m, p);
      if (!nc) continue;
      int off = 0;
      for (int d = 0; d < dim; ++d) off |= (p[d] % s2) != 0;
      if (!off) continue;
      int cov = 0;
      for (int c = 0; c < nc && !cov; ++c) {
        int in = 1;
        int64_t side = (int64_t)1 << (m->L - m->level[coarse[c]]);
        for (int d = 0; d < dim; ++d) {
          int64_t lo = (int64_t)m->anchor[coarse[c] * dim + d] * m->scale;
          int64_t hi = lo + side * m->scale;
          in &= (p[d] >= lo && p[d] <= hi);
        }
        cov = in;
      }
      hanging[i * P + k] = (char)cov;
    }
  }
  /* np.unique(return_index, return_inverse) + logical_or.at */
  int64_t* order = (int64_t*)malloc(N * sizeof(int64_t));
  for (int64_t i = 0; i < N; ++i) order[i] = i;
  g_codes_sort = codes;
  qsort(order, N, sizeof(int64_t), cmp_by_code);
  int64_t* uniq_first = (int64_t*)malloc(N * sizeof(int64_t));
  char* uniq_hang = (char*)calloc(N, 1);
  int64_t* inverse = (int64_t*)malloc(N * sizeof(int64_t));
  int64_t nu = 0;
  for (int64_t k = 0; k < N; ++k) {
    int64_t idx = order[k];
    if (k == 0 || codes[order[k - 1]] != codes[idx]) {
      uniq_first[nu] = idx; /* order is (code, index)-sorted: first is the minimum index */
      ++nu;
    }
    inverse[idx] = nu - 1;
    uniq_hang[nu - 1] |= hanging[idx];
  }
  /* gids in discovery (first-occurrence) order over real points */
  int64_t* by_first = (int64_t*)malloc(nu * sizeof(int64_t));
  char* seen = (char*)calloc(N, 1);
  int64_t nb_ = 0;
  for (int64_t k = 0; k < N; ++k) {
    int64_t u = inverse[k];
    if (uniq_first[u] == k) by_first[nb_++] = u;
  }
  (void)seen;
  int64_t* gid_of_u = (int64_t*)malloc(nu * sizeof(int64_t));
  int64_t g = 0;
  for (int64_t k = 0; k < nu; ++k) {
    int64_t u = by_first[k];
    gid_of_u[u] = uniq_hang[u] ? -1 : g++;
  }
  m->n_nodes = g;
  m->leaf_gids = (int64_t*)malloc(N * sizeof(int64_t));
  m->leaf_start = (int64_t*)calloc(n + 1, sizeof(int64_t));
  for (int64_t k = 0; k < N; ++k) m->leaf_gids[k] = gid_of_u[inverse[k]];
  for (int64_t i = 0; i < n; ++i) {
    int64_t cnt = 0;
    for (int64_t k = 0; k < P; ++k) {
      int64_t idx = i * P + k;
      cnt += (uniq_first[inverse[idx]] == idx && m->leaf_gids[idx] >= 0);
    }
    m->leaf_start[i + 1] = m->leaf_start[i] + cnt;
  }
  m->node_coords = (int32_t*)malloc((m->n_nodes + 1) * dim * sizeof(int32_t));
  m->sorted_codes = (int64_t*)malloc((m->n_nodes + 1) * sizeof(int64_t));
  m->sorted_gids = (int64_t*)malloc((m->n_nodes + 1) * sizeof(int64_t));
  {
    int64_t r = 0;
    for (int64_t k = 0; k < N; ++k) {
      int64_t idx = order[k];
      if (k > 0 && codes[order[k - 1]] == codes[idx]) continue;
      int64_t gg = gid_of_u[inverse[idx]];
      if (gg < 0) continue;
      int64_t p[3];
      leaf_point(m, idx / P, idx % P, p);
      for (int d = 0; d < dim; ++d) m->node_coords[gg * dim + d] = (int32_t)p[d];
      m->sorted_codes[r] = codes[idx];
      m->sorted_gids[r] = gg;
      ++r;
    }
  }
  free(codes);
  free(hanging);
  free(order);
  free(uniq_first);
  free(uniq_hang);
  free(inverse);
  free(by_first);
  free(seen);
  free(gid_of_u);
  return 0;
}

static int64_t lookup_gid(const OraMesh* m, int64_t code) {
  int64_t lo = 0, hi = m->n_nodes;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (m->sorted_codes[mid] < code) lo = mid + 1;
    else hi = mid;
  }
  if (lo < m->n_nodes && m->sorted_codes[lo] == code) return m->sorted_gids[lo];
  return -1;
}

/* _containing_leaves (mesh.py:293-314) */
static int containing_leaves(const OraMesh* m, const int64_t* p, int64_t* out) {
  int n = 0;
  for (int sig = 0; sig < (1 << m->dim); ++sig) {
    int32_t cell[3];
    int ok = 1;
    for (int d = 0; d < m->dim; ++d) {
      int64_t q = ((sig >> d) & 1) ? p[d] : p[d] - 1;
      if (q < 0 || q >= m->top_nodes) ok = 0;
      cell[d] = (int32_t)(q / m->scale);
    }
    if (!ok) continue;
    for (int lvl = m->L; lvl >= 0; --lvl) {
      int sh = m->L - lvl;
      int32_t a[3];
      for (int d = 0; d < m->dim; ++d) a[d] = (cell[d] >> sh) << sh;
      int64_t j = find_leaf(m, a, lvl);
      if (j >= 0) {
        int dup = 0;
        for (int k = 0; k < n; ++k) dup |= out[k] == j;
        if (!dup) out[n++] = j;
        break;
      }
    }
  }
  qsort(out, n, sizeof(int64_t), cmp_i64);
  return n;
}

/* _lagrange_weights (mesh.py:138-150) */
static int lagrange(double xi, int nn, double* ws, int* npts) {
  int np_ = nn < 4 ? nn : 4;
  int w0 = (int)floor(xi) - 1;
  if (w0 > nn - np_) w0 = nn - np_;
  if (w0 < 0) w0 = 0;
  for (int a = 0; a < np_; ++a) {
    ws[a] = 1.0;
    for (int b = 0; b < np_; ++b)
      if (a != b) ws[a] *= (xi - (double)(w0 + b)) / ((double)(w0 + a) - (double)(w0 + b));
  }
  *npts = np_;
  return w0;
}

static int64_t new_row(OraMesh* m) {
  if (m->n_rows == m->rows_cap) {
    m->rows_cap = m->rows_cap ? 2 * m->rows_cap : 1024;
    m->rows = (Row*)realloc(m->rows, m->rows_cap * sizeof(Row));
  }
  memset(&m->rows[m->n_rows], 0, sizeof(Row));
  return m->n_rows++;
}

/* _point_weights (mesh.py:316-351): dict insertion order preserved */
static int64_t point_weights(OraMesh* m, const int64_t* p, int* err) {
  int64_t code = enc(m, p);
  int64_t hit = hm_get(&m->memo, (uint64_t)code, -1);
  if (hit >= 0) return hit;
  int64_t gid = lookup_gid(m, code);
  if (gid >= 0) {
    int64_t r = new_row(m);
    m->rows[r].n = 1;
    m->rows[r].gid = (int64_t*)malloc(sizeof(int64_t));
    m->rows[r].w = (double*)malloc(sizeof(double));
    m->rows[r].gid[0] = gid;
    m->rows[r].w[0] = 1.0;
    *hm_slot(&m->memo, (uint64_t)code, 1) = r;
    return r;
  }
  int64_t cont[8];
  int nc = containing_leaves(m, p, cont);
  if (!nc) {
    *err = 1;
    return -1;
  }
  int lvl = 1 << 30;
  for (int k = 0; k < nc; ++k)
    if (m->level[cont[k]] < lvl) lvl = m->level[cont[k]];
  int64_t leaf = -1;
  for (int k = 0; k < nc; ++k)
    if (m->level[cont[k]] == lvl) {
      leaf = cont[k];
      break;
    }
  int64_t s = spacing(m, m->level[leaf]);
  int64_t org[3];
  double ws[3][4];
  int w0[3], npt[3];
  for (int d = 0; d < m->dim; ++d) {
    org[d] = (int64_t)m->anchor[leaf * m->dim + d] * m->scale;
    double xi = (double)(p[d] - org[d]) / (double)s;
    w0[d] = lagrange(xi, m->ppo, ws[d], &npt[d]);
  }
  int64_t cap = 256, cnt = 0;
  int64_t* ag = (int64_t*)malloc(cap * sizeof(int64_t));
  double* aw = (double*)malloc(cap * sizeof(double));
  int tot = 1;
  for (int d = 0; d < m->dim; ++d) tot *= npt[d];
  for (int combo = 0; combo < tot; ++combo) {
    int c[3], r = combo;
    for (int d = m->dim - 1; d >= 0; --d) {
      c[d] = r % npt[d];
      r /= npt[d];
    }
    double w = 1.0;
    int64_t qpt[3];
    for (int d = 0; d < m->dim; ++d) {
      w *= ws[d][c[d]];
      qpt[d] = org[d] + (int64_t)(w0[d] + c[d]) * s;
    }
    if (w == 0.0) continue;
    int64_t sub = point_weights(m, qpt, err);
    if (*err) break;
    Row* sr = &m->rows[sub];
    for (int64_t k = 0; k < sr->n; ++k) {
      int64_t gg = sr->gid[k];
      double gw = sr->w[k];
      int64_t f = -1;
      for (int64_t t = 0; t < cnt; ++t)
        if (ag[t] == gg) {
          f = t;
          break;
        }
      if (f >= 0) {
        aw[f] = aw[f] + w * gw;
      } else {
        if (cnt == cap) {
          cap *= 2;
          ag = (int64_t*)realloc(ag, cap * sizeof(int64_t));
          aw = (double*)realloc(aw, cap * sizeof(double));
        }
        ag[cnt] = gg;
        aw[cnt] = 0.0 + w * gw;
        ++cnt;
      }
      sr = &m->rows[sub]; /* rows may have moved */
    }
  }
  int64_t r = new_row(m);
  m->rows[r].n = cnt;
  m->rows[r].gid = ag;
  m->rows[r].w = aw;
  *hm_slot(&m->memo, (uint64_t)code, 1) = r;
  return r;
}

static void sort_row(int64_t n, int64_t* g, double* w) {
  for (int64_t i = 1; i < n; ++i) {
    int64_t gk = g[i];
    double wk = w[i];
    int64_t j = i - 1;
    while (j >= 0 && g[j] > gk) {
      g[j + 1] = g[j];
      w[j + 1] = w[j];
      --j;
    }
    g[j + 1] = gk;
    w[j + 1] = wk;
  }
}

/* _build_gathers (mesh.py:355-398) */
static int build_gathers(OraMesh* m) {
  const int dim = m->dim;
  int err = 0;
  for (int64_t bi = 0; bi < m->n_blocks; ++bi) {
    OraBlock* b = &m->blocks[bi];
    int64_t s = spacing(m, b->leaf_level), n = b->n_pad;
    int64_t total = 1;
    for (int d = 0; d < dim; ++d) total *= n;
    int64_t org[3];
    for (int d = 0; d < dim; ++d) org[d] = (int64_t)b->anchor[d] * m->scale - m->pad * s;
    int64_t cap = total * 2 + 16, nnz = 0;
    b->g_ptr = (int64_t*)malloc((total + 1) * sizeof(int64_t));
    b->g_col = (int64_t*)malloc(cap * sizeof(int64_t));
    b->g_val = (double*)malloc(cap * sizeof(double));
    b->g_ptr[0] = 0;
    for (int64_t r = 0; r < total; ++r) {
      int64_t p[3], rem = r;
      int in_dom = 1;
      for (int d = dim - 1; d >= 0; --d) {
        p[d] = org[d] + s * (rem % n);
        rem /= n;
        in_dom &= (p[d] >= 0 && p[d] <= m->top_nodes);
      }
      if (in_dom) {
        int64_t gid = lookup_gid(m, enc(m, p));
        int64_t cnt;
        int64_t* gg;
        double* ww;
        int64_t one_g;
        double one_w = 1.0;
        int64_t tmpg[512];
        double tmpw[512];
        if (gid >= 0) {
          one_g = gid;
          gg = &one_g;
          ww = &one_w;
          cnt = 1;
        } else {
          int64_t row = point_weights(m, p, &err);
          if (err) return ora_fail("lattice point outside the domain");
          cnt = m->rows[row].n;
          if (cnt > 512) return ora_fail("interpolation row too long");
          memcpy(tmpg, m->rows[row].gid, cnt * sizeof(int64_t));
          memcpy(tmpw, m->rows[row].w, cnt * sizeof(double));
          sort_row(cnt, tmpg, tmpw);
          gg = tmpg;
          ww = tmpw;
        }
        if (nnz + cnt > cap) {
          cap = 2 * (nnz + cnt);
          b->g_col = (int64_t*)realloc(b->g_col, cap * sizeof(int64_t));
          b->g_val = (double*)realloc(b->g_val, cap * sizeof(double));
        }
        for (int64_t k = 0; k < cnt; ++k) {
          b->g_col[nnz] = gg[k];
          b->g_val[nnz] = ww[k];
          ++nnz;
        }
      }
      b->g_ptr[r + 1] = nnz;
    }
    /* read leaves: owners of the support (mesh.py:396-398) */
    int64_t* sup = (int64_t*)malloc((nnz + 1) * sizeof(int64_t));
    memcpy(sup, b->g_col, nnz * sizeof(int64_t));
    qsort(sup, nnz, sizeof(int64_t), cmp_i64);
    b->reads = (int64_t*)malloc((nnz + 1) * sizeof(int64_t));
    b->n_reads = 0;
    for (int64_t k = 0; k < nnz; ++k) {
      if (k && sup[k] == sup[k - 1]) continue;
      int64_t lo = 0, hi = m->n_leaves; /* searchsorted(starts, g, right) - 1 */
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (m->leaf_start[mid] <= sup[k]) lo = mid + 1;
        else hi = mid;
      }
      int64_t leaf = lo - 1;
      if (!b->n_reads || b->reads[b->n_reads - 1] != leaf) b->reads[b->n_reads++] = leaf;
    }
    free(sup);
  }
  return 0;
}

OraMesh* ora_mesh_build(int dim, int L, int ppo, int pad, int64_t n, const int32_t* anchors, const int32_t* levels,
                        const int32_t* owners, const double* lo, const double* hi) {
  OraMesh* m = (OraMesh*)calloc(1, sizeof(OraMesh));
  m->dim = dim;
  m->L = L;
  m->ppo = ppo;
  m->pad = pad;
  m->scale = ppo - 1;
  m->top_nodes = (int64_t)m->scale << L;
  m->n_leaves = n;
  m->per_leaf = 1;
  for (int d = 0; d < dim; ++d) m->per_leaf *= ppo;
  m->anchor = (int32_t*)malloc(n * dim * sizeof(int32_t));
  m->level = (int32_t*)malloc(n * sizeof(int32_t));
  m->owner = (int32_t*)calloc(n, sizeof(int32_t));
  memcpy(m->anchor, anchors, n * dim * sizeof(int32_t));
  memcpy(m->level, levels, n * sizeof(int32_t));
  if (owners) memcpy(m->owner, owners, n * sizeof(int32_t));
  for (int d = 0; d < dim; ++d) {
    m->lo[d] = lo[d];
    m->hi[d] = hi[d];
  }
  hm_init(&m->leaf_index, n);
  for (int64_t i = 0; i < n; ++i) *hm_slot(&m->leaf_index, key_of(anchors + i * dim, dim, levels[i]), 1) = i;
  int32_t root[3] = {0, 0, 0};
  decompose(m, root, 0, 0, n);
  m->leaf_block = (int64_t*)malloc(n * sizeof(int64_t));
  for (int64_t b = 0; b < m->n_blocks; ++b)
    for (int64_t i = m->blocks[b].a; i < m->blocks[b].b; ++i) m->leaf_block[i] = b;
  build_registry(m);
  hm_init(&m->memo, 1024);
  if (build_gathers(m)) return NULL;
  /* zip positions: owned points -> flat padded position in the block */
  m->zip_pos = (int64_t*)malloc((m->n_nodes + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    OraBlock* b = &m->blocks[m->leaf_block[i]];
    int64_t s = spacing(m, b->leaf_level);
    int64_t g0 = m->leaf_start[i], k2 = 0;
    for (int64_t k = 0; k < m->per_leaf; ++k) {
      int64_t g = m->leaf_gids[i * m->per_leaf + k];
      if (g < g0 || g >= m->leaf_start[i + 1]) continue;
      int64_t p[3], flat = 0;
      leaf_point(m, i, k, p);
      for (int d = 0; d < dim; ++d) {
        int64_t org = (int64_t)b->anchor[d] * m->scale - m->pad * s;
        flat = flat * b->n_pad + (p[d] - org) / s;
      }
      m->zip_pos[g0 + k2++] = flat;
    }
  }
  return m;
}

void ora_mesh_free(OraMesh* m) {
  if (!m) return;
  for (int64_t b = 0; b < m->n_blocks; ++b) {
    free(m->blocks[b].g_ptr);
    free(m->blocks[b].g_col);
    free(m->blocks[b].g_val);
    free(m->blocks[b].reads);
  }
  for (int64_t r = 0; r < m->n_rows; ++r) {
    free(m->rows[r].gid);
    free(m->rows[r].w);
  }
  free(m->rows);
  free(m->blocks);
  free(m->anchor);
  free(m->level);
  free(m->owner);
  free(m->leaf_start);
  free(m->leaf_gids);
  free(m->zip_pos);
  free(m->sorted_codes);
  free(m->sorted_gids);
  free(m->node_coords);
  free(m->leaf_block);
  hm_free(&m->leaf_index);
  hm_free(&m->memo);
  free(m);
}

int64_t ora_mesh_n_nodes(const OraMesh* m) { return m->n_nodes; }
int64_t ora_mesh_n_blocks(const OraMesh* m) { return m->n_blocks; }
int ora_mesh_leaf_starts(const OraMesh* m, int64_t* out) {
  memcpy(out, m->leaf_start, (m->n_leaves + 1) * sizeof(int64_t));
  return 0;
}
int ora_mesh_leaf_gids(const OraMesh* m, int64_t* out) {
  memcpy(out, m->leaf_gids, m->n_leaves * m->per_leaf * sizeof(int64_t));
  return 0;
}
int ora_mesh_node_coords(const OraMesh* m, int32_t* out) {
  memcpy(out, m->node_coords, m->n_nodes * m->dim * sizeof(int32_t));
  return 0;
}
int ora_mesh_blocks(const OraMesh* m, int64_t* leaf_range, int32_t* root_level, int32_t* leaf_level) {
  for (int64_t b = 0; b < m->n_blocks; ++b) {
    leaf_range[2 * b] = m->blocks[b].a;
    leaf_range[2 * b + 1] = m->blocks[b].b;
    root_level[b] = m->blocks[b].root_level;
    leaf_level[b] = m->blocks[b].leaf_level;
  }
  return 0;
}
/* gather CSR of block b: two-call (ptr NULL -> sizes) */
int ora_mesh_block_gather(const OraMesh* m, int64_t b, int64_t* rows, int64_t* nnz, int64_t* ptr, int64_t* col,
                          double* val) {
  const OraBlock* blk = &m->blocks[b];
  int64_t total = 1;
  for (int d = 0; d < m->dim; ++d) total *= blk->n_pad;
  *rows = total;
  *nnz = blk->g_ptr[total];
  if (ptr) {
    memcpy(ptr, blk->g_ptr, (total + 1) * sizeof(int64_t));
    memcpy(col, blk->g_col, *nnz * sizeof(int64_t));
    memcpy(val, blk->g_val, *nnz * sizeof(double));
  }
  return 0;
}

/* --------------------------------------------------------------- engine -- */
typedef struct {
  double d2c[5], d2e0[6], d2e1[6], d1c[5], d1e0[5], d1e1[5];
} Stencils;

typedef struct {
  OraMesh* m;
  int p;
  double a[MAXP][MAXP], w[MAXP];
  double cfl, dt_fine, r_eps;
  int nonlinear; /* 0,1 sin,2 cubic */
  double k_chi, k_phi;
  int l_max;
  int* cadence; /* per block */
  int* leaf_cad;
  Stencils st;
  /* records in zip layout (reference LeafRecord fields) */
  double* u_pre;  /* [2][n] */
  double* u_curr; /* [2][n] */
  double* K;      /* [p][2][n] */
  int64_t* t0;    /* per leaf */
  int64_t* dtu;   /* per leaf */
  /* padded block state */
  double** bu; /* st.u per block [2][pad^D] */
  double** bK; /* [p][2][int^D] per block */
  double** unz; /* current unzip per block */
  double* src;  /* zip-space stage source [2][n] (single rank: one group per level) */
  int64_t i_fine;
} OraEngine;

OraEngine* ora_engine_new(OraMesh* m, int p, const double* a, const double* w, double cfl, int mode_lts,
                          int nonlinear, double k_chi, double k_phi, const double* stencils) {
  OraEngine* e = (OraEngine*)calloc(1, sizeof(OraEngine));
  e->m = m;
  e->p = p;
  for (int i = 0; i < p; ++i) {
    e->w[i] = w[i];
    for (int j = 0; j < p; ++j) e->a[i][j] = a[i * p + j];
  }
  e->cfl = cfl;
  /* finest_spacing (mesh.py:480-481) = min over blocks of extent0*s/top */
  double hmin = INFINITY;
  int lmax = 0;
  for (int64_t b = 0; b < m->n_blocks; ++b) {
    double h = (m->hi[0] - m->lo[0]) * (double)spacing(m, m->blocks[b].leaf_level) / (double)m->top_nodes;
    if (h < hmin) hmin = h;
    if (m->blocks[b].leaf_level > lmax) lmax = m->blocks[b].leaf_level;
  }
  e->dt_fine = cfl * hmin;
  e->r_eps = hmin;
  e->l_max = lmax;
  e->nonlinear = nonlinear;
  e->k_chi = k_chi;
  e->k_phi = k_phi;
  memcpy(&e->st, stencils, sizeof(Stencils));
  e->cadence = (int*)malloc(m->n_blocks * sizeof(int));
  e->leaf_cad = (int*)malloc(m->n_leaves * sizeof(int));
  for (int64_t b = 0; b < m->n_blocks; ++b) {
    e->cadence[b] = mode_lts ? m->blocks[b].leaf_level : lmax;
    for (int64_t i = m->blocks[b].a; i < m->blocks[b].b; ++i) e->leaf_cad[i] = e->cadence[b];
  }
  int64_t n = m->n_nodes;
  e->u_pre = (double*)calloc(2 * n, sizeof(double));
  e->u_curr = (double*)calloc(2 * n, sizeof(double));
  e->K = (double*)calloc((size_t)p * 2 * n, sizeof(double));
  e->src = (double*)calloc(2 * n, sizeof(double));
  e->t0 = (int64_t*)calloc(m->n_leaves, sizeof(int64_t));
  e->dtu = (int64_t*)calloc(m->n_leaves, sizeof(int64_t));
  e->bu = (double**)calloc(m->n_blocks, sizeof(double*));
  e->bK = (double**)calloc(m->n_blocks, sizeof(double*));
  e->unz = (double**)calloc(m->n_blocks, sizeof(double*));
  for (int64_t b = 0; b < m->n_blocks; ++b) {
    int64_t np_ = 1, ni = 1;
    for (int d = 0; d < m->dim; ++d) {
      np_ *= m->blocks[b].n_pad;
      ni *= m->blocks[b].n_int;
    }
    e->bu[b] = (double*)calloc(2 * np_, sizeof(double));
    e->unz[b] = (double*)calloc(2 * np_, sizeof(double));
    e->bK[b] = (double*)calloc((size_t)p * 2 * np_, sizeof(double));
  }
  return e;
}

void ora_engine_free(OraEngine* e) {
  if (!e) return;
  for (int64_t b = 0; b < e->m->n_blocks; ++b) {
    free(e->bu[b]);
    free(e->bK[b]);
    free(e->unz[b]);
  }
  free(e->bu);
  free(e->bK);
  free(e->unz);
  free(e->u_pre);
  free(e->u_curr);
  free(e->K);
  free(e->src);
  free(e->t0);
  free(e->dtu);
  free(e->cadence);
  free(e->leaf_cad);
  free(e);
}

double ora_engine_dt_fine(const OraEngine* e) { return e->dt_fine; }

static void gather_block(const OraMesh* m, const OraBlock* b, const double* src, double* out) {
  int64_t total = 1, n = m->n_nodes;
  for (int d = 0; d < m->dim; ++d) total *= b->n_pad;
  for (int64_t r = 0; r < total; ++r) {
    double s0 = 0.0, s1 = 0.0;
    for (int64_t k = b->g_ptr[r]; k < b->g_ptr[r + 1]; ++k) {
      s0 = s0 + b->g_val[k] * src[b->g_col[k]];
      s1 = s1 + b->g_val[k] * src[n + b->g_col[k]];
    }
    out[r] = s0;
    out[total + r] = s1;
  }
}

/* load_zip (stepper.py:209-230) */
int ora_engine_load(OraEngine* e, const double* z) {
  OraMesh* m = e->m;
  int64_t n = m->n_nodes;
  memcpy(e->u_pre, z, 2 * n * sizeof(double));
  memcpy(e->u_curr, z, 2 * n * sizeof(double));
  memset(e->K, 0, (size_t)e->p * 2 * n * sizeof(double));
  for (int64_t i = 0; i < m->n_leaves; ++i) {
    e->t0[i] = 0;
    e->dtu[i] = (int64_t)1 << (e->l_max - e->leaf_cad[i]);
  }
  for (int64_t b = 0; b < m->n_blocks; ++b) gather_block(m, &m->blocks[b], z, e->bu[b]);
  e->i_fine = 0;
  return 0;
}

int ora_engine_current(const OraEngine* e, double* z) {
  memcpy(z, e->u_curr, 2 * e->m->n_nodes * sizeof(double));
  return 0;
}

/* derivative row on a padded block along one axis (wave.py:57-109) */
static double deriv(const Stencils* S, const double* arr, int64_t idx, int64_t stride, int order, int pos, int64_t nint,
                    int lo, int hi, double hp) {
  const double* w;
  int nw, off0, sign = 1;
  if (order == 2) {
    if (lo && pos == 0) { w = S->d2e0; nw = 6; off0 = 0; }
    else if (lo && pos == 1) { w = S->d2e1; nw = 6; off0 = -1; }
    else if (hi && pos == nint - 1) { w = S->d2e0; nw = 6; off0 = 0; sign = -1; }
    else if (hi && pos == nint - 2) { w = S->d2e1; nw = 6; off0 = 1; sign = -1; }
    else { w = S->d2c; nw = 5; off0 = -2; }
  } else {
    if (lo && pos == 0) { w = S->d1e0; nw = 5; off0 = 0; }
    else if (lo && pos == 1) { w = S->d1e1; nw = 5; off0 = -1; }
    else if (hi && pos == nint - 1) { w = S->d1e0; nw = 5; off0 = 0; sign = -1; }
    else if (hi && pos == nint - 2) { w = S->d1e1; nw = 5; off0 = 1; sign = -1; }
    else { w = S->d1c; nw = 5; off0 = -2; }
  }
  double ws = (order == 1 && sign < 0) ? -1.0 : 1.0; /* w * (-1)**order */
  double t = 0.0;
  for (int k = 0; k < nw; ++k) {
    int off = sign > 0 ? off0 + k : off0 - k; /* hi rows: negated offsets */
    double term = (w[k] * ws) * arr[idx + off * stride];
    t = k ? t + term : term;
  }
  return t / hp;
}

/* wave_rhs on one padded block (wave.py:147-201); out = K_s interior [2][nint^D] */
static void block_rhs(const OraEngine* e, const OraBlock* b, const double* y, double* out) {
  const OraMesh* m = e->m;
  const int dim = m->dim;
  const int64_t ni = b->n_int, np_ = b->n_pad, g = m->pad;
  int64_t tot_i = 1, tot_p = 1;
  for (int d = 0; d < dim; ++d) {
    tot_i *= ni;
    tot_p *= np_;
  }
  double h = (m->hi[0] - m->lo[0]) * (double)spacing(m, b->leaf_level) / (double)m->top_nodes;
  double h2 = pow(h, 2.0), r_eps2 = pow(e->r_eps, 2.0); /* Python h**2 / r_eps**2 -> libm pow */
  int64_t s = spacing(m, b->leaf_level);
  int64_t stride[3];
  stride[dim - 1] = 1;
  for (int d = dim - 2; d >= 0; --d) stride[d] = stride[d + 1] * np_;
  for (int64_t t = 0; t < tot_i; ++t) {
    int64_t pos[3], r = t, idx = 0;
    for (int d = dim - 1; d >= 0; --d) {
      pos[d] = r % ni;
      r /= ni;
    }
    for (int d = 0; d < dim; ++d) idx += (pos[d] + g) * stride[d];
    double x[3];
    for (int d = 0; d < dim; ++d) {
      int64_t lat = (int64_t)b->anchor[d] * m->scale - g * s + s * (pos[d] + g);
      x[d] = m->lo[d] + ((double)lat / (double)m->top_nodes) * (m->hi[d] - m->lo[d]);
    }
    double lap = 0.0;
    for (int d = 0; d < dim; ++d) {
      double term = deriv(&e->st, y, idx, stride[d], 2, (int)pos[d], ni, (b->faces >> (2 * d)) & 1,
                          (b->faces >> (2 * d + 1)) & 1, h2);
      lap = d ? lap + term : term;
    }
    double chi = y[idx], phi = y[tot_p + idx];
    double dchi = phi, dphi = lap;
    double r2 = 0.0 + x[0] * x[0];
    for (int d = 1; d < dim; ++d) r2 = r2 + x[d] * x[d];
    if (e->nonlinear == 1) dphi = dphi - sin(2.0 * chi) / (r2 > r_eps2 ? r2 : r_eps2);
    int face = 0;
    for (int d = 0; d < dim; ++d)
      face |= (((b->faces >> (2 * d)) & 1) && pos[d] == 0) || (((b->faces >> (2 * d + 1)) & 1) && pos[d] == ni - 1);
    if (e->nonlinear == 2 && !face) dphi = dphi - (chi * chi) * chi;
    if (face) {
      double rr = sqrt(r2);
      if (rr < e->r_eps) rr = e->r_eps;
      double rad[2];
      for (int v = 0; v < 2; ++v) {
        double acc = 0.0;
        for (int d = 0; d < dim; ++d) {
          double gr = deriv(&e->st, y + v * tot_p, idx, stride[d], 1, (int)pos[d], ni, (b->faces >> (2 * d)) & 1,
                            (b->faces >> (2 * d + 1)) & 1, h);
          acc = d ? acc + x[d] * gr : x[d] * gr;
        }
        rad[v] = acc / rr;
      }
      dchi = rad[0] - e->k_chi * (chi - 0.0);
      dphi = rad[1] - e->k_phi * (phi - 0.0);
    }
    out[t] = dchi;
    out[tot_i + t] = dphi;
  }
}

/* transfer matrices for this slice, supplied by the Python wrapper:
 * keys[k] = (delta, from, to), mats[k] = p x p (tril already applied) */
typedef struct {
  int64_t n;
  const int64_t* keys;
  const double* mats;
} Transfers;

static const double* find_M(const Transfers* T, int64_t d, int64_t f, int64_t t) {
  for (int64_t k = 0; k < T->n; ++k)
    if (T->keys[3 * k] == d && T->keys[3 * k + 1] == f && T->keys[3 * k + 2] == t) return T->mats + k * MAXP * MAXP;
  return NULL;
}

/* K' = M @ K for one record slice (np.tensordot -> OpenBLAS dgemm = ascending FMA chain) */
static void apply_M(const double* M, int p, const double* K, int64_t nn, int64_t g0, int64_t cnt, int j, double* out) {
  for (int v = 0; v < 2; ++v)
    for (int64_t q = 0; q < cnt; ++q) {
      double acc = 0.0;
      for (int k = 0; k < p; ++k) acc = fma(M[j * MAXP + k], K[((int64_t)k * 2 + v) * nn + g0 + q], acc);
      out[v * cnt + q] = acc;
    }
}

/* one fine slice (stepper.py:370-456), single rank */
int ora_engine_advance(OraEngine* e, int64_t n_keys, const int64_t* keys, const double* mats) {
  OraMesh* m = e->m;
  const int64_t i = e->i_fine, n = m->n_nodes;
  const int p = e->p;
  Transfers T = {n_keys, keys, mats};
  char* elig = (char*)calloc(m->n_blocks, 1);
  for (int64_t b = 0; b < m->n_blocks; ++b) elig[b] = (i % ((int64_t)1 << (e->l_max - e->cadence[b]))) == 0;
  /* groups by cadence level; read leaves per group */
  for (int s = 0; s < p; ++s) {
    for (int lvl = 0; lvl <= e->l_max; ++lvl) {
      int any = 0;
      for (int64_t b = 0; b < m->n_blocks; ++b) any |= elig[b] && e->cadence[b] == lvl;
      if (!any) continue;
      char* rl = (char*)calloc(m->n_leaves, 1);
      for (int64_t b = 0; b < m->n_blocks; ++b)
        if (elig[b] && e->cadence[b] == lvl)
          for (int64_t k = 0; k < m->blocks[b].n_reads; ++k) rl[m->blocks[b].reads[k]] = 1;
      const int64_t to = (int64_t)1 << (e->l_max - lvl);
      const double dt_to = (double)to * e->dt_fine;
      /* _stage_source (stepper.py:274-314) */
#pragma omp parallel for schedule(dynamic, 32)
      for (int64_t leaf = 0; leaf < m->n_leaves; ++leaf) {
        if (!rl[leaf]) continue;
        int64_t g0 = m->leaf_start[leaf], cnt = m->leaf_start[leaf + 1] - g0;
        if (!cnt) continue;
        int64_t blk = m->leaf_block[leaf];
        if (elig[blk] && e->dtu[leaf] == to) {
          for (int v = 0; v < 2; ++v)
            for (int64_t q = 0; q < cnt; ++q) {
              double val = 0.0 + e->u_curr[v * n + g0 + q];
              for (int j = 0; j < s; ++j)
                if (e->a[s][j] != 0.0) val = val + (dt_to * e->a[s][j]) * e->K[((int64_t)j * 2 + v) * n + g0 + q];
              e->src[v * n + g0 + q] = val;
            }
          continue;
        }
        int64_t delta;
        double* base = (double*)malloc(2 * cnt * sizeof(double));
        double* kp = (double*)malloc(2 * cnt * sizeof(double));
        if (elig[blk]) {
          delta = 0;
          for (int v = 0; v < 2; ++v) memcpy(base + v * cnt, e->u_curr + v * n + g0, cnt * sizeof(double));
        } else {
          int64_t per = (int64_t)1 << (e->l_max - e->cadence[blk]);
          delta = i - (i / per) * per;
          /* _virtual_state */
          const double* Mv = (delta == e->dtu[leaf]) ? NULL : find_M(&T, 0, e->dtu[leaf], delta);
          if (delta == e->dtu[leaf]) {
            for (int v = 0; v < 2; ++v) memcpy(base + v * cnt, e->u_curr + v * n + g0, cnt * sizeof(double));
          } else {
            for (int v = 0; v < 2; ++v) memcpy(base + v * cnt, e->u_pre + v * n + g0, cnt * sizeof(double));
            double dt = (double)delta * e->dt_fine;
            for (int q = 0; q < p; ++q) {
              if (e->w[q] == 0.0) continue;
              apply_M(Mv, p, e->K, n, g0, cnt, q, kp);
              for (int64_t r = 0; r < 2 * cnt; ++r) base[r] = base[r] + (dt * e->w[q]) * kp[r];
            }
          }
        }
        const double* M = find_M(&T, delta, e->dtu[leaf], to);
        for (int j = 0; j < s; ++j) {
          if (e->a[s][j] == 0.0) continue;
          apply_M(M, p, e->K, n, g0, cnt, j, kp);
          for (int64_t r = 0; r < 2 * cnt; ++r) base[r] = base[r] + (dt_to * e->a[s][j]) * kp[r];
        }
        for (int v = 0; v < 2; ++v) memcpy(e->src + v * n + g0, base + v * cnt, cnt * sizeof(double));
        free(base);
        free(kp);
      }
      /* unzip every eligible block of this group */
#pragma omp parallel for schedule(dynamic, 4)
      for (int64_t b = 0; b < m->n_blocks; ++b)
        if (elig[b] && e->cadence[b] == lvl) gather_block(m, &m->blocks[b], e->src, e->unz[b]);
      free(rl);
    }
    /* RHS + zip of K_s (stepper.py:405-429) */
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t b = 0; b < m->n_blocks; ++b) {
      if (!elig[b]) continue;
      OraBlock* blk = &m->blocks[b];
      int64_t tot_p = 1, tot_i = 1;
      for (int d = 0; d < m->dim; ++d) {
        tot_p *= blk->n_pad;
        tot_i *= blk->n_int;
      }
      if (s == 0) memcpy(e->bu[b], e->unz[b], 2 * tot_p * sizeof(double));
      double* kin = (double*)malloc(2 * tot_i * sizeof(double));
      block_rhs(e, blk, e->unz[b], kin);
      /* K[s] stored padded (interior filled), zip by positions */
      double* Kp = e->bK[b] + (int64_t)s * 2 * tot_p;
      for (int64_t t = 0; t < tot_i; ++t) {
        int64_t r = t, idx = 0, pos[3];
        for (int d = m->dim - 1; d >= 0; --d) {
          pos[d] = r % blk->n_int;
          r /= blk->n_int;
        }
        for (int d = 0; d < m->dim; ++d) idx = idx * blk->n_pad + pos[d] + m->pad;
        Kp[idx] = kin[t];
        Kp[tot_p + idx] = kin[tot_i + t];
      }
      free(kin);
      for (int64_t leaf = blk->a; leaf < blk->b; ++leaf)
        for (int64_t g = m->leaf_start[leaf]; g < m->leaf_start[leaf + 1]; ++g)
          for (int v = 0; v < 2; ++v) e->K[((int64_t)s * 2 + v) * n + g] = Kp[v * tot_p + m->zip_pos[g]];
    }
  }
  /* combine + record rotation (stepper.py:432-453) */
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t b = 0; b < m->n_blocks; ++b) {
    if (!elig[b]) continue;
    OraBlock* blk = &m->blocks[b];
    int64_t tot_p = 1;
    for (int d = 0; d < m->dim; ++d) tot_p *= blk->n_pad;
    double dt = (double)((int64_t)1 << (e->l_max - e->cadence[b])) * e->dt_fine;
    for (int64_t leaf = blk->a; leaf < blk->b; ++leaf) {
      for (int64_t g = m->leaf_start[leaf]; g < m->leaf_start[leaf + 1]; ++g) {
        int64_t pos = m->zip_pos[g];
        for (int v = 0; v < 2; ++v) {
          double un = e->bu[b][v * tot_p + pos];
          for (int q = 0; q < p; ++q)
            if (e->w[q] != 0.0) un = un + (dt * e->w[q]) * e->bK[b][((int64_t)q * 2 + v) * tot_p + pos];
          e->u_pre[v * n + g] = e->u_curr[v * n + g];
          e->u_curr[v * n + g] = un;
        }
      }
      e->t0[leaf] = i;
      e->dtu[leaf] = (int64_t)1 << (e->l_max - e->cadence[b]);
    }
  }
  free(elig);
  e->i_fine++;
  return 0;
}

/* ------------------------------------------------------------ wavelet -- */
/* Interpolation residual of n octants (wavelet.py:94-103), TEST ORACLE.
 * values [n][npd^dim] (last axis fastest), W [npd][nc].  Restates the
 * reference literally: recon = coarse; for each axis in order, recon =
 * tensordot(W, recon, axis) (an ascending FMA chain from 0 over the full
 * coarse axis, the OpenBLAS dgemm bits on the generating host); then the max
 * of |values - recon| over nodes with any odd index, NaN-propagating like
 * np.max.  Full tensors at every step, as the reference builds them. */
int ora_wavelet_coeff(int dim, int npd, int64_t n, const double* values, const double* W, double* coeff) {
  if (dim < 1 || dim > 3 || npd < 3 || (npd % 2) == 0) return ora_fail("ora_wavelet_coeff: bad dim/npd");
  const int nc = (npd + 1) / 2;
  int64_t nv = 1;
  for (int d = 0; d < dim; ++d) nv *= npd;
#pragma omp parallel for schedule(static)
  for (int64_t o = 0; o < n; ++o) {
    const double* v = values + o * nv;
    double a[15 * 15 * 15], b[15 * 15 * 15];
    int shp[3];
    for (int d = 0; d < dim; ++d) shp[d] = nc;
    /* coarse = values[::2, ::2, ...] */
    int64_t nco = 1;
    for (int d = 0; d < dim; ++d) nco *= nc;
    for (int64_t t = 0; t < nco; ++t) {
      int64_t r = t, src = 0, mul = 1;
      for (int d = dim - 1; d >= 0; --d) {
        int idx = (int)(r % nc);
        r /= nc;
        src += (int64_t)(2 * idx) * mul;
        mul *= npd;
      }
      a[t] = v[src];
    }
    for (int ax = 0; ax < dim; ++ax) {
      int nshp[3];
      for (int d = 0; d < dim; ++d) nshp[d] = shp[d];
      nshp[ax] = npd;
      int64_t tot = 1;
      for (int d = 0; d < dim; ++d) tot *= nshp[d];
      for (int64_t t = 0; t < tot; ++t) {
        int idx[3];
        int64_t r = t;
        for (int d = dim - 1; d >= 0; --d) { idx[d] = (int)(r % nshp[d]); r /= nshp[d]; }
        double acc = 0.0;
        for (int k = 0; k < nc; ++k) {
          int64_t s = 0;
          for (int d = 0; d < dim; ++d) s = s * shp[d] + (d == ax ? k : idx[d]);
          acc = fma(W[idx[ax] * nc + k], a[s], acc);
        }
        b[t] = acc;
      }
      memcpy(a, b, sizeof(double) * tot);
      for (int d = 0; d < dim; ++d) shp[d] = nshp[d];
    }
    double m = 0.0;
    int any = 0;
    for (int64_t t = 0; t < nv; ++t) {
      int64_t r = t;
      int odd = 0;
      for (int d = dim - 1; d >= 0; --d) { odd |= (int)(r % npd) & 1; r /= npd; }
      if (!odd) continue;
      double dlt = fabs(v[t] - a[t]);
      if (!any) m = dlt;
      else if (!isnan(m) && (isnan(dlt) || dlt > m)) m = dlt;
      any = 1;
    }
    coeff[o] = m;
  }
  return 0;
}
