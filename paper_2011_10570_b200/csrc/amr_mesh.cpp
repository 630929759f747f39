// amr_mesh.cpp — host-side (C++/OpenMP) octree balance, node registry and
// leaf-tile unzip tables for the B200 wave solver.
//
// This is setup code, not the per-step hot path: it produces the integer
// tables the stage kernel (amr_kernels.cu) consumes.  The algorithms are
// restated B200-first rather than translated:
//  * balance_2to1 (octree.py:289-330) keeps the reference's forced-split
//    ripple (its fixed point is the unique minimal balanced refinement) on a
//    hash set of packed Morton keys;
//  * the node registry (mesh.py:214-277) is computed per leaf without a global
//    sort: under 2:1 balance a lattice point is a real (non-hanging) node iff
//    it lies on the lattice of every leaf whose closed box contains it, and its
//    owner is the lowest-SFC of those leaves ("first claim").  Owned points in
//    C order give the same gids as the reference's np.unique/first-occurrence
//    pass;
//  * interpolation rows follow _point_weights (mesh.py:316-351) exactly,
//    including the dict insertion order that fixes the accumulation order.
// Compiled with -ffp-contract=off: every weight must round like numpy.
#include "../../include/amr_b200.h"

#include <omp.h>

#include <chrono>
#include <cstdlib>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

inline uint64_t morton_code(const int32_t* a, int dim, int L) {
  uint64_t code = 0;
  for (int bit = 0; bit < L; ++bit)
    for (int d = 0; d < dim; ++d) code |= (uint64_t)((a[d] >> bit) & 1) << (bit * dim + d);
  return code;
}

inline void morton_decode(uint64_t code, int dim, int L, int32_t* a) {
  for (int d = 0; d < dim; ++d) a[d] = 0;
  for (int bit = 0; bit < L; ++bit)
    for (int d = 0; d < dim; ++d) a[d] |= (int32_t)((code >> (bit * dim + d)) & 1) << bit;
}

inline uint64_t pack_key(uint64_t code, int level) { return (code << 5) | (uint64_t)level; }

inline int ipow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

}  // namespace

struct AmrTree {
  int dim, L;
  std::vector<int32_t> anchors;  // n*dim
  std::vector<int32_t> levels;
};

extern "C" const char* amr_last_error(void) { return g_err.c_str(); }
extern "C" void amr_set_error_internal(const char* msg) { g_err = msg; }
extern "C" int amr_abi_version(void) { return 1; }

extern "C" int amr_morton_sort(int dim, int max_depth, int64_t n, const int32_t* anchors,
                               const int32_t* levels, int64_t* perm) {
  if (dim != 2 && dim != 3) return fail(AMR_EINVAL, "dimension must be 2 or 3");
  if (max_depth < 0 || max_depth * dim > 58) return fail(AMR_EINVAL, "max_depth too large for Morton keys");
  std::vector<std::pair<uint64_t, int32_t>> keys(n);
  for (int64_t i = 0; i < n; ++i) keys[i] = {morton_code(anchors + i * dim, dim, max_depth), levels[i]};
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  std::stable_sort(perm, perm + n, [&](int64_t a, int64_t b) { return keys[a] < keys[b]; });
  return AMR_OK;
}

// ---------------------------------------------------------------------------
// 2:1 balance (octree.py:289-330)
// ---------------------------------------------------------------------------

extern "C" AmrTree* amr_balance(int dim, int L, int64_t n, const int32_t* anchors,
                                const int32_t* levels, int64_t* n_out) {
  if (dim != 2 && dim != 3) {
    fail(AMR_EINVAL, "dimension must be 2 or 3");
    return nullptr;
  }
  if (L < 0 || L > 30 || dim * L > 58) {  // pack_key keeps dim*L code bits above 5 level bits
    fail(AMR_EINVAL, "max_depth too large for 64-bit Morton keys");
    return nullptr;
  }
  const int32_t top = 1 << L;
  std::unordered_set<uint64_t> leafset;
  leafset.reserve((size_t)(n * 4 + 16));
  std::vector<std::pair<int, uint64_t>> init(n);
  for (int64_t i = 0; i < n; ++i) {
    uint64_t k = pack_key(morton_code(anchors + i * dim, dim, L), levels[i]);
    leafset.insert(k);
    init[i] = {-levels[i], k};
  }
  std::stable_sort(init.begin(), init.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  std::deque<uint64_t> work;
  for (auto& p : init) work.push_back(p.second);
  // directions: every non-zero vector in {-1,0,1}^dim (octree.py:274-276)
  std::vector<std::array<int, 3>> dirs;
  for (int a = -1; a <= 1; ++a)
    for (int b = -1; b <= 1; ++b)
      for (int c = (dim == 3 ? -1 : 0); c <= (dim == 3 ? 1 : 0); ++c)
        if (a || b || c) dirs.push_back({a, b, c});
  auto containing = [&](const int32_t* cell, int32_t* anc, int* lvl) -> bool {
    for (int l = L; l >= 0; --l) {
      int sh = L - l;
      int32_t an[3];
      for (int d = 0; d < dim; ++d) an[d] = (cell[d] >> sh) << sh;
      uint64_t k = pack_key(morton_code(an, dim, L), l);
      if (leafset.count(k)) {
        for (int d = 0; d < dim; ++d) anc[d] = an[d];
        *lvl = l;
        return true;
      }
    }
    return false;
  };
  while (!work.empty()) {
    uint64_t key = work.front();
    work.pop_front();
    if (!leafset.count(key)) continue;
    int level = (int)(key & 31);
    int32_t anchor[3] = {0, 0, 0};
    morton_decode(key >> 5, dim, L, anchor);
    int32_t side = 1 << (L - level);
    for (auto& dv : dirs) {
      int32_t cell[3];
      bool ok = true;
      for (int d = 0; d < dim; ++d) {
        int32_t c = dv[d] < 0 ? anchor[d] - 1 : (dv[d] > 0 ? anchor[d] + side : anchor[d]);
        if (c < 0 || c >= top) {
          ok = false;
          break;
        }
        cell[d] = c;
      }
      if (!ok) continue;
      int32_t nb[3];
      int nl;
      bool found = containing(cell, nb, &nl);
      while (found && nl < level - 1) {
        leafset.erase(pack_key(morton_code(nb, dim, L), nl));
        int32_t half = 1 << (L - nl - 1);
        for (int code = 0; code < (1 << dim); ++code) {
          int32_t ch[3];
          for (int d = 0; d < dim; ++d) ch[d] = nb[d] + (((code >> d) & 1) * half);
          uint64_t ck = pack_key(morton_code(ch, dim, L), nl + 1);
          leafset.insert(ck);
          work.push_back(ck);
        }
        found = containing(cell, nb, &nl);
      }
    }
  }
  std::vector<uint64_t> keys(leafset.begin(), leafset.end());
  // Morton order, ancestors first: (code, level)
  std::sort(keys.begin(), keys.end(), [](uint64_t a, uint64_t b) {
    uint64_t ca = a >> 5, cb = b >> 5;
    if (ca != cb) return ca < cb;
    return (a & 31) < (b & 31);
  });
  AmrTree* t = new AmrTree();
  t->dim = dim;
  t->L = L;
  t->anchors.resize(keys.size() * dim);
  t->levels.resize(keys.size());
  for (size_t i = 0; i < keys.size(); ++i) {
    int32_t a[3];
    morton_decode(keys[i] >> 5, dim, L, a);
    for (int d = 0; d < dim; ++d) t->anchors[i * dim + d] = a[d];
    t->levels[i] = (int32_t)(keys[i] & 31);
  }
  *n_out = (int64_t)keys.size();
  return t;
}

extern "C" int amr_tree_fetch(const AmrTree* t, int32_t* anchors_out, int32_t* levels_out) {
  if (!t) return fail(AMR_EINVAL, "null tree");
  std::memcpy(anchors_out, t->anchors.data(), t->anchors.size() * sizeof(int32_t));
  std::memcpy(levels_out, t->levels.data(), t->levels.size() * sizeof(int32_t));
  return AMR_OK;
}

extern "C" void amr_tree_free(AmrTree* t) { delete t; }

// ---------------------------------------------------------------------------
// mesh
// ---------------------------------------------------------------------------

struct AmrBlock {
  int32_t anchor[3];
  int32_t root_level, leaf_level, owner;
  int64_t a, b;
};

using Row = std::vector<std::pair<int32_t, double>>;

struct AmrMesh {
  int dim, L, ppo, pad, scale, per_leaf, nthreads;
  int64_t top_nodes, n_leaves, n_nodes = 0, E = 0;
  std::vector<int32_t> anchor;  // n*3
  std::vector<int32_t> level, owner;
  std::vector<uint64_t> mcodes;  // Morton-sorted leaf codes
  std::vector<int32_t> mperm;    // -> leaf index
  std::vector<int32_t> leaf_gids;
  std::vector<int64_t> starts;
  std::vector<int32_t> table;
  std::vector<int64_t> iptr{0};
  std::vector<int32_t> igid;
  std::vector<double> iw;
  std::unordered_map<int64_t, int32_t> row_of_code;  // rows added after the build (API gathers)
  std::vector<int64_t> hang_codes;                    // sorted codes of the build's rows (row id = index)
  std::unordered_map<int64_t, Row> memo;
  std::vector<AmrBlock> blocks;

  int64_t encode(const int64_t* p) const {
    int64_t m = top_nodes + 1, c = p[0];
    for (int d = 1; d < dim; ++d) c = c * m + p[d];
    return c;
  }
  int64_t spacing(int lvl) const { return (int64_t)1 << (L - lvl); }

  int32_t find_leaf(const int32_t* cell) const {
    uint64_t m = morton_code(cell, dim, L);
    auto it = std::upper_bound(mcodes.begin(), mcodes.end(), m);
    return mperm[(it - mcodes.begin()) - 1];
  }

  // leaves whose closed box contains lattice point p, sorted ascending
  // (mesh.py:293-314)
  int containing(const int64_t* p, int32_t* out) const {
    int n = 0;
    for (int sig = 0; sig < (1 << dim); ++sig) {
      int32_t cell[3];
      bool ok = true;
      for (int d = 0; d < dim; ++d) {
        int64_t q = ((sig >> d) & 1) ? p[d] : p[d] - 1;
        if (q < 0 || q >= top_nodes) {
          ok = false;
          break;
        }
        cell[d] = (int32_t)(q / scale);
      }
      if (!ok) continue;
      int32_t j = find_leaf(cell);
      bool dup = false;
      for (int k = 0; k < n; ++k) dup |= (out[k] == j);
      if (!dup) out[n++] = j;
    }
    std::sort(out, out + n);
    return n;
  }

  int local_index(int32_t leaf, const int64_t* p) const {
    int64_t s = spacing(level[leaf]);
    int idx = 0;
    for (int d = 0; d < dim; ++d) idx = idx * ppo + (int)((p[d] - (int64_t)anchor[leaf * 3 + d] * scale) / s);
    return idx;
  }
  bool on_lattice(int32_t leaf, const int64_t* p) const {
    int64_t s = spacing(level[leaf]);
    for (int d = 0; d < dim; ++d)
      if ((p[d] - (int64_t)anchor[leaf * 3 + d] * scale) % s != 0) return false;
    return true;
  }
  // owner leaf of a real node, -1 if p is not a real node
  int32_t real_owner(const int64_t* p) const {
    int32_t c[8];
    int n = containing(p, c);
    if (n == 0) return -1;
    for (int k = 0; k < n; ++k)
      if (!on_lattice(c[k], p)) return -1;
    return c[0];
  }
  int32_t gid_of(const int64_t* p) const {
    int32_t o = real_owner(p);
    if (o < 0) return -1;
    return leaf_gids[(int64_t)o * per_leaf + local_index(o, p)];
  }

  // _lagrange_weights (mesh.py:138-150)
  void lagrange(double xi, int n, int* w0_out, double* ws, int* npts_out) const {
    int npts = std::min(4, n);
    int w0 = (int)std::floor(xi) - 1;
    w0 = std::max(0, std::min(w0, n - npts));
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

  // _point_weights (mesh.py:316-351): insertion-ordered sparse row.  `memo`
  // only caches (any memo gives the same rows), so threads may use their own.
  const Row& point_weights(const int64_t* p, int* err) { return point_weights_m(p, memo, err); }

  const Row& point_weights_m(const int64_t* p, std::unordered_map<int64_t, Row>& memo, int* err) const {
    int64_t code = encode(p);
    auto hit = memo.find(code);
    if (hit != memo.end()) return hit->second;
    int32_t g = gid_of(p);
    if (g >= 0) {
      Row r{{g, 1.0}};
      return memo.emplace(code, std::move(r)).first->second;
    }
    int32_t c[8];
    int n = containing(p, c);
    if (n == 0) {
      *err = 1;
      static Row empty;
      return empty;
    }
    int lvl = 1 << 30;
    for (int k = 0; k < n; ++k) lvl = std::min(lvl, level[c[k]]);
    int32_t leaf = -1;
    for (int k = 0; k < n; ++k)
      if (level[c[k]] == lvl) {
        leaf = c[k];
        break;
      }
    int64_t s = spacing(level[leaf]);
    int64_t org[3];
    int w0[3], np[3];
    double ws[3][4];
    for (int d = 0; d < dim; ++d) {
      org[d] = (int64_t)anchor[leaf * 3 + d] * scale;
      double xi = (double)(p[d] - org[d]) / (double)s;
      lagrange(xi, ppo, &w0[d], ws[d], &np[d]);
    }
    Row acc;
    int total = 1;
    for (int d = 0; d < dim; ++d) total *= np[d];
    for (int combo = 0; combo < total; ++combo) {
      int cidx[3];
      int rem = combo;
      for (int d = dim - 1; d >= 0; --d) {
        cidx[d] = rem % np[d];
        rem /= np[d];
      }
      double w = 1.0;
      int64_t q[3];
      for (int d = 0; d < dim; ++d) {
        w *= ws[d][cidx[d]];
        q[d] = org[d] + (int64_t)(w0[d] + cidx[d]) * s;
      }
      if (w == 0.0) continue;
      Row sub = point_weights_m(q, memo, err);  // copy: memo may rehash
      if (*err) break;
      for (auto& gw : sub) {
        bool found = false;
        for (auto& a : acc)
          if (a.first == gw.first) {
            a.second = a.second + w * gw.second;
            found = true;
            break;
          }
        if (!found) acc.push_back({gw.first, 0.0 + w * gw.second});
      }
    }
    return memo.emplace(code, std::move(acc)).first->second;
  }

  int32_t row_for(const int64_t* p, int* err) {
    int64_t code = encode(p);
    auto hb = std::lower_bound(hang_codes.begin(), hang_codes.end(), code);
    if (hb != hang_codes.end() && *hb == code) return (int32_t)(hb - hang_codes.begin());
    auto it = row_of_code.find(code);
    if (it != row_of_code.end()) return it->second;
    Row r = point_weights(p, err);
    if (*err) return -1;
    std::sort(r.begin(), r.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    int32_t id = (int32_t)(iptr.size() - 1);
    for (auto& gw : r) {
      igid.push_back(gw.first);
      iw.push_back(gw.second);
    }
    iptr.push_back((int64_t)igid.size());
    row_of_code.emplace(code, id);
    return id;
  }
};

namespace {

// cross-region enumeration shared with the kernel: interior ppo^dim (C order)
// then, per axis, the 2*pad layers below and above (pad*2 layers), each a
// ppo^(dim-1) C-ordered cross-section over the remaining axes.
void cross_entry_local(int e, int dim, int ppo, int pad, int* loc /* padded coords */) {
  int NI = ipow(ppo, dim), NF = ipow(ppo, dim - 1);
  if (e < NI) {
    int r = e;
    for (int d = dim - 1; d >= 0; --d) {
      loc[d] = pad + r % ppo;
      r /= ppo;
    }
    return;
  }
  int r = e - NI;
  int axis = r / (2 * pad * NF);
  r %= 2 * pad * NF;
  int layer = r / NF;  // 0..2pad-1
  int within = r % NF;
  int lp = layer < pad ? layer : ppo + layer;  // 0,1 | ppo+2, ppo+3 (pad=2)
  for (int d = dim - 1; d >= 0; --d) {
    if (d == axis) continue;
    loc[d] = pad + within % ppo;
    within /= ppo;
  }
  loc[axis] = lp;
}

void decompose(AmrMesh* m, const int32_t* node, int nlevel, int64_t a, int64_t b) {
  int lvl = m->level[a];
  bool uniform = true;
  for (int64_t i = a; i < b && uniform; ++i) uniform = (m->level[i] == lvl);
  bool single = m->owner[a] == m->owner[b - 1];
  if (uniform && single) {
    AmrBlock blk;
    for (int d = 0; d < 3; ++d) blk.anchor[d] = d < m->dim ? node[d] : 0;
    blk.root_level = nlevel;
    blk.leaf_level = lvl;
    blk.owner = m->owner[a];
    blk.a = a;
    blk.b = b;
    m->blocks.push_back(blk);
    return;
  }
  // children in SFC order = maximal runs of leaves sharing the child digit
  int sh = m->L - (nlevel + 1);
  int64_t pos = a;
  while (pos < b) {
    int32_t ch[3];
    for (int d = 0; d < m->dim; ++d) ch[d] = (m->anchor[pos * 3 + d] >> sh) << sh;
    int64_t end = pos;
    while (end < b) {
      bool inside = true;
      for (int d = 0; d < m->dim; ++d) inside &= ((m->anchor[end * 3 + d] >> sh) << sh) == ch[d];
      if (!inside) break;
      ++end;
    }
    decompose(m, ch, nlevel + 1, pos, end);
    pos = end;
  }
}

}  // namespace

extern "C" int64_t amr_tile_entries(int dim, int ppo) {
  return (int64_t)ipow(ppo, dim) + 2 * dim * 2 * (int64_t)ipow(ppo, dim - 1);
}

extern "C" AmrMesh* amr_mesh_build(int dim, int L, int ppo, int pad, int64_t n_leaves,
                                   const int32_t* anchors, const int32_t* levels,
                                   const int32_t* owners, int n_threads) {
  if (dim != 2 && dim != 3) {
    fail(AMR_EINVAL, "dimension must be 2 or 3");
    return nullptr;
  }
  if (ppo < 5 || ppo % 2 == 0) {
    fail(AMR_EINVAL, "points_per_octant must be odd and >= 5");
    return nullptr;
  }
  if (pad != 2) {
    fail(AMR_EINVAL, "the B200 stage kernel is built for pad=2 (the 5-point stencil reach)");
    return nullptr;
  }
  AmrMesh* m = new AmrMesh();
  m->dim = dim;
  m->L = L;
  m->ppo = ppo;
  m->pad = pad;
  m->scale = ppo - 1;
  m->top_nodes = (int64_t)m->scale << L;
  m->n_leaves = n_leaves;
  m->per_leaf = ipow(ppo, dim);
  m->nthreads = n_threads > 0 ? n_threads : omp_get_max_threads();
  {
    double mm = (double)(m->top_nodes + 1);
    if (std::pow(mm, dim) >= 4.611686018427388e18) {
      fail(AMR_EINVAL, "max_depth too large for the node lattice encoding");
      delete m;
      return nullptr;
    }
  }
  m->anchor.assign(n_leaves * 3, 0);
  m->level.resize(n_leaves);
  m->owner.assign(n_leaves, 0);
  for (int64_t i = 0; i < n_leaves; ++i) {
    for (int d = 0; d < dim; ++d) m->anchor[i * 3 + d] = anchors[i * dim + d];
    m->level[i] = levels[i];
    if (owners) m->owner[i] = owners[i];
  }
  // Morton lookup index
  {
    std::vector<std::pair<uint64_t, int32_t>> kv(n_leaves);
    for (int64_t i = 0; i < n_leaves; ++i) kv[i] = {morton_code(&m->anchor[i * 3], dim, L), (int32_t)i};
    std::sort(kv.begin(), kv.end());
    m->mcodes.resize(n_leaves);
    m->mperm.resize(n_leaves);
    for (int64_t i = 0; i < n_leaves; ++i) {
      m->mcodes[i] = kv[i].first;
      m->mperm[i] = kv[i].second;
      if (i && kv[i].first == kv[i - 1].first) {
        fail(AMR_EINVAL, "duplicate leaf anchors: tree is not a valid linear octree");
        delete m;
        return nullptr;
      }
    }
  }
  const bool timing = std::getenv("AMR_MESH_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto tick = [&](const char* what) {
    if (!timing) return;
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[amr_mesh_build] %-14s %8.3f s\n", what,
                 std::chrono::duration<double>(now - t_last).count());
    t_last = now;
  };
  const int P = m->per_leaf;
  m->leaf_gids.assign((size_t)n_leaves * P, -1);
  std::vector<int64_t> counts(n_leaves, 0);
  // pass 1: ownership status per leaf point (1 owned, 0 real not owned, -1 hanging)
  std::vector<int8_t> status((size_t)n_leaves * P);
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) num_threads(m->nthreads) reduction(+ : bad)
  for (int64_t i = 0; i < n_leaves; ++i) {
    int64_t s = m->spacing(m->level[i]);
    int64_t cnt = 0;
    for (int k = 0; k < P; ++k) {
      int loc[3];
      int r = k;
      bool interior = true;
      for (int d = dim - 1; d >= 0; --d) {
        loc[d] = r % ppo;
        r /= ppo;
        interior &= (loc[d] > 0 && loc[d] < ppo - 1);
      }
      int8_t st;
      if (interior) {
        st = 1;
      } else {
        int64_t p[3];
        for (int d = 0; d < dim; ++d) p[d] = (int64_t)m->anchor[i * 3 + d] * m->scale + s * loc[d];
        int32_t c[8];
        int n = m->containing(p, c);
        if (n == 0) {
          ++bad;
          st = -1;
        } else {
          bool real = true;
          for (int q = 0; q < n; ++q) real &= m->on_lattice(c[q], p);
          st = !real ? -1 : (c[0] == i ? 1 : 0);
        }
      }
      status[(size_t)i * P + k] = st;
      cnt += (st == 1);
    }
    counts[i] = cnt;
  }
  tick("ownership");
  if (bad) {
    fail(AMR_EINVAL, "leaf point outside every leaf: tree is not complete");
    delete m;
    return nullptr;
  }
  m->starts.assign(n_leaves + 1, 0);
  for (int64_t i = 0; i < n_leaves; ++i) m->starts[i + 1] = m->starts[i] + counts[i];
  m->n_nodes = m->starts[n_leaves];
  if (m->n_nodes >= (int64_t)1 << 31) {
    fail(AMR_EINVAL, "more than 2^31 zip nodes: int32 gids overflow");
    delete m;
    return nullptr;
  }
  // pass 2a: owned gids
#pragma omp parallel for schedule(static) num_threads(m->nthreads)
  for (int64_t i = 0; i < n_leaves; ++i) {
    int32_t g = (int32_t)m->starts[i];
    for (int k = 0; k < P; ++k)
      if (status[(size_t)i * P + k] == 1) m->leaf_gids[(size_t)i * P + k] = g++;
  }
  // pass 2b: shared (real, not owned) points take the owner's gid
#pragma omp parallel for schedule(dynamic, 64) num_threads(m->nthreads)
  for (int64_t i = 0; i < n_leaves; ++i) {
    int64_t s = m->spacing(m->level[i]);
    for (int k = 0; k < P; ++k) {
      if (status[(size_t)i * P + k] != 0) continue;
      int loc[3];
      int r = k;
      for (int d = dim - 1; d >= 0; --d) {
        loc[d] = r % ppo;
        r /= ppo;
      }
      int64_t p[3];
      for (int d = 0; d < dim; ++d) p[d] = (int64_t)m->anchor[i * 3 + d] * m->scale + s * loc[d];
      int32_t o = m->real_owner(p);
      m->leaf_gids[(size_t)i * P + k] = m->leaf_gids[(size_t)o * P + m->local_index(o, p)];
    }
  }
  tick("gids");
  // tile tables over the stencil cross
  const int64_t E = amr_tile_entries(dim, ppo);
  m->E = E;
  m->table.assign((size_t)n_leaves * E, -1);
  std::vector<int> lut((size_t)E * 3);
  for (int e = 0; e < E; ++e) cross_entry_local(e, dim, ppo, pad, &lut[e * 3]);
  int nt = m->nthreads;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> hang(nt);  // (table pos, code)
  std::vector<std::vector<std::array<int64_t, 3>>> hang_pt(nt);
#pragma omp parallel num_threads(nt)
  {
    int tid = omp_get_thread_num();
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = 0; i < n_leaves; ++i) {
      int64_t s = m->spacing(m->level[i]);
      for (int e = 0; e < E; ++e) {
        const int* lp = &lut[e * 3];
        int64_t p[3] = {0, 0, 0};
        bool in_dom = true, in_leaf = true;
        int loc[3];
        for (int d = 0; d < dim; ++d) {
          loc[d] = lp[d] - pad;
          p[d] = (int64_t)m->anchor[i * 3 + d] * m->scale + s * loc[d];
          in_dom &= (p[d] >= 0 && p[d] <= m->top_nodes);
          in_leaf &= (loc[d] >= 0 && loc[d] < ppo);
        }
        int32_t ent;
        if (!in_dom) {
          ent = -1;
        } else if (in_leaf) {
          int idx = 0;
          for (int d = 0; d < dim; ++d) idx = idx * ppo + loc[d];
          ent = m->leaf_gids[(size_t)i * P + idx];
        } else {
          ent = m->gid_of(p);
        }
        if (in_dom && ent < 0) {
          hang[tid].push_back({(int64_t)i * E + e, 0});
          hang_pt[tid].push_back({p[0], p[1], p[2]});
          ent = -2;
        }
        m->table[(size_t)i * E + e] = ent;
      }
    }
  }
  tick("tile tables");
  // unique hanging codes -> rows, computed in parallel with thread-local memos
  std::vector<std::pair<int64_t, std::array<int64_t, 3>>> hc;
  for (int t = 0; t < nt; ++t)
    for (size_t k = 0; k < hang[t].size(); ++k)
      hc.push_back({m->encode(hang_pt[t][k].data()), hang_pt[t][k]});
  std::sort(hc.begin(), hc.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  hc.erase(std::unique(hc.begin(), hc.end(), [](const auto& a, const auto& b) { return a.first == b.first; }),
           hc.end());
  std::vector<Row> rows(hc.size());
  int err = 0;
#pragma omp parallel num_threads(nt) reduction(| : err)
  {
    std::unordered_map<int64_t, Row> memo;
#pragma omp for schedule(dynamic, 256)
    for (int64_t k = 0; k < (int64_t)hc.size(); ++k) {
      int e = 0;
      Row r = m->point_weights_m(hc[k].second.data(), memo, &e);
      if (e) {
        err |= 1;
        continue;
      }
      std::sort(r.begin(), r.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      rows[k] = std::move(r);
    }
  }
  if (err) {
    fail(AMR_ESTATE, "lattice point outside the domain during interpolation");
    delete m;
    return nullptr;
  }
  m->iptr.assign(rows.size() + 1, 0);
  for (size_t k = 0; k < rows.size(); ++k) m->iptr[k + 1] = m->iptr[k] + (int64_t)rows[k].size();
  m->igid.resize(m->iptr.back());
  m->iw.resize(m->iptr.back());
#pragma omp parallel for schedule(static) num_threads(nt)
  for (int64_t k = 0; k < (int64_t)rows.size(); ++k)
    for (size_t j = 0; j < rows[k].size(); ++j) {
      m->igid[m->iptr[k] + j] = rows[k][j].first;
      m->iw[m->iptr[k] + j] = rows[k][j].second;
    }
  m->hang_codes.resize(hc.size());
  for (size_t k = 0; k < hc.size(); ++k) m->hang_codes[k] = hc[k].first;
#pragma omp parallel for schedule(static, 1) num_threads(nt)
  for (int t = 0; t < nt; ++t)
    for (size_t k = 0; k < hang[t].size(); ++k) {
      const int64_t code = m->encode(hang_pt[t][k].data());
      const auto it = std::lower_bound(hc.begin(), hc.end(), code,
                                       [](const auto& a, int64_t c) { return a.first < c; });
      m->table[hang[t][k].first] = -2 - (int32_t)(it - hc.begin());
    }
  tick("interp rows");
  int32_t root[3] = {0, 0, 0};
  if (n_leaves > 0) decompose(m, root, 0, 0, n_leaves);
  tick("blocks");
  return m;
}

// A mesh handle around tables built elsewhere (the device builder,
// amr_devmesh.cu): the registry, tile table and interpolation rows are taken
// as given; the Morton index, blocks and the lazy API gathers work as after
// amr_mesh_build.
extern "C" AmrMesh* amr_mesh_from_tables(int dim, int L, int ppo, int pad, int64_t n_leaves,
                                         const int32_t* anchors, const int32_t* levels, const int32_t* owners,
                                         const int64_t* starts, const int32_t* leaf_gids, const int32_t* table,
                                         int64_t n_rows, const int64_t* hang_codes, const int64_t* iptr,
                                         const int32_t* igid, const double* iw) {
  if ((dim != 2 && dim != 3) || ppo < 5 || ppo % 2 == 0 || pad != 2) {
    fail(AMR_EINVAL, "amr_mesh_from_tables: dim 2/3, odd ppo >= 5, pad 2");
    return nullptr;
  }
  AmrMesh* m = new AmrMesh();
  m->dim = dim;
  m->L = L;
  m->ppo = ppo;
  m->pad = pad;
  m->scale = ppo - 1;
  m->top_nodes = (int64_t)m->scale << L;
  m->n_leaves = n_leaves;
  m->per_leaf = ipow(ppo, dim);
  m->nthreads = omp_get_max_threads();
  m->anchor.assign(n_leaves * 3, 0);
  m->level.assign(levels, levels + n_leaves);
  m->owner.assign(n_leaves, 0);
  for (int64_t i = 0; i < n_leaves; ++i) {
    for (int d = 0; d < dim; ++d) m->anchor[i * 3 + d] = anchors[i * dim + d];
    if (owners) m->owner[i] = owners[i];
  }
  std::vector<std::pair<uint64_t, int32_t>> kv(n_leaves);
  for (int64_t i = 0; i < n_leaves; ++i) kv[i] = {morton_code(&m->anchor[i * 3], dim, L), (int32_t)i};
  std::sort(kv.begin(), kv.end());
  m->mcodes.resize(n_leaves);
  m->mperm.resize(n_leaves);
  for (int64_t i = 0; i < n_leaves; ++i) {
    m->mcodes[i] = kv[i].first;
    m->mperm[i] = kv[i].second;
  }
  m->starts.assign(starts, starts + n_leaves + 1);
  m->n_nodes = m->starts[n_leaves];
  m->E = amr_tile_entries(dim, ppo);
  if (leaf_gids && table) {  // NULL: a light handle (blocks and leaf slices only)
    m->leaf_gids.assign(leaf_gids, leaf_gids + (size_t)n_leaves * m->per_leaf);
    m->table.assign(table, table + (size_t)n_leaves * m->E);
    m->hang_codes.assign(hang_codes, hang_codes + n_rows);
    m->iptr.assign(iptr, iptr + n_rows + 1);
    m->igid.assign(igid, igid + m->iptr.back());
    m->iw.assign(iw, iw + m->iptr.back());
  }
  int32_t root[3] = {0, 0, 0};
  if (n_leaves > 0) decompose(m, root, 0, 0, n_leaves);
  return m;
}

extern "C" void amr_mesh_free(AmrMesh* m) { delete m; }

// read-only views for the program builder (amr_programs.cpp)
extern "C" int amr_mesh_view(const AmrMesh* m, int* dim, int* L, int* ppo, int64_t* n_leaves, int64_t* E,
                             const int32_t** table, const int64_t** starts, const int32_t** anchor,
                             const int32_t** level, const int64_t** iptr, const int32_t** igid, const double** iw) {
  if (!m || m->table.empty()) return AMR_ESTATE;
  *dim = m->dim;
  *L = m->L;
  *ppo = m->ppo;
  *n_leaves = m->n_leaves;
  *E = m->E;
  *table = m->table.data();
  *starts = m->starts.data();
  *anchor = m->anchor.data();
  *level = m->level.data();
  *iptr = m->iptr.data();
  *igid = m->igid.data();
  *iw = m->iw.data();
  return AMR_OK;
}
extern "C" int64_t amr_mesh_n_nodes(const AmrMesh* m) { return m ? m->n_nodes : -1; }

extern "C" int amr_mesh_leaf_starts(const AmrMesh* m, int64_t* starts) {
  std::memcpy(starts, m->starts.data(), m->starts.size() * sizeof(int64_t));
  return AMR_OK;
}

extern "C" int amr_mesh_leaf_gids(const AmrMesh* m, int32_t* gids) {
  std::memcpy(gids, m->leaf_gids.data(), m->leaf_gids.size() * sizeof(int32_t));
  return AMR_OK;
}

extern "C" int amr_mesh_node_coords(const AmrMesh* m, int32_t* coords) {
  const int P = m->per_leaf, dim = m->dim, ppo = m->ppo;
#pragma omp parallel for schedule(static) num_threads(m->nthreads)
  for (int64_t i = 0; i < m->n_leaves; ++i) {
    int64_t s = m->spacing(m->level[i]);
    int64_t g0 = m->starts[i];
    for (int k = 0; k < P; ++k) {
      int32_t g = m->leaf_gids[(size_t)i * P + k];
      if (g < g0 || g >= m->starts[i + 1]) continue;
      int r = k;
      int loc[3];
      for (int d = dim - 1; d >= 0; --d) {
        loc[d] = r % ppo;
        r /= ppo;
      }
      for (int d = 0; d < dim; ++d)
        coords[(size_t)g * dim + d] = (int32_t)((int64_t)m->anchor[i * 3 + d] * m->scale + s * loc[d]);
    }
  }
  return AMR_OK;
}

extern "C" int amr_mesh_tile_table(const AmrMesh* m, int32_t* table) {
  std::memcpy(table, m->table.data(), m->table.size() * sizeof(int32_t));
  return AMR_OK;
}

extern "C" int64_t amr_mesh_interp_rows(const AmrMesh* m) { return (int64_t)m->iptr.size() - 1; }
extern "C" int64_t amr_mesh_interp_nnz(const AmrMesh* m) { return (int64_t)m->igid.size(); }

extern "C" int amr_mesh_interp_csr(const AmrMesh* m, int64_t* row_ptr, int32_t* gid, double* w) {
  std::memcpy(row_ptr, m->iptr.data(), m->iptr.size() * sizeof(int64_t));
  std::memcpy(gid, m->igid.data(), m->igid.size() * sizeof(int32_t));
  std::memcpy(w, m->iw.data(), m->iw.size() * sizeof(double));
  return AMR_OK;
}

extern "C" int64_t amr_mesh_n_blocks(const AmrMesh* m) { return (int64_t)m->blocks.size(); }

extern "C" int amr_mesh_blocks(const AmrMesh* m, int32_t* root_anchor, int32_t* root_level,
                               int32_t* leaf_level, int64_t* leaf_range, int32_t* owner) {
  for (size_t i = 0; i < m->blocks.size(); ++i) {
    const AmrBlock& b = m->blocks[i];
    for (int d = 0; d < m->dim; ++d) root_anchor[i * m->dim + d] = b.anchor[d];
    root_level[i] = b.root_level;
    leaf_level[i] = b.leaf_level;
    leaf_range[2 * i] = b.a;
    leaf_range[2 * i + 1] = b.b;
    owner[i] = b.owner;
  }
  return AMR_OK;
}

extern "C" int amr_mesh_block_gather(AmrMesh* m, int64_t block, int64_t* rows, int64_t* nnz,
                                     int64_t* row_ptr, int64_t* col, double* val) {
  if (block < 0 || block >= (int64_t)m->blocks.size()) return fail(AMR_EINVAL, "block index out of range");
  const AmrBlock& b = m->blocks[block];
  const int dim = m->dim;
  int64_t s = m->spacing(b.leaf_level);
  int64_t interior = (int64_t)(m->ppo - 1) * ((int64_t)1 << (b.leaf_level - b.root_level)) + 1;
  int64_t n = interior + 2 * m->pad;
  int64_t total = 1;
  for (int d = 0; d < dim; ++d) total *= n;
  int64_t org[3];
  for (int d = 0; d < dim; ++d) org[d] = (int64_t)b.anchor[d] * m->scale - m->pad * s;
  int64_t cnt = 0;
  int err = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (int64_t r = 0; r < total; ++r) {
    int64_t p[3];
    int64_t rem = r;
    bool in_dom = true;
    for (int d = dim - 1; d >= 0; --d) {
      p[d] = org[d] + s * (rem % n);
      rem /= n;
      in_dom &= (p[d] >= 0 && p[d] <= m->top_nodes);
    }
    if (in_dom) {
      int32_t g = m->gid_of(p);
      if (g >= 0) {
        if (col) {
          col[cnt] = g;
          val[cnt] = 1.0;
        }
        ++cnt;
      } else {
        int32_t row = m->row_for(p, &err);
        if (err) return fail(AMR_ESTATE, "lattice point outside the domain during interpolation");
        for (int64_t k = m->iptr[row]; k < m->iptr[row + 1]; ++k) {
          if (col) {
            col[cnt] = m->igid[k];
            val[cnt] = m->iw[k];
          }
          ++cnt;
        }
      }
    }
    if (row_ptr) row_ptr[r + 1] = cnt;
  }
  *rows = total;
  *nnz = cnt;
  return AMR_OK;
}

