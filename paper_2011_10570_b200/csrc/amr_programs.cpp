// amr_programs.cpp — native (C++/OpenMP) builder of the stage kernel's
// per-tile programs.  It produces byte for byte what
// paper_2011_10570_b200/tileprog.py (the readable specification, tested
// against this file in tests/test_programs_native.py) produces, straight from
// the mesh's leaf tables, one tile per OpenMP iteration:
//   * the owned cross of the tile (owned nodes +-1, +-2 along each axis, the
//     biased rows' windows at physical faces);
//   * hanging rows of the cross (longest first) with their taps padded to
//     quads, their unique source nodes ("slots", ascending gid);
//   * LTS interface pairs (source node, reader cadence) where the source
//     steps with another cadence (unique over all tiles, finest reader first);
//   * copy runs along the box rows, bucketed by length, and the head/tail
//     byte layout of tileprog.py.
// Setup code (once per Engine), not the per-step hot path.
#include "../../include/amr_b200.h"

#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

extern "C" void amr_set_error_internal(const char* msg);

// views of the mesh that the builder needs (amr_mesh.cpp)
extern "C" int amr_mesh_view(const AmrMesh* m, int* dim, int* L, int* ppo, int64_t* n_leaves, int64_t* E,
                             const int32_t** table, const int64_t** starts, const int32_t** anchor,
                             const int32_t** level, const int64_t** iptr, const int32_t** igid, const double** iw);

namespace {

constexpr int HDR_WORDS = 16;
constexpr int MAX_BASES = 63;
constexpr int RUN_MAX = 8;

inline int64_t r16(int64_t b) { return (b + 15) / 16 * 16; }

struct TileOut {
  std::vector<uint32_t> head;  // header + bases + runs + slots (uint32 words)
  std::vector<uint16_t> tail;  // rows (as pairs of uint16) + taps
  int64_t head_bytes = 0, tail_bytes = 0;
};

// cross enumeration of amr_mesh.cpp / tileprog.cross_cells: padded local coordinates
void cross_loc(int e, int dim, int ppo, int* loc) {
  const int pad = 2;
  int NI = 1, NF = 1;
  for (int d = 0; d < dim; ++d) NI *= ppo;
  for (int d = 0; d < dim - 1; ++d) NF *= ppo;
  if (e < NI) {
    int r = e;
    for (int d = dim - 1; d >= 0; --d) {
      loc[d] = pad + r % ppo;
      r /= ppo;
    }
    return;
  }
  int r = e - NI;
  const int axis = r / (2 * pad * NF);
  r %= 2 * pad * NF;
  const int layer = r / NF;
  int within = r % NF;
  for (int d = dim - 1; d >= 0; --d) {
    if (d == axis) continue;
    loc[d] = pad + within % ppo;
    within /= ppo;
  }
  loc[axis] = layer < pad ? layer : ppo + layer;
}

}  // namespace

struct AmrProg {
  int64_t n_tiles = 0, max_head = 0, max_tail = 0, max_slots = 0, n_rows = 0, n_cells = 0;
  std::vector<uint8_t> heads;
  std::vector<uint16_t> tail;
  std::vector<int32_t> if_gid, if_cad;
  std::vector<double> wtab;
};

extern "C" AmrProg* amr_programs_build(const AmrMesh* mesh, int64_t n_tiles, const int32_t* tiles,
                                       const int32_t* leaf_cad, int lts, int row_stride, int n_threads) {
  int dim, L, ppo;
  int64_t n_leaves, E;
  const int32_t *table, *anchor, *level, *igid;
  const int64_t *starts, *iptr;
  const double* iw;
  if (amr_mesh_view(mesh, &dim, &L, &ppo, &n_leaves, &E, &table, &starts, &anchor, &level, &iptr, &igid, &iw)) {
    amr_set_error_internal("amr_programs_build: mesh has no tile tables");
    return nullptr;
  }
  const int nth = n_threads > 0 ? n_threads : omp_get_max_threads();
  const int NP = ppo + 4;
  const int RS = row_stride > NP ? row_stride : NP;
  int bs[3];  // box strides
  if (dim == 3) {
    bs[0] = NP * RS;
    bs[1] = RS;
    bs[2] = 1;
  } else {
    bs[0] = RS;
    bs[1] = 1;
  }
  const int box_n = (dim == 3 ? NP : 1) * NP * RS;
  int NI = 1;
  for (int d = 0; d < dim; ++d) NI *= ppo;
  std::vector<int32_t> cell(E), cell2e(box_n, -1);
  std::vector<int16_t> pos(NI * 3);
  for (int e = 0; e < E; ++e) {
    int loc[3] = {0, 0, 0};
    cross_loc(e, dim, ppo, loc);
    int c = 0;
    for (int d = 0; d < dim; ++d) c += loc[d] * bs[d];
    cell[e] = c;
    cell2e[c] = e;
    if (e < NI)
      for (int d = 0; d < dim; ++d) pos[e * 3 + d] = (int16_t)(loc[d] - 2);
  }
  auto node_leaf = [&](int64_t g) {  // owner leaf of zip node g
    return (int64_t)(std::upper_bound(starts, starts + n_leaves + 1, g) - starts) - 1;
  };
  std::vector<uint8_t> ncad_leaf(n_leaves);
  for (int64_t i = 0; i < n_leaves; ++i) ncad_leaf[i] = (uint8_t)leaf_cad[i];

  // ---- pass 1 (per tile): needed entries; global sets of pair keys and weights
  std::vector<std::vector<uint64_t>> keys_t(nth);
  std::vector<std::vector<double>> w_t(nth);
  std::vector<std::vector<uint8_t>> need_all(n_tiles);
  int err = 0;
  // AMR_MAX_BASES lowers the source-group limit (tests of the refusal path)
  const char* mb_env = std::getenv("AMR_MAX_BASES");
  const int max_bases = mb_env ? std::min(MAX_BASES, std::max(1, std::atoi(mb_env))) : MAX_BASES;
#pragma omp parallel num_threads(nth) reduction(| : err)
  {
    const int tid = omp_get_thread_num();
    auto& keys = keys_t[tid];
    auto& ws = w_t[tid];
#pragma omp for schedule(dynamic, 64)
    for (int64_t t = 0; t < n_tiles; ++t) {
      const int64_t leaf = tiles[t];
      const int32_t* row = table + leaf * E;
      const int64_t g0 = starts[leaf], g1 = starts[leaf + 1];
      int faces = 0;
      const int64_t side = (int64_t)1 << (L - level[leaf]);
      for (int d = 0; d < dim; ++d) {
        if (anchor[leaf * 3 + d] == 0) faces |= 1 << (2 * d);
        if (anchor[leaf * 3 + d] + side == ((int64_t)1 << L)) faces |= 2 << (2 * d);
      }
      std::vector<uint8_t>& need = need_all[t];
      need.assign(E, 0);
      for (int e = 0; e < NI; ++e) {
        if (!(row[e] >= g0 && row[e] < g1)) continue;
        need[e] = 1;
        for (int d = 0; d < dim; ++d) {
          for (int o = -2; o <= 2; ++o) need[cell2e[cell[e] + o * bs[d]]] = 1;
          const int p = pos[e * 3 + d];
          const bool lo = (faces >> (2 * d)) & 1, hi = (faces >> (2 * d + 1)) & 1;
          for (int o = -5; o <= 5; ++o) {
            if (p + o < 0 || p + o >= ppo) continue;
            if ((lo && p <= 1) || (hi && p >= ppo - 2)) need[cell2e[cell[e] + o * bs[d]]] = 1;
          }
        }
      }
      const int tc = leaf_cad[leaf];
      for (int64_t e = 0; e < E; ++e) {
        if (!need[e]) continue;
        const int32_t v = row[e];
        if (v >= 0) {
          if (lts && ncad_leaf[node_leaf(v)] != tc) keys.push_back(((uint64_t)(31 - tc) << 32) | (uint32_t)v);
        } else if (v <= -2) {
          const int64_t r = -(int64_t)v - 2;
          for (int64_t k = iptr[r]; k < iptr[r + 1]; ++k) {
            ws.push_back(iw[k]);
            if (lts && ncad_leaf[node_leaf(igid[k])] != tc)
              keys.push_back(((uint64_t)(31 - tc) << 32) | (uint32_t)igid[k]);
          }
        }
      }
    }
  }
  if (err) return nullptr;
  // global unique pair keys (finest reader first, then gid) and weights
  std::vector<uint64_t> ukeys;
  for (auto& v : keys_t) ukeys.insert(ukeys.end(), v.begin(), v.end());
  std::sort(ukeys.begin(), ukeys.end());
  ukeys.erase(std::unique(ukeys.begin(), ukeys.end()), ukeys.end());
  std::vector<double> wtab{0.0};
  for (auto& v : w_t) wtab.insert(wtab.end(), v.begin(), v.end());
  std::sort(wtab.begin(), wtab.end());
  wtab.erase(std::unique(wtab.begin(), wtab.end()), wtab.end());  // == comparison, like np.unique
  if (wtab.size() > 64) {
    amr_set_error_internal(("programs: " + std::to_string(wtab.size()) + " distinct interpolation weights (> 64)").c_str());
    return nullptr;
  }
  const int64_t n_iface = (int64_t)ukeys.size();
  auto* P = new AmrProg();
  P->n_tiles = n_tiles;
  P->wtab = wtab;
  P->if_gid.resize(n_iface);
  P->if_cad.resize(n_iface);
  std::vector<int64_t> grp_start(n_iface);
  for (int64_t i = 0; i < n_iface; ++i) {
    const int64_t g = (int64_t)(ukeys[i] & 0xFFFFFFFFu);
    const int rc = 31 - (int)(ukeys[i] >> 32);
    P->if_gid[i] = (int32_t)g;
    P->if_cad[i] = rc | ((int)ncad_leaf[node_leaf(g)] << 8);
    const bool nw = i == 0 || (ukeys[i] >> 32) != (ukeys[i - 1] >> 32) ||
                    node_leaf(g) != node_leaf((int64_t)(ukeys[i - 1] & 0xFFFFFFFFu));
    grp_start[i] = nw ? i : grp_start[i - 1];
  }
  auto widx_of = [&](double w) { return (int)(std::lower_bound(wtab.begin(), wtab.end(), w) - wtab.begin()); };
  const int zero_w = widx_of(0.0);

  // ---- pass 2 (per tile): encode
  std::vector<TileOut> outs(n_tiles);
  std::vector<int64_t> n_rows_t(n_tiles), n_cells_t(n_tiles), n_slots_t(n_tiles);
#pragma omp parallel for schedule(dynamic, 64) num_threads(nth) reduction(| : err)
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int64_t leaf = tiles[t];
    const int32_t* row = table + leaf * E;
    const int64_t g0 = starts[leaf], g1 = starts[leaf + 1];
    const int tc = leaf_cad[leaf];
    std::vector<uint8_t>& need = need_all[t];
    int faces = 0;
    const int64_t side = (int64_t)1 << (L - level[leaf]);
    for (int d = 0; d < dim; ++d) {
      if (anchor[leaf * 3 + d] == 0) faces |= 1 << (2 * d);
      if (anchor[leaf * 3 + d] + side == ((int64_t)1 << L)) faces |= 2 << (2 * d);
    }
    // a source of the tile: (base value, offset)
    auto src_of_gid = [&](int64_t g, int64_t& base, int64_t& off) {
      if (lts && ncad_leaf[node_leaf(g)] != tc) {
        const uint64_t key = ((uint64_t)(31 - tc) << 32) | (uint32_t)g;
        const int64_t p = std::lower_bound(ukeys.begin(), ukeys.end(), key) - ukeys.begin();
        base = -grp_start[p] - 1;
        off = p - grp_start[p];
      } else {
        const int64_t lf = node_leaf(g);
        base = starts[lf];
        off = g - base;
      }
    };
    // hanging rows: (count desc, entry asc)
    std::vector<std::pair<int64_t, int64_t>> hr;  // (-count, e)
    int64_t ncells = 0;
    for (int64_t e = 0; e < E; ++e) {
      if (!need[e]) continue;
      ++ncells;
      if (row[e] <= -2) {
        const int64_t r = -(int64_t)row[e] - 2;
        hr.push_back({-(iptr[r + 1] - iptr[r]), e});
      }
    }
    std::sort(hr.begin(), hr.end());
    // slots: unique tap gids, ascending
    std::vector<int64_t> slots;
    for (auto& x : hr) {
      const int64_t r = -(int64_t)row[x.second] - 2;
      for (int64_t k = iptr[r]; k < iptr[r + 1]; ++k) slots.push_back(igid[k]);
    }
    std::sort(slots.begin(), slots.end());
    slots.erase(std::unique(slots.begin(), slots.end()), slots.end());
    const int64_t nslot = (int64_t)slots.size();
    if (nslot >= 1023) {
      err |= 1;
      continue;
    }
    // sources: copies (needed, v >= 0) and slots -> (base, off); per-tile base table
    struct Src {
      int64_t cell, base, off;
    };
    std::vector<Src> copies;
    for (int64_t e = 0; e < E; ++e) {
      if (!need[e] || row[e] < 0) continue;
      Src s;
      s.cell = cell[e];
      src_of_gid(row[e], s.base, s.off);
      copies.push_back(s);
    }
    std::vector<std::pair<int64_t, int64_t>> sslot(nslot);  // (base, off)
    for (int64_t k = 0; k < nslot; ++k) src_of_gid(slots[k], sslot[k].first, sslot[k].second);
    std::vector<int64_t> bases;
    for (auto& s : copies) bases.push_back(s.base);
    for (auto& s : sslot) bases.push_back(s.first);
    std::sort(bases.begin(), bases.end());
    bases.erase(std::unique(bases.begin(), bases.end()), bases.end());
    if ((int64_t)bases.size() > max_bases) {
      err |= 2;
      continue;
    }
    auto bidx = [&](int64_t b) { return (int64_t)(std::lower_bound(bases.begin(), bases.end(), b) - bases.begin()); };
    bool bad = false;
    for (auto& s : copies) bad |= s.off >= 1024;
    for (auto& s : sslot) bad |= s.second >= 1024;
    if (bad) {
      err |= 4;
      continue;
    }
    // runs
    std::sort(copies.begin(), copies.end(), [](const Src& a, const Src& b) { return a.cell < b.cell; });
    struct Run {
      int64_t cell, len, code, bucket;
    };
    std::vector<Run> runs;
    for (size_t i = 0; i < copies.size();) {
      const int64_t code0 = (bidx(copies[i].base) << 10) | copies[i].off;
      size_t j = i + 1;
      while (j < copies.size() && (int64_t)(j - i) < RUN_MAX) {
        const int64_t cj = (bidx(copies[j].base) << 10) | copies[j].off;
        const int64_t cp = (bidx(copies[j - 1].base) << 10) | copies[j - 1].off;
        if (copies[j].cell != copies[j - 1].cell + 1 || copies[j].cell % RS == 0 || (cj >> 10) != (cp >> 10) ||
            (cj & 1023) != (cp & 1023) + 1)
          break;
        ++j;
      }
      const int64_t len = (int64_t)(j - i);
      runs.push_back({copies[i].cell, len, code0, len > 4 ? 0 : len > 2 ? 1 : len > 1 ? 2 : 3});
      i = j;
    }
    std::sort(runs.begin(), runs.end(), [](const Run& a, const Run& b) {
      return a.bucket != b.bucket ? a.bucket < b.bucket : a.cell < b.cell;
    });
    int64_t bcnt[4] = {0, 0, 0, 0};
    for (auto& r : runs) ++bcnt[r.bucket];
    // rows and taps
    const int64_t nrow = (int64_t)hr.size();
    if (nrow >= 1024) {
      err |= 8;
      continue;
    }
    std::vector<uint32_t> row_words(nrow);
    std::vector<uint16_t> taps;
    for (int64_t i = 0; i < nrow; ++i) {
      const int64_t e = hr[i].second;
      const int64_t r = -(int64_t)row[e] - 2;
      const int64_t cnt = iptr[r + 1] - iptr[r];
      const int64_t nq = (cnt + 3) / 4;
      const int64_t qoff = (int64_t)taps.size() / 4;
      if (nq > 31 || qoff >= (1 << 15) || cell[e] >= (1 << 12)) {
        err |= 16;
        break;
      }
      row_words[i] = (uint32_t)(cell[e] | (nq << 12) | (qoff << 17));
      for (int64_t k = iptr[r]; k < iptr[r + 1]; ++k) {
        const int64_t sl = std::lower_bound(slots.begin(), slots.end(), (int64_t)igid[k]) - slots.begin();
        taps.push_back((uint16_t)((sl << 6) | widx_of(iw[k])));
      }
      for (int64_t k = cnt; k < 4 * nq; ++k) taps.push_back((uint16_t)((nslot << 6) | zero_w));
    }
    // head
    const int64_t nbase = (int64_t)bases.size(), nrun = (int64_t)runs.size();
    const int64_t off_base = 4 * HDR_WORDS;
    const int64_t off_run = off_base + r16(4 * nbase);
    const int64_t off_slot = off_run + r16(4 * nrun);
    const int64_t head_len = off_slot + r16(2 * nslot);
    const int64_t rows_b = r16(4 * nrow);
    const int64_t tail_len = rows_b + r16(2 * (int64_t)taps.size());
    TileOut& o = outs[t];
    o.head.assign(head_len / 4, 0u);
    o.head_bytes = head_len;
    o.tail_bytes = tail_len;
    const int64_t lmeta = level[leaf] | ((int64_t)tc << 8) | ((int64_t)faces << 16);
    const int64_t hdr[HDR_WORDS] = {g0, g1 - g0, lmeta, nrun, nslot, nrow, nbase, tail_len,
                                    anchor[leaf * 3], anchor[leaf * 3 + 1], anchor[leaf * 3 + 2],
                                    bcnt[0] | (bcnt[1] << 16), bcnt[2] | (bcnt[3] << 16), 0,
                                    0 /* tail offset: filled at assembly */, rows_b / 2};
    for (int i = 0; i < HDR_WORDS; ++i) o.head[i] = (uint32_t)hdr[i];
    for (int64_t i = 0; i < nbase; ++i) o.head[off_base / 4 + i] = (uint32_t)(int32_t)bases[i];
    for (int64_t i = 0; i < nrun; ++i)
      o.head[off_run / 4 + i] = (uint32_t)(runs[i].cell | ((runs[i].len - 1) << 12) | (runs[i].code << 16));
    uint16_t* h16 = reinterpret_cast<uint16_t*>(o.head.data());
    for (int64_t k = 0; k < nslot; ++k)
      h16[off_slot / 2 + k] = (uint16_t)((bidx(sslot[k].first) << 10) | sslot[k].second);
    o.tail.assign(tail_len / 2, 0);
    for (int64_t i = 0; i < nrow; ++i) std::memcpy(&o.tail[2 * i], &row_words[i], 4);
    std::copy(taps.begin(), taps.end(), o.tail.begin() + rows_b / 2);
    n_rows_t[t] = nrow;
    n_cells_t[t] = ncells;
    n_slots_t[t] = nslot;
  }
  if (err) {
    amr_set_error_internal(
        (err & 2) ? "programs: a tile reads more source groups than the encoding holds (> 63)"
                  : (err & 1) ? "programs: a tile reads too many interpolation sources (> 1022)"
                              : "programs: tile does not fit the compact encoding");
    delete P;
    return nullptr;
  }
  // ---- assembly: heads at a fixed stride, tails back to back (16-byte aligned)
  int64_t max_head = 64, tail_total = 0;
  for (auto& o : outs) {
    max_head = std::max(max_head, o.head_bytes);
    P->max_tail = std::max(P->max_tail, o.tail_bytes);
    tail_total += o.tail_bytes;
  }
  if (tail_total / 16 >= ((int64_t)1 << 31)) {
    amr_set_error_internal("programs: tile tails exceed 32 GB");
    delete P;
    return nullptr;
  }
  P->max_head = n_tiles ? max_head : 64;
  P->heads.assign((size_t)std::max<int64_t>(n_tiles, 1) * P->max_head, 0);
  P->tail.assign((size_t)std::max<int64_t>(tail_total / 2, 8), 0);
  std::vector<int64_t> tstart(n_tiles + 1, 0);
  for (int64_t t = 0; t < n_tiles; ++t) tstart[t + 1] = tstart[t] + outs[t].tail_bytes;
#pragma omp parallel for schedule(static) num_threads(nth)
  for (int64_t t = 0; t < n_tiles; ++t) {
    TileOut& o = outs[t];
    o.head[14] = (uint32_t)(tstart[t] / 16);
    std::memcpy(&P->heads[(size_t)t * P->max_head], o.head.data(), o.head_bytes);
    if (o.tail_bytes) std::memcpy(&P->tail[tstart[t] / 2], o.tail.data(), o.tail_bytes);
    std::vector<uint32_t>().swap(o.head);
    std::vector<uint16_t>().swap(o.tail);
  }
  for (int64_t t = 0; t < n_tiles; ++t) {
    P->n_rows += n_rows_t[t];
    P->n_cells += n_cells_t[t];
    P->max_slots = std::max(P->max_slots, n_slots_t[t]);
  }
  return P;
}

// info[0..7] = n_tiles, max_head, max_tail, max_slots, n_iface, n_wtab, tail uint16 count, n_rows; info[8] = n_cells
extern "C" int amr_programs_info(const AmrProg* P, int64_t* info) {
  info[0] = P->n_tiles;
  info[1] = P->max_head;
  info[2] = P->max_tail;
  info[3] = P->max_slots;
  info[4] = (int64_t)P->if_gid.size();
  info[5] = (int64_t)P->wtab.size();
  info[6] = (int64_t)P->tail.size();
  info[7] = P->n_rows;
  info[8] = P->n_cells;
  return AMR_OK;
}

extern "C" int amr_programs_fetch(const AmrProg* P, uint8_t* heads, uint16_t* tail, int32_t* if_gid, int32_t* if_cad,
                                  double* wtab) {
  std::memcpy(heads, P->heads.data(), P->heads.size());
  std::memcpy(tail, P->tail.data(), P->tail.size() * 2);
  if (!P->if_gid.empty()) {
    std::memcpy(if_gid, P->if_gid.data(), P->if_gid.size() * 4);
    std::memcpy(if_cad, P->if_cad.data(), P->if_cad.size() * 4);
  }
  std::memcpy(wtab, P->wtab.data(), P->wtab.size() * 8);
  return AMR_OK;
}

extern "C" void amr_programs_free(AmrProg* P) { delete P; }
