/*
 * amr_b200.h — C ABI of the B200-native LTS/GTS octree wave solver.
 *
 * The reference (`amrlts`, pure Python) has no FFI: its boundary is the Python
 * module API.  These entry points are what that API's hot calls bind to
 * (ctypes); each cites the reference function it replaces.
 * Plain pointers and sizes only.  Device pointers are owned by the caller
 * (torch tensors in our Python facade); nothing here allocates or frees
 * caller memory.  Every function returns 0 on success, otherwise an AMR_E*
 * code; amr_last_error() returns a message for the calling thread.
 *
 * Index conventions: a leaf is identified by its position in the tree's SFC
 * order; anchors are in finest-cell units (octree.py:5-8); lattice points are
 * in units of a finest cell / (ppo-1) (mesh.py:8-11); gids are the zip-node
 * ids of the reference (first-claim order, mesh.py:235-245).
 */
#ifndef AMR_B200_H
#define AMR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  AMR_OK = 0,
  AMR_EINVAL = 1,     /* bad argument (maps to ValueError) */
  AMR_ESTATE = 2,     /* inconsistent state (maps to RuntimeError) */
  AMR_ECUDA = 3,      /* CUDA launch/runtime failure */
  AMR_ENOMEM = 4
};

const char* amr_last_error(void);
int amr_abi_version(void);

/* ---------------------------------------------------------------- octree -- */

/* Morton order (x lowest bit, ancestors first) of n octants:
 * perm[k] = index of the k-th octant.  Replaces the sort in construct /
 * balance_2to1 / parse_dump with SfcOrdering("morton") (octree.py:175-198,270,329). */
int amr_morton_sort(int dim, int max_depth, int64_t n, const int32_t* anchors,
                    const int32_t* levels, int64_t* perm);

/* Unique minimal 2:1 (face+edge+corner) balanced refinement
 * (octree.py:289-330).  Two-call: first with anchors_out == NULL returns the
 * leaf count in *n_out; the second fills Morton-sorted outputs. */
typedef struct AmrTree AmrTree;
AmrTree* amr_balance(int dim, int max_depth, int64_t n, const int32_t* anchors,
                     const int32_t* levels, int64_t* n_out);
int amr_tree_fetch(const AmrTree* t, int32_t* anchors_out, int32_t* levels_out);
void amr_tree_free(AmrTree* t);

/* Device octree (octree.py:249-330 on the GPU; csrc/amr_octree.cu).  An
 * octant is the 64-bit key morton(anchor) << 6 | level; a linear octree is a
 * sorted key array in device memory.  Refinement (construct, octree.py:249-271)
 * and the 2:1 balance ripple (octree.py:289-330) are rounds of
 * mark -> exclusive prefix sum of the output counts (1, or 2^dim when marked;
 * the caller's) -> amr_oct_split, which keeps the array sorted.
 * amr_oct_balance_mark marks every leaf that is more than one level coarser
 * than a leaf probing it (the reference's diagonal probe cells); mark must be
 * zero on entry; balance is reached when it stays zero.  All pointers are
 * device pointers. */
int amr_oct_keys(int dim, int max_depth, int64_t n, const int32_t* anchors, const int32_t* levels,
                 uint64_t* keys, void* stream);
int amr_oct_octants(int dim, int max_depth, int64_t n, const uint64_t* keys, int32_t* anchors,
                    int32_t* levels, void* stream);
int amr_oct_split(int dim, int max_depth, int64_t n, const uint64_t* keys, const int32_t* mark,
                  const int64_t* offsets, uint64_t* out, void* stream);
int amr_oct_balance_mark(int dim, int max_depth, int64_t n, const uint64_t* keys, int32_t* mark,
                         void* stream);

/* ------------------------------------------------------------------ mesh -- */

/* Node registry + leaf-tile gather tables (mesh.py:214-398).  `owners` (may be
 * NULL) are the partition ranks used only to split the public maximal blocks
 * (decompose_blocks, mesh.py:87-135).  Leaves must be in the tree's SFC
 * order (any SFC), complete and 2:1 balanced. */
typedef struct AmrMesh AmrMesh;
AmrMesh* amr_mesh_build(int dim, int max_depth, int ppo, int pad, int64_t n_leaves,
                        const int32_t* anchors, const int32_t* levels, const int32_t* owners,
                        int n_threads);
/* The same tables built on the device (csrc/amr_devmesh.cu; all pointers are
 * device pointers; keys = the tree's sorted 64-bit keys, amr_oct_keys).  The
 * passes of amr_mesh_build, one launch each:
 *   amr_dm_ownership  status[n][ppo^dim] (1 owned, 0 shared, -1 hanging), owner leaf, owned count per leaf;
 *   amr_dm_gids       leaf_gids from the exclusive prefix sum `starts` of the counts (the caller's);
 *   amr_dm_table      tile table with -2 at hanging points, and their number per leaf;
 *   amr_dm_hang_list  (table position, lattice code) of every hanging entry, at the exclusive prefix sum hang_off;
 *   amr_dm_table_rows table[pos] = -2 - row, row = index of the code among the sorted unique codes (the caller's);
 *   amr_dm_rows       interpolation rows of those codes: with row_ptr == NULL the tap counts, else the
 *                     gid-sorted taps at row_ptr (exclusive prefix sum of the counts).
 * err (device int, zero on entry) collects: 1 point outside every leaf, 2 row longer than 128 taps,
 * 4 hanging taps nested deeper than 6.  amr_mesh_from_tables wraps host copies of the results in a
 * mesh handle (blocks, views and the program builder work as after amr_mesh_build). */
int amr_dm_ownership(int dim, int max_depth, int ppo, int pad, int64_t n, const uint64_t* keys,
                     const int32_t* anchors, const int32_t* levels, int8_t* status, int32_t* owner,
                     int64_t* counts, int* err, void* stream);
int amr_dm_gids(int dim, int max_depth, int ppo, int pad, int64_t n, const uint64_t* keys, const int32_t* anchors,
                const int32_t* levels, const int8_t* status, const int32_t* owner, const int64_t* starts,
                int32_t* leaf_gids, void* stream);
int amr_dm_table(int dim, int max_depth, int ppo, int pad, int64_t n, const uint64_t* keys, const int32_t* anchors,
                 const int32_t* levels, const int32_t* leaf_gids, int32_t* table, int32_t* n_hang, void* stream);
int amr_dm_hang_list(int dim, int max_depth, int ppo, int pad, int64_t n, const uint64_t* keys,
                     const int32_t* anchors, const int32_t* levels, const int32_t* table, const int64_t* hang_off,
                     int64_t* pos, int64_t* code, void* stream);
int amr_dm_table_rows(int64_t n_hang, const int64_t* pos, const int64_t* code, int64_t n_rows, const int64_t* rows,
                      int32_t* table, void* stream);
int amr_dm_rows(int dim, int max_depth, int ppo, int pad, int64_t n, const uint64_t* keys, const int32_t* anchors,
                const int32_t* levels, const int32_t* leaf_gids, int64_t n_rows, const int64_t* codes,
                const int64_t* row_ptr, int32_t* counts, int32_t* gid_out, double* w_out, int* err, void* stream);
AmrMesh* amr_mesh_from_tables(int dim, int max_depth, int ppo, int pad, int64_t n_leaves, const int32_t* anchors,
                              const int32_t* levels, const int32_t* owners, const int64_t* starts,
                              const int32_t* leaf_gids, const int32_t* table, int64_t n_rows,
                              const int64_t* hang_codes, const int64_t* row_ptr, const int32_t* gid,
                              const double* w);
void amr_mesh_free(AmrMesh* m);

int64_t amr_mesh_n_nodes(const AmrMesh* m);
/* leaf_slices (mesh.py:250-254): starts[n_leaves+1]; leaf i owns [starts[i], starts[i+1]) */
int amr_mesh_leaf_starts(const AmrMesh* m, int64_t* starts);
/* leaf_gids (mesh.py:249): [n_leaves][ppo^dim], -1 = hanging */
int amr_mesh_leaf_gids(const AmrMesh* m, int32_t* gids);
/* node_coords (mesh.py:257-265): [n_nodes][dim] lattice coordinates */
int amr_mesh_node_coords(const AmrMesh* m, int32_t* coords);

/* Leaf-tile unzip tables: per leaf, amr_tile_entries(dim,ppo) int32 entries
 * over the stencil cross (ppo^dim interior + 2*dim*pad*ppo^(dim-1) face halo).
 * entry >= 0: copy of zip node `entry`; -1: outside the domain (zero row);
 * <= -2: interpolation row (-entry-2) of the CSR below (the engine remaps
 * these to the tile's own interpolation rows, and LTS copies whose source
 * steps differently to interface pairs: entry <= -(1<<20)). */
int64_t amr_tile_entries(int dim, int ppo);
int amr_mesh_tile_table(const AmrMesh* m, int32_t* table);
int64_t amr_mesh_interp_rows(const AmrMesh* m);
int64_t amr_mesh_interp_nnz(const AmrMesh* m);
/* rows sorted by gid (mesh.py:391-393); weights from the recursive
 * tensor-product Lagrange resolution (mesh.py:316-351) */
int amr_mesh_interp_csr(const AmrMesh* m, int64_t* row_ptr, int32_t* gid, double* w);

/* Per-tile stage programs (the native builder of paper_2011_10570_b200/
 * tileprog.py, byte-identical to it): tiles = leaves in launch order,
 * leaf_cad = each leaf's cadence (time level), lts = 1 to form LTS interface
 * pairs, row_stride = the stencil box's row stride (Tile::RS).  info[9]:
 * n_tiles, max_head, max_tail, max_slots, n_iface, n_wtab, tail uint16
 * count, hanging rows, owned-cross cells.  fetch fills heads
 * [n_tiles][max_head], tail, if_gid/if_cad [n_iface], wtab [n_wtab]. */
typedef struct AmrProg AmrProg;
AmrProg* amr_programs_build(const AmrMesh* m, int64_t n_tiles, const int32_t* tiles, const int32_t* leaf_cad,
                            int lts, int row_stride, int n_threads);
int amr_programs_info(const AmrProg* p, int64_t* info);
int amr_programs_fetch(const AmrProg* p, uint8_t* heads, uint16_t* tail, int32_t* if_gid, int32_t* if_cad,
                       double* wtab);
void amr_programs_free(AmrProg* p);

/* The same programs built on the device (csrc/amr_devprog.cu), byte-identical
 * to amr_programs_build.  All pointers are device pointers.  cell / cell2e /
 * pos are the cross-entry lookup tables of tileprog.cross_cells (box cell of an
 * entry, its inverse, interior positions [NI][3]); ukeys / grp_start / wtab
 * are filled in by the caller between the passes (sort/unique of the candidate
 * keys and of the used rows' weights):
 *   amr_dp_need    need[n_tiles][E], row_used[n_rows], n_keys[n_tiles];
 *   amr_dp_keys    candidate keys at the exclusive prefix offsets key_off;
 *   amr_dp_encode  heads == NULL: sizes[n_tiles][5] = head bytes, tail bytes, slots, rows, cells;
 *                  else heads at stride max_head and tails at tail_off (bytes, 16-aligned).
 * Kernels run `blocks` x `threads` threads over the tiles; scratch holds
 * amr_dp_scratch_bytes(blocks * threads).  err bits: 1 > 1022 slots, 2 > 63
 * source groups, 4 offset >= 1024, 8 > 1023 rows, 16 row word overflow. */
typedef struct {
  int dim, max_depth, ppo, lts, row_stride, n_wtab, max_bases;
  int64_t n_leaves, n_tiles, n_iface;
  const int32_t* table;
  const int64_t* starts;
  const int32_t* anchors;   /* [n_leaves][dim] */
  const int32_t* levels;
  const int32_t* leaf_cad;
  const int32_t* tiles;
  const int64_t* row_ptr;
  const int32_t* gid;
  const double* w;
  const int32_t* cell;
  const int32_t* cell2e;
  const int16_t* pos;
  const int64_t* ukeys;
  const int64_t* grp_start;
  const double* wtab;
} AmrDevProg;
int amr_dp_scratch_bytes(int threads_total, int64_t* bytes);
int amr_dp_need(const AmrDevProg* a, uint8_t* need, uint8_t* row_used, int64_t* n_keys, int blocks, int threads,
                void* stream);
int amr_dp_keys(const AmrDevProg* a, const uint8_t* need, const int64_t* key_off, int64_t* keys, int blocks,
                int threads, void* stream);
int amr_dp_encode(const AmrDevProg* a, const uint8_t* need, void* scratch, int64_t* sizes, uint8_t* heads,
                  int64_t max_head, const int64_t* tail_off, uint16_t* tail, int* err, int blocks, int threads,
                  void* stream);

/* Public maximal blocks (decompose_blocks, mesh.py:87-135) */
int64_t amr_mesh_n_blocks(const AmrMesh* m);
int amr_mesh_blocks(const AmrMesh* m, int32_t* root_anchor, int32_t* root_level,
                    int32_t* leaf_level, int64_t* leaf_range, int32_t* owner);
/* Gather CSR of one block's padded grid (mesh.py:355-398).  Two-call: with
 * row_ptr == NULL returns rows and nnz; then fills (row_ptr[rows+1]). */
int amr_mesh_block_gather(AmrMesh* m, int64_t block, int64_t* rows, int64_t* nnz,
                          int64_t* row_ptr, int64_t* col, double* val);

/* --------------------------------------------------------------- kernels -- */

/* Per-slice LTS coefficient block (device memory, built by the host from
 * rkcorrect.stage_transfer_matrix, stepper.py:238-314).  Levels are absolute
 * octree levels < AMR_MAXL. */
#define AMR_MAXL 16
#define AMR_MAXP 4
typedef struct {
  int32_t cur[AMR_MAXL];                 /* u_curr buffer (0/1) per cadence level */
  int32_t mode[AMR_MAXL][AMR_MAXL];      /* [reader][source]: 0 verbatim, 1 delta=0 transfer, 2 virtual substep */
  double cstage[AMR_MAXL][AMR_MAXP][AMR_MAXP]; /* dt_to * a[s][j] per reader level */
  double comb[AMR_MAXL][AMR_MAXP];       /* dt * w[s] per stepping level */
  double M[AMR_MAXL][AMR_MAXL][AMR_MAXP][AMR_MAXP];  /* stage transfer (tril when delta=0) */
  double Mv[AMR_MAXL][AMR_MAXL][AMR_MAXP][AMR_MAXP]; /* virtual-substep transfer */
  double dtw[AMR_MAXL][AMR_MAXL][AMR_MAXP];          /* delta*dt_fine*w[i] */
} AmrSliceCoef;

typedef struct {
  int dim, ppo, pad;
  int lts;             /* 0: global stepping (all verbatim), 1: local stepping */
  int stage, n_stages; /* s, p */
  int nonlinear;       /* 0 none, 1 sin(2chi)/r^2 (wave.py:162-163), 2 cubic chi^3 */
  int gts_cur;         /* GTS: u_curr buffer index */
  int64_t n_tiles;     /* tiles of this launch: a prefix of the launch order (finest cadence first) */
  int64_t n_nodes;
  int64_t ld;          /* row stride (elements) of U0/U1/K/Y: even, >= n_nodes + 1 */
  /* per-tile stage programs in launch order (paper_2011_10570_b200/tileprog.py):
   * heads (header, source bases, copy runs, slot codes) at a fixed stride of
   * max_head bytes, bulk-copied into shared memory; tails (hanging rows, taps)
   * 16-byte aligned, read through L2 */
  const uint8_t* heads;
  const uint16_t* tail;
  int max_head;
  int max_tail;                /* largest tail in bytes (bulk-copied into shared memory) */
  int max_slots;               /* largest interpolation-source set of any tile (shared memory) */
  int threads;                 /* threads per CTA: 128 or 256 */
  int lean;                    /* 1: every tile of this launch is off the physical faces (and the source is not
                                  sin): run the lean kernel instance (no face / coordinate paths) */
  long long* probe;            /* NULL, or [n_tiles][8] phase timestamps (builds with -DAMR_PHASE_PROBE) */
  const double* wtab;          /* distinct interpolation weights (<= 64, device) */
  int n_wtab;
  /* LTS interface pairs (zip node, reader cadence) whose source steps differently
   * from the reader: computed once per stage by amr_iface into ibuf */
  int64_t n_iface;             /* pairs of this launch (prefix: finest readers first) */
  int64_t n_iface_total;
  const int32_t* if_gid;
  const int32_t* if_cad;       /* reader cadence | source cadence << 8 */
  double* ibuf;                /* [2][n_iface_total]: the slab of this stage, read by amr_stage */
  double* ibuf0;               /* [n_stages][2][n_iface_total]: all slabs, written by amr_iface */
  int if_phase;                /* amr_iface: 0 every pair for this stage; 1 (stage 0) also all stages of the
                                  pairs whose source is not stepping now; 2 (later stages) skip those pairs */
  int n_vt;                    /* verbatim stage-source terms of stage s+1 (a[s+1][j] != 0) */
  int vt_j[AMR_MAXP];          /* their j */
  double* Y;                   /* [2 buffers][2][ld]: verbatim sources; stage s reads buffer s&1 and its
                                  owners write stage s+1's into buffer (s+1)&1 */
  double* U0;                  /* [2][ld]: the reference's zip layout (chi row, phi row) */
  double* U1;
  double* K;                   /* [n_stages][2][ld] */
  const AmrSliceCoef* coef;    /* LTS only (device): read by amr_iface */
  /* LTS values the stage kernel reads, by value (copies of coef's entries for this slice and stage) */
  uint32_t l_cur_mask;                 /* bit c: u_curr buffer of cadence c (coef->cur) */
  double l_cnext[AMR_MAXL][AMR_MAXP];  /* coef->cstage[c][stage + 1][j] */
  double l_comb[AMR_MAXL][AMR_MAXP];   /* coef->comb[c][j] */
  /* GTS coefficients */
  double g_cstage[AMR_MAXP][AMR_MAXP];
  double g_comb[AMR_MAXP];
  /* geometry (mesh.py:459-492, wave.py:124-144) */
  int max_depth;
  int64_t top_nodes;
  double lo[3], extent[3];
  double h[AMR_MAXL], h2[AMR_MAXL];
  int32_t h2_pow2[AMR_MAXL];   /* 1: h**2 is a power of two -> multiply by inv_h2 (bit-identical) */
  double inv_h2[AMR_MAXL];
  double r_eps, r_eps2;
  double k_chi, k_phi, f0_chi, f0_phi;
  /* stencil weights: the reference's Fornberg arrays, bit for bit (wave.py:49-54) */
  double d2c[5], d2e0[6], d2e1[6], d1c[5], d1e0[5], d1e1[5];
} AmrStageParams;

/* One RK stage over a prefix of the tile list: fused unzip on each tile's
 * owned cross (copies, LTS interface sources, hanging rows summed in
 * ascending-gid order) + RHS stencil + zip of K_s and the next stage's
 * verbatim source; the last stage also fuses the RK combine and record
 * rotation.  Replaces Engine._stage_source +
 * gathers[b].dot + wave_rhs + the K/state scatter (stepper.py:274-314,
 * 395-453). */
int amr_stage(const AmrStageParams* p, void* stream);

/* Layout self-check for bindings: out[0] = sizeof(AmrStageParams), then the
 * byte offsets of n_tiles, heads, max_tail, probe, wtab, n_iface, ibuf, vt_j,
 * Y, coef, g_cstage, g_comb, max_depth, top_nodes, lo, h2_pow2, inv_h2, r_eps,
 * f0_phi, d2c, d1e1.  Returns the number of values written (<= cap). */
int amr_stage_params_layout(int64_t* out, int cap);

/* LTS interface pass of a stage (before amr_stage): ibuf[i] = stage source of
 * zip node if_gid[i] as seen by readers of cadence if_cad[i] — the delta=0
 * stage transfer or the virtual substep + transfer (stepper.py:256-314). */
int amr_iface(const AmrStageParams* p, void* stream);



/* Mesh.unzip (mesh.py:413-420): out[v][r] = 0 + sum_k w_k * z[v][col_k] over
 * CSR rows (ascending col), z/out in (nv, n) layout. */
int amr_gather_rows(int64_t n_rows, const int64_t* row_ptr, const int64_t* col,
                    const double* val, int nv, const double* z, int64_t z_stride,
                    double* out, int64_t out_stride, void* stream);

/* wave_rhs on one padded block array (wave.py:147-201).  y: [2][n+2pad]^dim,
 * out: [2][n]^dim; faces bitmask bit(2*axis+side); coords: per-axis interior
 * physical coordinates (n each). */
int amr_block_rhs(int dim, int n, int pad, const double* y, double* out, double h, double h2,
                  const double* coords, double r_eps, int faces, int nonlinear,
                  double k_chi, double k_phi, double f0_chi, double f0_phi,
                  const AmrStageParams* weights, void* stream);

/* Ghost-leaf records between ranks (Engine._ship, stepper.py:318-361;
 * exchange, partition.py:182-207).  A shipment is a list of whole-leaf zip
 * ranges, finest cadence first, so the leaves that stepped at a slice are a
 * prefix (n_ranges, total).  pack writes buf[row * buf_ld + node]; unpack reads
 * it back into the receiver's rows.  Each row has two base pointers: a range
 * uses row1 when par[its cadence] is 1 (the two u buffers, selected per
 * cadence by the step parity); K and Y rows pass the same pointer twice. */
#define AMR_GHOST_ROWS 8
typedef struct {
  int64_t n_ranges;       /* ranges moved: a prefix of the list */
  int64_t total;          /* zip nodes in that prefix */
  const int64_t* start;   /* first node of each range in the rank's rows (device) */
  const int64_t* off;     /* exclusive prefix sum of the range lengths (device) */
  const int32_t* cad;     /* cadence of each range (device) */
  int n_rows;             /* field rows moved per node (<= AMR_GHOST_ROWS) */
  int64_t buf_ld;         /* row stride of buf in doubles; 0 = total (rows back to back) */
  double* row0[AMR_GHOST_ROWS];
  double* row1[AMR_GHOST_ROWS];
  int32_t par[AMR_MAXL];  /* parity per cadence */
} AmrGhostMove;
int amr_ghost_pack(const AmrGhostMove* m, double* buf, void* stream);
int amr_ghost_unpack(const AmrGhostMove* m, const double* buf, void* stream);

/* -------------------------------------------------------------- wavelet -- */

/* Interpolation-residual refinement coefficient of n octants
 * (wavelet_coefficient, wavelet.py:70-105) and, when `flags` is non-NULL, the
 * per-octant decision in the same launch: mode 0 = refine_flags
 * (wavelet.py:108-124; 1 refine, 0 keep, -1 coarsen, coarsen_thr =
 * coarsen_factor*tolerance), mode 1 = refinement_predicate (wavelet.py:127-144;
 * 1 split, 0 leaf).  values: device [n][npd^dim] samples on each octant's
 * closed tensor grid (octant_samples, wavelet.py:57-67; last axis fastest);
 * W: device [npd][(npd+1)/2], the reference's _lagrange_matrix(xs[::2], xs)
 * (wavelet.py:41-54); levels: device [n] (NULL when flags is NULL); coeff:
 * device [n] or NULL.  npd odd, 3..15; dim 2 or 3. */
int amr_wavelet_coeff(int dim, int npd, int64_t n, const double* values, const double* W,
                      const int32_t* levels, int mode, double tol, double coarsen_thr,
                      int min_level, int max_level, double* coeff, int8_t* flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif
