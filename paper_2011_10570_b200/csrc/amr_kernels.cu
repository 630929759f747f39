// amr_kernels.cu — sm_100a kernels of the B200 LTS/GTS wave solver.
//
// Hot path: amr_stage.  One CTA owns one leaf tile (ppo^D computed nodes,
// (ppo-1)^D owned when interior).  Per RK stage it
//   1. builds the tile's stage input on the stencil cross in shared memory:
//      for every cross point the unzip entry is a copy of one zip node, a
//      sorted interpolation row, or zero (outside the domain), and every zip
//      node read is first turned into the reader's stage source — verbatim
//      u + sum_j dt a_sj K_j, or, at LTS level interfaces, the stage-transfer
//      product M K (and the virtual substep for non-eligible coarse sources);
//      (Engine._stage_source + Mesh.unzip, stepper.py:274-314, mesh.py:413-420)
//   2. evaluates the 4th-order RHS (biased rows and radiative overwrite at
//      physical faces; linear, sin or cubic source) only at the nodes the
//      leaf owns and writes K_s for them contiguously (wave.py:147-201 and the
//      zip of stepper.py:422-429);
//   3. on the last stage also does the RK combine u_new = u + sum dt w_s K_s
//      into the other u buffer (record rotation u_pre <- u_curr without a
//      copy: the live buffer of a leaf is the parity of its step count).
//
// Arithmetic follows the reference bit for bit: -fmad=false for the whole
// file, numpy's operation order, the reference's Fornberg weight arrays, and
// fma() only where the reference goes through OpenBLAS dgemm (np.tensordot at
// stepper.py:264,305 — an ascending-k FMA chain on the generating host).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/amr_b200.h"

extern "C" void amr_set_error_internal(const char* msg);

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  amr_set_error_internal((std::string(what) + ": " + cudaGetErrorString(e)).c_str());
  return AMR_ECUDA;
}

constexpr int cpow(int b, int e) { return e == 0 ? 1 : b * cpow(b, e - 1); }
constexpr int AMR_IFACE_BASE = -(1 << 20);  // table entries <= this: interface pair AMR_IFACE_BASE - entry

template <int DIM, int PPO>
struct Tile {
  static constexpr int PAD = 2;
  static constexpr int NP = PPO + 2 * PAD;
  static constexpr int NI = cpow(PPO, DIM);
  static constexpr int NF = cpow(PPO, DIM - 1);
  static constexpr int NE = NI + DIM * 2 * PAD * NF;
  static constexpr int NS = cpow(NP, DIM);
  static constexpr int THREADS = DIM == 3 ? 256 : 128;
};

// smem cell of cross entry e (same enumeration as cross_entry_local in amr_mesh.cpp)
template <int DIM, int PPO>
__device__ __forceinline__ int cross_cell(int e) {
  using T = Tile<DIM, PPO>;
  int loc[3];
  if (e < T::NI) {
    int r = e;
#pragma unroll
    for (int d = DIM - 1; d >= 0; --d) {
      loc[d] = T::PAD + r % PPO;
      r /= PPO;
    }
  } else {
    int r = e - T::NI;
    int axis = r / (2 * T::PAD * T::NF);
    r %= 2 * T::PAD * T::NF;
    int layer = r / T::NF;
    int within = r % T::NF;
    int lp = layer < T::PAD ? layer : PPO + layer;
#pragma unroll
    for (int d = DIM - 1; d >= 0; --d) {
      if (d == axis) continue;
      loc[d] = T::PAD + within % PPO;
      within /= PPO;
    }
    loc[axis] = lp;
  }
  int c = 0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) c = c * T::NP + loc[d];
  return c;
}


// Fields are SoA, the reference's (nvars, n_nodes) zip layout: var v of node g
// at base[v*n + g]; stage j of K at K + j*2n.
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ double2 ld_pair(const double* __restrict__ base, int64_t n, int64_t g) {
  return make_double2(__ldg(base + g), __ldg(base + n + g));
}

// --------------------------------------------------------------------------
// stage source of one zip node as seen by a reader of cadence lr (LTS):
// verbatim, delta=0 stage transfer, or virtual substep + transfer
// (Engine._stage_source / _virtual_state, stepper.py:256-314)
// --------------------------------------------------------------------------
__device__ __forceinline__ double2 lts_source(const double* __restrict__ U0, const double* __restrict__ U1,
                                              const double* __restrict__ K, int64_t n, int p, int g, int s, int lr,
                                              int ls, const AmrSliceCoef* __restrict__ C) {
  const int mode = C->mode[lr][ls];
  const int cur = C->cur[ls];
  const double* Uc = cur ? U1 : U0;
  if (mode == 0) {  // eligible, same step size: verbatim (stepper.py:290-296)
    const double2 u = ld_pair(Uc, n, g);
    double2 y = make_double2(0.0 + u.x, 0.0 + u.y);
    for (int j = 0; j < s; ++j) {
      const double c = C->cstage[lr][s][j];
      if (c != 0.0) {
        const double2 k = ld_pair(K + (int64_t)j * 2 * n, n, g);
        y.x = y.x + c * k.x;
        y.y = y.y + c * k.y;
      }
    }
    return y;
  }
  double2 kk[AMR_MAXP];
  const int nk = (mode == 1) ? s : p;  // delta=0 transfer is lower triangular
#pragma unroll
  for (int k = 0; k < AMR_MAXP; ++k)
    kk[k] = (k < nk) ? ld_pair(K + (int64_t)k * 2 * n, n, g) : make_double2(0.0, 0.0);
  double2 y;
  if (mode == 1) {
    y = ld_pair(Uc, n, g);
  } else {  // virtual substep from u_pre (stepper.py:256-270)
    y = ld_pair(cur ? U0 : U1, n, g);
    const double(*Mv)[AMR_MAXP] = C->Mv[lr][ls];
#pragma unroll
    for (int i = 0; i < AMR_MAXP; ++i) {
      if (i >= p) break;
      const double c = C->dtw[lr][ls][i];
      if (c == 0.0) continue;
      double ax = 0.0, ay = 0.0;
#pragma unroll
      for (int k = 0; k <= i; ++k) {
        ax = fma(Mv[i][k], kk[k].x, ax);
        ay = fma(Mv[i][k], kk[k].y, ay);
      }
      y.x = y.x + c * ax;
      y.y = y.y + c * ay;
    }
  }
  const double(*M)[AMR_MAXP] = C->M[lr][ls];
#pragma unroll
  for (int j = 0; j < AMR_MAXP; ++j) {
    if (j >= s) break;
    const double c = C->cstage[lr][s][j];
    if (c == 0.0) continue;
    const int kmax = (mode == 1) ? j : p - 1;
    double ax = 0.0, ay = 0.0;
#pragma unroll
    for (int k = 0; k < AMR_MAXP; ++k) {
      if (k > kmax) break;
      ax = fma(M[j][k], kk[k].x, ax);
      ay = fma(M[j][k], kk[k].y, ay);
    }
    y.x = y.x + c * ax;
    y.y = y.y + c * ay;
  }
  return y;
}

// --------------------------------------------------------------------------
// RHS at one interior point (wave.py:57-201), generic over the data accessor
// --------------------------------------------------------------------------
// Stencil weights are read straight from the by-value kernel parameter block
// (constant bank, compile-time indices after unrolling).
using Weights = AmrStageParams;

// derivative along one axis: centred, or the biased row near a physical face
// (derivative_axis, wave.py:67-109).  get(o) returns the value at offset o.
template <class Get>
__device__ __forceinline__ double deriv(const Get& get, int order, int pos, int n, bool lo, bool hi,
                                        const Weights& W, double hp, bool pow2, double inv_hp) {
  double t;
  if (order == 2) {
    if (lo && pos == 0) {
      t = W.d2e0[0] * get(0);
#pragma unroll
      for (int k = 1; k < 6; ++k) t = t + W.d2e0[k] * get(k);
    } else if (lo && pos == 1) {
      t = W.d2e1[0] * get(-1);
#pragma unroll
      for (int k = 1; k < 6; ++k) t = t + W.d2e1[k] * get(k - 1);
    } else if (hi && pos == n - 1) {
      t = W.d2e0[0] * get(0);
#pragma unroll
      for (int k = 1; k < 6; ++k) t = t + W.d2e0[k] * get(-k);
    } else if (hi && pos == n - 2) {
      t = W.d2e1[0] * get(1);
#pragma unroll
      for (int k = 1; k < 6; ++k) t = t + W.d2e1[k] * get(1 - k);
    } else {
      t = W.d2c[0] * get(-2);
#pragma unroll
      for (int k = 1; k < 5; ++k) t = t + W.d2c[k] * get(k - 2);
    }
  } else {
    if (lo && pos == 0) {
      t = W.d1e0[0] * get(0);
#pragma unroll
      for (int k = 1; k < 5; ++k) t = t + W.d1e0[k] * get(k);
    } else if (lo && pos == 1) {
      t = W.d1e1[0] * get(-1);
#pragma unroll
      for (int k = 1; k < 5; ++k) t = t + W.d1e1[k] * get(k - 1);
    } else if (hi && pos == n - 1) {
      t = (-W.d1e0[0]) * get(0);
#pragma unroll
      for (int k = 1; k < 5; ++k) t = t + (-W.d1e0[k]) * get(-k);
    } else if (hi && pos == n - 2) {
      t = (-W.d1e1[0]) * get(1);
#pragma unroll
      for (int k = 1; k < 5; ++k) t = t + (-W.d1e1[k]) * get(1 - k);
    } else {
      t = W.d1c[0] * get(-2);
#pragma unroll
      for (int k = 1; k < 5; ++k) t = t + W.d1c[k] * get(k - 2);
    }
  }
  return pow2 ? t * inv_hp : t / hp;
}

struct RhsConst {
  double h, h2, inv_h2;
  bool pow2;
  double r_eps, r_eps2;
  double k_chi, k_phi, f0_chi, f0_phi;
  int nonlinear;
};

// Acc: at(var, axis, offset) -> value; pos[d] interior index, n interior extent
template <int DIM, class Acc>
__device__ __forceinline__ double2 rhs_point(const Acc& acc, const int* pos, int n, int faces,
                                             const double* x, const Weights& W, const RhsConst& R) {
  double lap = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    auto get = [&](int o) { return acc.at(0, d, o); };
    double t = deriv(get, 2, pos[d], n, faces & (1 << (2 * d)), faces & (2 << (2 * d)), W, R.h2, R.pow2,
                     R.inv_h2);
    lap = (d == 0) ? t : lap + t;
  }
  const double chi = acc.at(0, 0, 0);
  const double phi = acc.at(1, 0, 0);
  double dchi = phi, dphi = lap;
  bool on_face = false;
#pragma unroll
  for (int d = 0; d < DIM; ++d)
    on_face |= (((faces >> (2 * d)) & 1) && pos[d] == 0) || (((faces >> (2 * d + 1)) & 1) && pos[d] == n - 1);
  if (R.nonlinear && !on_face) {
    if (R.nonlinear == 1) {
      double r2 = x[0] * x[0];
#pragma unroll
      for (int d = 1; d < DIM; ++d) r2 = r2 + x[d] * x[d];
      double r2_reg = r2 > R.r_eps2 ? r2 : R.r_eps2;
      dphi = dphi - sin(2.0 * chi) / r2_reg;
    } else {
      dphi = dphi - (chi * chi) * chi;
    }
  }
  if (on_face) {  // radiative rows (wave.py:173-201)
    double r2 = x[0] * x[0];
#pragma unroll
    for (int d = 1; d < DIM; ++d) r2 = r2 + x[d] * x[d];
    double r = sqrt(r2);
    r = r > R.r_eps ? r : R.r_eps;
    double rad[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      double a = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        auto get = [&](int o) { return acc.at(v, d, o); };
        double g = deriv(get, 1, pos[d], n, faces & (1 << (2 * d)), faces & (2 << (2 * d)), W, R.h, false, 0.0);
        double term = x[d] * g;
        a = (d == 0) ? term : a + term;
      }
      rad[v] = a / r;
    }
    dchi = rad[0] - R.k_chi * (chi - R.f0_chi);
    dphi = rad[1] - R.k_phi * (phi - R.f0_phi);
  }
  return make_double2(dchi, dphi);
}

// interior fast path: no physical face on the tile and no coordinate-dependent
// source: centred 4th-order Laplacian (+ cubic), dchi = phi (wave.py:147-170)
template <int DIM, class Acc>
__device__ __forceinline__ double2 rhs_interior(const Acc& acc, const Weights& W, const RhsConst& R) {
  double lap = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    double t = W.d2c[0] * acc.at(0, d, -2);
#pragma unroll
    for (int k = 1; k < 5; ++k) t = t + W.d2c[k] * acc.at(0, d, k - 2);
    t = R.pow2 ? t * R.inv_h2 : t / R.h2;
    lap = (d == 0) ? t : lap + t;
  }
  const double chi = acc.at(0, 0, 0);
  double dphi = lap;
  if (R.nonlinear == 2) dphi = dphi - (chi * chi) * chi;
  return make_double2(acc.at(1, 0, 0), dphi);
}

// centred 4th-order Laplacian at box pointer b when h**2 is a power of two
// (the division by h**2 is then an exact multiplication): the operation order
// of rhs_interior / derivative_axis (wave.py:57-109)
template <int DIM, int PPO>
__device__ __forceinline__ double lap_pow2(const double* b, const AmrStageParams& W, double inv_h2) {
  constexpr int NP = Tile<DIM, PPO>::NP;
  double lap = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const int S = (DIM == 3) ? (d == 0 ? NP * NP : (d == 1 ? NP : 1)) : (d == 0 ? NP : 1);
    double t = W.d2c[0] * b[-2 * S];
    t = t + W.d2c[1] * b[-S];
    t = t + W.d2c[2] * b[0];
    t = t + W.d2c[3] * b[S];
    t = t + W.d2c[4] * b[2 * S];
    t = t * inv_h2;
    lap = (d == 0) ? t : lap + t;
  }
  return lap;
}

template <int DIM, int PPO>
struct SmemAcc {
  const double* chi;
  const double* phi;
  int cell;
  __device__ __forceinline__ double at(int v, int d, int o) const {
    constexpr int NP = Tile<DIM, PPO>::NP;
    const int stride = (DIM == 3) ? (d == 0 ? NP * NP : (d == 1 ? NP : 1)) : (d == 0 ? NP : 1);
    return (v == 0 ? chi : phi)[cell + o * stride];
  }
};

// --------------------------------------------------------------------------
// the stage kernel: one CTA per leaf tile.  Tables are stored in launch
// (tile) order, so the table load does not wait for the tile's leaf id.
// --------------------------------------------------------------------------

// LTS interface pass: the stage source of every (zip node, reader cadence)
// pair whose step size or time differs from the reader's (delta=0 transfer or
// virtual substep + transfer, stepper.py:256-314), once per stage, so the
// stage kernel reads it like a copy.  Pairs are sorted finest reader first:
// the eligible readers of a slice are a prefix.
__global__ void __launch_bounds__(256) iface_kernel(const AmrStageParams P) {
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= P.n_iface) return;
  const int g = __ldg(P.if_gid + i);
  const int cc = __ldg(P.if_cad + i);  // reader cadence | source cadence << 8 (no dependent lookup)
  const double2 v = lts_source(P.U0, P.U1, P.K, P.ld, P.n_stages, g, P.stage, cc & 0xFF, cc >> 8, P.coef);
  P.ibuf[i] = v.x;
  P.ibuf[P.n_iface_total + i] = v.y;
}

#ifndef AMR_MIN_BLOCKS
#define AMR_MIN_BLOCKS 4  // resident CTAs per SM the register budget is sized for (tuned: 2,3,4 -> 8.0,9.7,10.2 G LTS upd/s)
#endif

// The stage kernel.  Per tile:
//  1a  table entries + slot ids (independent of the leaf-id load)
//  1b  all gathers in flight: chi (u and the K_j of the verbatim source) for
//      every copy entry and slot; phi only where the stencil needs it (owned
//      nodes: dchi = phi; every entry of tiles on a physical face: radiative
//      gradients)
//  1c  copy rows (0 + 1.0*src) -> smem cross; slot stage sources -> smem
//  1d  hanging rows: 0 + sum w*src in ascending-gid order -> smem cross
//  2   RHS at the owned nodes; K_s out (last stage: RK combine into the other u)
template <int DIM, int PPO, bool LTS, int NT>
__global__ void __launch_bounds__(Tile<DIM, PPO>::THREADS, AMR_MIN_BLOCKS)
    stage_kernel(const AmrStageParams P) {
  using T = Tile<DIM, PPO>;
  constexpr int EPT = (T::NE + T::THREADS - 1) / T::THREADS;
  constexpr int EPI = (T::NI + T::THREADS - 1) / T::THREADS;  // entries per thread inside the leaf (e < NI)
  constexpr int SPT = 2;                                      // slots per thread issued with the gathers
  __shared__ int s_own[T::NI];  // owned node k: its smem cell | packed interior position << 12
  // dynamic: the tile's slot sources (+ zero slot), the stencil input (chi,
  // phi) on the padded box, the interpolation weights
  extern __shared__ double2 dyn_smem[];
  double2* slotv = dyn_smem;                                    // [max_slots + 1]
  double* s_chi = reinterpret_cast<double*>(slotv + P.max_slots + 1);  // [NS]
  double* s_phi = s_chi + T::NS;                                // [NS]
  double* s_w = s_phi + T::NS;                                  // [n_wtab]
  const int64_t tile = blockIdx.x;
  const int32_t* __restrict__ tab = P.tile_table + tile * T::NE;
  // ---- 1a
  int ent[EPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = threadIdx.x + i * T::THREADS;
    ent[i] = (e < T::NE) ? __ldg(tab + e) : -1;
  }
  const int64_t sl0 = __ldg(P.tile_slot_ptr + tile), sl1 = __ldg(P.tile_slot_ptr + tile + 1);
  const int64_t j0 = __ldg(P.tile_in_ptr + tile), j1 = __ldg(P.tile_in_ptr + tile + 1);
  const int nin = (int)(j1 - j0);
  const int nslot = (int)(sl1 - sl0);
  int sg[SPT];
#pragma unroll
  for (int i = 0; i < SPT; ++i) {
    const int k = threadIdx.x + i * T::THREADS;
    sg[i] = k < nslot ? __ldg(P.slot_gid + sl0 + k) : INT32_MIN;
  }
  for (int i = threadIdx.x; i < P.n_wtab; i += T::THREADS) s_w[i] = P.wtab[i];
  if (threadIdx.x == 0) slotv[nslot] = make_double2(0.0, 0.0);  // zero slot of padding taps
  // L2 prefetch for the tile that will take this CTA slot one wave later:
  // its table, tap program and owned field ranges (compulsory DRAM misses
  // then meet that tile in L2)
  if (P.prefetch_dist > 0) {
    const int64_t nt = tile + P.prefetch_dist;
    if (nt < P.n_tiles) {
      const char* tb = reinterpret_cast<const char*>(P.tile_table + nt * T::NE);
      for (int off = threadIdx.x * 128; off < T::NE * 4; off += T::THREADS * 128) prefetch_l2(tb + off);
      const int4 nm = __ldg(reinterpret_cast<const int4*>(P.tile_meta) + nt);
      const int64_t a0 = __ldg(P.tile_tap_ptr + nt), a1 = __ldg(P.tile_tap_ptr + nt + 1);
      const char* tp = reinterpret_cast<const char*>(P.tap + a0);
      for (int64_t off = threadIdx.x * 128; off < (a1 - a0) * 4; off += T::THREADS * 128) prefetch_l2(tp + off);
      const int ncur = LTS ? P.coef->cur[(nm.z >> 8) & 0xFF] : P.gts_cur;
      const double* Un = ncur ? P.U1 : P.U0;
      const int64_t nb = (int64_t)(nm.y - nm.x) * 8;
      const int nstreams = 2 + 2 * NT;  // u chi/phi, and the verbatim K_j chi/phi
      for (int64_t w = threadIdx.x; w < nstreams * ((nb + 127) / 128); w += T::THREADS) {
        const int st = (int)(w / ((nb + 127) / 128));
        const int64_t off = (w % ((nb + 127) / 128)) * 128;
        const double* base = st < 2 ? Un + (int64_t)st * P.ld
                                    : P.K + (int64_t)P.vt_j[(st - 2) >> 1] * 2 * P.ld + ((st - 2) & 1) * P.ld;
        prefetch_l2(reinterpret_cast<const char*>(base + nm.x) + off);
      }
    }
  }
  const int4 meta = __ldg(reinterpret_cast<const int4*>(P.tile_meta) + tile);  // {g0, g1, lvl|cad<<8|faces<<16, leaf}
  const int leaf = meta.w;
  const int64_t g0 = meta.x;
  const int64_t g1 = meta.y;
  const int lvl = meta.z & 0xFF;
  const int cad = (meta.z >> 8) & 0xFF;
  const int faces = (meta.z >> 16) & 0x3F;
  const int s = P.stage;
  const int64_t n = P.ld;  // row stride of the field arrays
  const int p = P.n_stages;
  const double* U0 = P.U0;
  const double* U1 = P.U1;
  const double* K = P.K;
  const double* IB = P.ibuf;  // interface sources of this stage: chi row, then phi row
  const int64_t nib = P.n_iface_total;
  const AmrSliceCoef* C = P.coef;
  const bool phi_all = faces != 0;  // radiative rows need phi gradients: phi on the whole cross
  const int cur = LTS ? C->cur[cad] : P.gts_cur;
  const double* Ucur = cur ? U1 : U0;
  // verbatim stage sources: u at stage 0; at stage s > 0 the Y the owners wrote
  // in stage s-1 (Y = (0 + u) + sum_j dt a_sj K_j, stepper.py:290-296)
  // Y is double-buffered by stage parity: stage s reads Y[s&1], writes Y[(s+1)&1]
  const double* V = (s == 0) ? Ucur : P.Y + (int64_t)(s & 1) * 2 * n;

  // ---- 1b: every gather of this thread in flight at once: one verbatim value
  //      per copy entry and slot (chi; phi only where the stencil reads it);
  //      LTS interface entries read the transfer of the interface pass.
  double cu[EPT], pu[EPI];
  double2 su[SPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int g = ent[i];
    if (g >= 0) {
#ifdef AMR_ABLATE
      if (P.dbg_skip & 1) {  // ablation (tools/ablate.py): no field gathers
        cu[i] = 1.0;
        pu[i] = 1.0;
        continue;
      }
#endif
      cu[i] = __ldg(V + g);
      if (i < EPI && (phi_all || (g >= g0 && g < g1))) pu[i] = __ldg(V + n + g);
    } else if (LTS && g <= AMR_IFACE_BASE) {
      cu[i] = __ldg(IB + (AMR_IFACE_BASE - g));
    }
  }
#pragma unroll
  for (int i = 0; i < SPT; ++i) {
    const int g = sg[i];
    if (g >= 0) {
      su[i] = ld_pair(V, n, g);
    } else if (LTS && g != INT32_MIN) {
      su[i] = make_double2(__ldg(IB + (-g - 1)), __ldg(IB + nib + (-g - 1)));
    }
  }
  // ---- 1c
#pragma unroll
  for (int i = 0; i < EPT; ++i) {
    const int e = threadIdx.x + i * T::THREADS;
    const int g = ent[i];
    if (e >= T::NE || (g <= -2 && g > AMR_IFACE_BASE)) continue;  // hanging rows are written in 1d
    const int cell = __ldg(P.cross_cells + e);
    const bool own = e < T::NI && g >= g0 && g < g1;
    if (own) s_own[g - g0] = cell | ((int)__ldg(P.cross_pos + e) << 12);
    double yc = 0.0, yp = 0.0;
    if (g >= 0) {
      // copy row 0 + 1.0*src; at stage 0 the source itself is 0 + u
      yc = (s == 0) ? 0.0 + (0.0 + cu[i]) : 0.0 + cu[i];
      if (phi_all || own) {
        const double vp = (i < EPI) ? pu[i] : __ldg(V + n + g);  // halo phi of a face tile (rare)
        yp = (s == 0) ? 0.0 + (0.0 + vp) : 0.0 + vp;
      }
    } else if (LTS && g <= AMR_IFACE_BASE) {
      yc = 0.0 + cu[i];
      if (phi_all) yp = 0.0 + __ldg(IB + nib + (AMR_IFACE_BASE - g));
    }
    s_chi[cell] = yc;
    s_phi[cell] = yp;
  }
#pragma unroll
  for (int i = 0; i < SPT; ++i) {
    const int g = sg[i];
    if (g == INT32_MIN) continue;
    double2 y = su[i];  // interface source, or the verbatim source
    if (g >= 0 && s == 0) y = make_double2(0.0 + su[i].x, 0.0 + su[i].y);
    slotv[threadIdx.x + i * T::THREADS] = y;
  }
  for (int k = threadIdx.x + SPT * T::THREADS; k < nslot; k += T::THREADS) {  // very large interface tiles
    const int g = __ldg(P.slot_gid + sl0 + k);
    if (LTS && g < 0) {
      slotv[k] = make_double2(__ldg(IB + (-g - 1)), __ldg(IB + nib + (-g - 1)));
    } else {
      double2 y = ld_pair(V, n, g);
      if (s == 0) y = make_double2(0.0 + y.x, 0.0 + y.y);
      slotv[k] = y;
    }
  }
  __syncthreads();
  // u at this thread's owned nodes, for the epilogue: loaded now, in flight
  // during the hanging-row sums (owned node k is handled by thread k % THREADS)
  constexpr int OPT = (T::NI + T::THREADS - 1) / T::THREADS;
  double2 uo[OPT];
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int64_t g = g0 + threadIdx.x + r * T::THREADS;
    uo[r] = g < g1 ? ld_pair(Ucur, n, g) : make_double2(0.0, 0.0);
  }
  // ---- 1d: hanging rows, 0 + sum_k w_k src(g_k) in ascending-gid order
  //      (mesh.py:316-351; scipy csr_matvecs, mesh.py:418).  Rows hold a
  //      multiple of 4 taps (padding taps: weight 0 on the zero slot, which
  //      leaves the running sum unchanged), 16-byte aligned: one uint4 of tap
  //      words per 4 taps.  in_cell is the row's smem cell.
#ifdef AMR_ABLATE
  if (P.dbg_skip & 2) {  // ablation: no hanging-row sums
  } else
#endif
  if (phi_all) {
    for (int li = threadIdx.x; li < nin; li += T::THREADS) {
      const int64_t k0 = __ldg(P.in_tap_ptr + j0 + li), k1 = __ldg(P.in_tap_ptr + j0 + li + 1);
      double ax = 0.0, ay = 0.0;
      for (int64_t k = k0; k < k1; k += 4) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(P.tap + k));
        const uint32_t tq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double w = s_w[tq[u] & 0xFFFF];
          const double2 v = slotv[tq[u] >> 16];
          ax = ax + w * v.x;
          ay = ay + w * v.y;
        }
      }
      const int cell = __ldg(P.in_cell + j0 + li);
      s_chi[cell] = ax;
      s_phi[cell] = ay;
    }
  } else {
    for (int li = threadIdx.x; li < nin; li += T::THREADS) {
      const int64_t k0 = __ldg(P.in_tap_ptr + j0 + li), k1 = __ldg(P.in_tap_ptr + j0 + li + 1);
      double ax = 0.0;
      for (int64_t k = k0; k < k1; k += 4) {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(P.tap + k));
        const uint32_t tq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) ax = ax + s_w[tq[u] & 0xFFFF] * slotv[tq[u] >> 16].x;
      }
      const int cell = __ldg(P.in_cell + j0 + li);
      s_chi[cell] = ax;
      s_phi[cell] = 0.0;
    }
  }
  __syncthreads();

  // ---- 2: RHS at the owned nodes, K_s (and the RK combine) out
  const Weights& W = P;
  RhsConst R;
  R.h = P.h[lvl];
  R.h2 = P.h2[lvl];
  R.inv_h2 = P.inv_h2[lvl];
  R.pow2 = P.h2_pow2[lvl] != 0;
  R.r_eps = P.r_eps;
  R.r_eps2 = P.r_eps2;
  R.k_chi = P.k_chi;
  R.k_phi = P.k_phi;
  R.f0_chi = P.f0_chi;
  R.f0_phi = P.f0_phi;
  R.nonlinear = P.nonlinear;
  constexpr int scale = PPO - 1;
  const bool need_x = faces != 0 || P.nonlinear == 1;  // radiative rows / sin(2chi)/r^2 need coordinates
  const bool fast_rhs = !need_x;
  const int64_t side_len = (int64_t)1 << (P.max_depth - lvl);
  int32_t anc[3] = {0, 0, 0};
  if (need_x) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) anc[d] = P.leaf_anchor[leaf * 3 + d];
  }
  const bool last = (s == p - 1);
  double* Unew = cur ? P.U0 : P.U1;
  double* Ks = P.K + (int64_t)s * 2 * n;
#ifdef AMR_ABLATE
  const int n_own = (P.dbg_skip & 4) ? 0 : (int)(g1 - g0);  // ablation: no RHS / epilogue
#else
  const int n_own = (int)(g1 - g0);
#endif
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = threadIdx.x + r * T::THREADS;
    if (k >= n_own) break;
    const int q = s_own[k];
    const int cell = q & 0xFFF;
    int pos[3];
#pragma unroll
    for (int d = 0; d < DIM; ++d) pos[d] = (q >> (12 + 4 * d)) & 15;
    double x[3] = {0.0, 0.0, 0.0};
    if (need_x) {
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const int64_t lat = (int64_t)anc[d] * scale + side_len * pos[d];
        x[d] = P.lo[d] + ((double)lat / (double)P.top_nodes) * P.extent[d];
      }
    }
    SmemAcc<DIM, PPO> acc{s_chi, s_phi, cell};
    const double2 ks = fast_rhs ? rhs_interior<DIM>(acc, W, R) : rhs_point<DIM>(acc, pos, PPO, faces, x, W, R);
    const int64_t g = g0 + k;
    if (!last || LTS) {
      Ks[g] = ks.x;
      Ks[n + g] = ks.y;
    }
    if (!last) {  // next stage's verbatim source of this owned node
      double yx = 0.0 + uo[r].x, yy = 0.0 + uo[r].y;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int j = P.vt_j[t];
        const double c = LTS ? C->cstage[cad][s + 1][j] : P.g_cstage[s + 1][j];
        const double kx = (j == s) ? ks.x : __ldg(K + (int64_t)j * 2 * n + g);
        const double ky = (j == s) ? ks.y : __ldg(K + (int64_t)j * 2 * n + n + g);
        yx = yx + c * kx;
        yy = yy + c * ky;
      }
      double* Yout = P.Y + (int64_t)((s + 1) & 1) * 2 * n;
      Yout[g] = yx;
      Yout[n + g] = yy;
    }
    if (last) {
      double ux = 0.0 + uo[r].x, uy = 0.0 + uo[r].y;
      for (int j = 0; j < p; ++j) {
        const double c = LTS ? C->comb[cad][j] : P.g_comb[j];
        if (c == 0.0) continue;
        const double kx = (j == s) ? ks.x : __ldg(K + (int64_t)j * 2 * n + g);
        const double ky = (j == s) ? ks.y : __ldg(K + (int64_t)j * 2 * n + n + g);
        ux = ux + c * kx;
        uy = uy + c * ky;
      }
      Unew[g] = ux;
      Unew[n + g] = uy;
    }
  }
}

#include "amr_stage_pipe.cuh"
#include "amr_stage_blob.cuh"
#include "amr_stage_cross.cuh"

// --------------------------------------------------------------------------
// Mesh.unzip over CSR rows
// --------------------------------------------------------------------------
__global__ void gather_rows_kernel(int64_t n_rows, const int64_t* __restrict__ ptr,
                                   const int64_t* __restrict__ col, const double* __restrict__ val, int nv,
                                   const double* __restrict__ z, int64_t zs, double* __restrict__ out,
                                   int64_t os) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_rows * nv) return;
  int64_t r = t % n_rows;
  int v = (int)(t / n_rows);
  double acc = 0.0;
  for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) acc = acc + val[k] * z[v * zs + col[k]];
  out[v * os + r] = acc;
}

// --------------------------------------------------------------------------
// wave_rhs on one padded block (API path)
// --------------------------------------------------------------------------
template <int DIM>
struct GlobalAcc {
  const double* y;
  int np, pad, cell;
  int64_t var_stride;
  __device__ __forceinline__ double at(int v, int d, int o) const {
    int stride = (DIM == 3) ? (d == 0 ? np * np : (d == 1 ? np : 1)) : (d == 0 ? np : 1);
    return y[v * var_stride + cell + o * stride];
  }
};

template <int DIM>
__global__ void block_rhs_kernel(int n, int pad, const double* __restrict__ y, double* __restrict__ out,
                                 RhsConst R, const double* __restrict__ coords, int faces,
                                 const AmrStageParams P) {
  int64_t total = 1;
  for (int d = 0; d < DIM; ++d) total *= n;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= total) return;
  int pos[3];
  int64_t r = t;
  for (int d = DIM - 1; d >= 0; --d) {
    pos[d] = (int)(r % n);
    r /= n;
  }
  int np = n + 2 * pad;
  int cell = 0;
  for (int d = 0; d < DIM; ++d) cell = cell * np + (pos[d] + pad);
  int64_t vs = 1;
  for (int d = 0; d < DIM; ++d) vs *= np;
  double x[3];
  for (int d = 0; d < DIM; ++d) x[d] = coords[d * n + pos[d]];
  const Weights& W = P;
  GlobalAcc<DIM> acc{y, np, pad, cell, vs};
  double2 v = rhs_point<DIM>(acc, pos, n, faces, x, W, R);
  out[t] = v.x;
  out[total + t] = v.y;
}

__global__ void pack_kernel(int64_t n_ranges, const int64_t* __restrict__ start,
                            const int64_t* __restrict__ len, const int64_t* __restrict__ off, int width,
                            const double* __restrict__ src, double* __restrict__ buf, int64_t total,
                            bool unpack) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= total) return;
  int64_t node = t / width, c = t % width;
  // binary search the range holding `node` (off = exclusive prefix of len)
  int64_t lo = 0, hi = n_ranges - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if (off[mid] <= node) lo = mid; else hi = mid - 1;
  }
  int64_t g = start[lo] + (node - off[lo]);
  if (!unpack) buf[t] = src[g * width + c];
  else const_cast<double*>(src)[g * width + c] = buf[t];
}

template <int DIM, int PPO, bool LTS, int NT>
int launch_stage_one(const AmrStageParams* p, cudaStream_t st) {
  using T = Tile<DIM, PPO>;
  const size_t dyn = sizeof(double2) * (size_t)(p->max_slots + 1) + sizeof(double) * (size_t)(2 * T::NS + p->n_wtab);
  static size_t configured = 0;
  if (dyn > configured) {
    cudaError_t e = cudaFuncSetAttribute(stage_kernel<DIM, PPO, LTS, NT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(stage_kernel)");
    configured = dyn;
  }
  // L2 prefetch distance: one wave of resident CTAs (AMR_PREFETCH=0 disables)
  static int wave = -1;
  if (wave < 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage_kernel<DIM, PPO, LTS, NT>, T::THREADS, dyn);
    const char* env = std::getenv("AMR_PREFETCH");
    wave = (env && std::atoi(env) == 0) ? 0 : sms * (per_sm > 0 ? per_sm : 1);
  }
  AmrStageParams q = *p;
  q.prefetch_dist = p->prefetch_dist < 0 ? wave : p->prefetch_dist;
  stage_kernel<DIM, PPO, LTS, NT><<<(unsigned)p->n_tiles, T::THREADS, dyn, st>>>(q);
  return AMR_OK;
}

template <int DIM, int PPO, bool LTS, int NT>
int launch_pipe_one(const AmrStageParams* p, cudaStream_t st) {
  using PP = Pipe<DIM, PPO>;
  const size_t dyn = PP::smem_bytes(p->max_slots, p->max_blob);
  static size_t configured = 0;
  static size_t occ_dyn = 0;
  static int grid_cap = 0;
  if (dyn > configured) {
    cudaError_t e = cudaFuncSetAttribute(stage_pipe<DIM, PPO, LTS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)dyn);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(stage_pipe)");
    configured = dyn;
  }
  if (dyn != occ_dyn) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage_pipe<DIM, PPO, LTS, NT>, PP::THREADS, dyn);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy(stage_pipe)");
    if (per_sm <= 0) {
      amr_set_error_internal("stage_pipe: tile program does not fit in shared memory");
      return AMR_EINVAL;
    }
    grid_cap = sms * per_sm;
    occ_dyn = dyn;
  }
  const int64_t grid = p->n_tiles < grid_cap ? p->n_tiles : grid_cap;
  stage_pipe<DIM, PPO, LTS, NT><<<(unsigned)grid, PP::THREADS, dyn, st>>>(*p);
  return AMR_OK;
}

template <int DIM, int PPO, bool LTS, int NT>
int launch_blob_one(const AmrStageParams* p, cudaStream_t st) {
  using BK = BlobK<DIM, PPO>;
  const size_t dyn = BK::smem_bytes(p->max_slots, p->max_blob);
  static size_t configured = 0;
  if (dyn > configured) {
    cudaError_t e = cudaFuncSetAttribute(stage_blob<DIM, PPO, LTS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)dyn);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(stage_blob)");
    configured = dyn;
  }
  // L2 prefetch distance: one wave of resident CTAs (AMR_PREFETCH=0 disables)
  static int wave = -1;
  if (wave < 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stage_blob<DIM, PPO, LTS, NT>, BK::THREADS, dyn);
    const char* env = std::getenv("AMR_PREFETCH");
    wave = (env && std::atoi(env) == 0) ? 0 : sms * (per_sm > 0 ? per_sm : 1);
  }
  AmrStageParams q = *p;
  q.prefetch_dist = p->prefetch_dist < 0 ? wave : p->prefetch_dist;
  stage_blob<DIM, PPO, LTS, NT><<<(unsigned)p->n_tiles, BK::THREADS, dyn, st>>>(q);
  return AMR_OK;
}

template <int DIM, int PPO, bool LTS, int NT, int NTH>
int launch_cross_one(const AmrStageParams* p, cudaStream_t st) {
  using CK = CrossK<DIM, PPO>;
  const size_t dyn = CK::smem_bytes(p->max_slots, p->max_blob);
  int dev = 0;
  cudaGetDevice(&dev);
  static size_t configured[64] = {0};
  if (dev < 64 && dyn > configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(stage_cross<DIM, PPO, LTS, NT, NTH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(stage_cross)");
    configured[dev] = dyn;
  }
  stage_cross<DIM, PPO, LTS, NT, NTH><<<(unsigned)p->n_tiles, NTH, dyn, st>>>(*p);
  return AMR_OK;
}

template <int DIM, int PPO, bool LTS, int NTH>
int launch_cross_nt(const AmrStageParams* p, cudaStream_t st) {
  switch (p->n_vt) {
    case 0: return launch_cross_one<DIM, PPO, LTS, 0, NTH>(p, st);
    case 1: return launch_cross_one<DIM, PPO, LTS, 1, NTH>(p, st);
    case 2: return launch_cross_one<DIM, PPO, LTS, 2, NTH>(p, st);
    case 3: return launch_cross_one<DIM, PPO, LTS, 3, NTH>(p, st);
    default: return AMR_EINVAL;
  }
}

template <int DIM, int PPO, bool LTS>
int launch_stage_nt(const AmrStageParams* p, cudaStream_t st) {
  if (p->kernel == 3) {
    if (p->threads == 256) return launch_cross_nt<DIM, PPO, LTS, 256>(p, st);
    return launch_cross_nt<DIM, PPO, LTS, 128>(p, st);
  }
  if (p->kernel == 2) {
    switch (p->n_vt) {
      case 0: return launch_blob_one<DIM, PPO, LTS, 0>(p, st);
      case 1: return launch_blob_one<DIM, PPO, LTS, 1>(p, st);
      case 2: return launch_blob_one<DIM, PPO, LTS, 2>(p, st);
      case 3: return launch_blob_one<DIM, PPO, LTS, 3>(p, st);
      default: return AMR_EINVAL;
    }
  }
  if (p->kernel == 1) {
    switch (p->n_vt) {
      case 0: return launch_pipe_one<DIM, PPO, LTS, 0>(p, st);
      case 1: return launch_pipe_one<DIM, PPO, LTS, 1>(p, st);
      case 2: return launch_pipe_one<DIM, PPO, LTS, 2>(p, st);
      case 3: return launch_pipe_one<DIM, PPO, LTS, 3>(p, st);
      default: return AMR_EINVAL;
    }
  }
  switch (p->n_vt) {
    case 0: return launch_stage_one<DIM, PPO, LTS, 0>(p, st);
    case 1: return launch_stage_one<DIM, PPO, LTS, 1>(p, st);
    case 2: return launch_stage_one<DIM, PPO, LTS, 2>(p, st);
    case 3: return launch_stage_one<DIM, PPO, LTS, 3>(p, st);
    default: return AMR_EINVAL;
  }
}

template <int DIM, int PPO>
int launch_stage_t(const AmrStageParams* p, cudaStream_t st) {
  if (p->n_tiles <= 0) return AMR_OK;
  int rc = p->lts ? launch_stage_nt<DIM, PPO, true>(p, st) : launch_stage_nt<DIM, PPO, false>(p, st);
  if (rc) return rc;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "amr_stage launch");
}

}  // namespace

extern "C" int amr_stage(const AmrStageParams* p, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (p->pad != 2) return AMR_EINVAL;
  if (p->n_stages < 1 || p->n_stages > AMR_MAXP || p->stage < 0 || p->stage >= p->n_stages) return AMR_EINVAL;
  if (p->dim == 2) {
    if (p->ppo == 5) return launch_stage_t<2, 5>(p, st);
    if (p->ppo == 7) return launch_stage_t<2, 7>(p, st);
    if (p->ppo == 9) return launch_stage_t<2, 9>(p, st);
  } else if (p->dim == 3) {
    if (p->ppo == 5) return launch_stage_t<3, 5>(p, st);
    if (p->ppo == 7) return launch_stage_t<3, 7>(p, st);
    if (p->ppo == 9) return launch_stage_t<3, 9>(p, st);
  }
  amr_set_error_internal("amr_stage: unsupported (dim, ppo)");
  return AMR_EINVAL;
}

extern "C" int amr_iface(const AmrStageParams* p, void* stream) {
  if (p->n_iface <= 0) return AMR_OK;
  iface_kernel<<<(unsigned)((p->n_iface + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "amr_iface launch");
}

extern "C" int amr_gather_rows(int64_t n_rows, const int64_t* row_ptr, const int64_t* col, const double* val,
                               int nv, const double* z, int64_t z_stride, double* out, int64_t out_stride,
                               void* stream) {
  int64_t total = n_rows * nv;
  if (total == 0) return AMR_OK;
  unsigned blocks = (unsigned)((total + 255) / 256);
  gather_rows_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_rows, row_ptr, col, val, nv, z, z_stride, out,
                                                               out_stride);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "amr_gather_rows launch");
}

extern "C" int amr_block_rhs(int dim, int n, int pad, const double* y, double* out, double h, double h2,
                             const double* coords, double r_eps, int faces, int nonlinear, double k_chi,
                             double k_phi, double f0_chi, double f0_phi, const AmrStageParams* weights,
                             void* stream) {
  RhsConst R;
  R.h = h;
  R.h2 = h2;
  R.inv_h2 = 0.0;
  R.pow2 = false;
  R.r_eps = r_eps;
  R.r_eps2 = weights->r_eps2;
  R.k_chi = k_chi;
  R.k_phi = k_phi;
  R.f0_chi = f0_chi;
  R.f0_phi = f0_phi;
  R.nonlinear = nonlinear;
  int64_t total = 1;
  for (int d = 0; d < dim; ++d) total *= n;
  if (total == 0) return AMR_OK;
  unsigned blocks = (unsigned)((total + 127) / 128);
  cudaStream_t st = (cudaStream_t)stream;
  if (dim == 2)
    block_rhs_kernel<2><<<blocks, 128, 0, st>>>(n, pad, y, out, R, coords, faces, *weights);
  else if (dim == 3)
    block_rhs_kernel<3><<<blocks, 128, 0, st>>>(n, pad, y, out, R, coords, faces, *weights);
  else
    return AMR_EINVAL;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "amr_block_rhs launch");
}

extern "C" int amr_pack_ranges(int64_t n_ranges, const int64_t* range_start, const int64_t* range_len,
                               const int64_t* range_off, int width, const double* src, double* buf,
                               int64_t total, void* stream) {
  if (total <= 0) return AMR_OK;
  unsigned blocks = (unsigned)((total * width + 255) / 256);
  pack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_ranges, range_start, range_len, range_off, width,
                                                        src, buf, total * width, false);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "amr_pack_ranges launch");
}

extern "C" int amr_unpack_ranges(int64_t n_ranges, const int64_t* range_start, const int64_t* range_len,
                                 const int64_t* range_off, int width, const double* buf, double* dst,
                                 int64_t total, void* stream) {
  if (total <= 0) return AMR_OK;
  unsigned blocks = (unsigned)((total * width + 255) / 256);
  pack_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(n_ranges, range_start, range_len, range_off, width,
                                                        dst, const_cast<double*>(buf), total * width, true);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "amr_unpack_ranges launch");
}
