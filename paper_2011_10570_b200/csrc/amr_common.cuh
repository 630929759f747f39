// amr_common.cuh — device code shared by the stage-kernel instances
// (amr_stage_inst.cu) and the API kernels (amr_kernels.cu): tile geometry,
// the LTS stage-source transfer, and the reference's finite-difference rows.
// Everything is in an anonymous namespace (one copy per translation unit).
#pragma once
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

template <int DIM, int PPO>
struct Tile {
  static constexpr int PAD = 2;
  static constexpr int NP = PPO + 2 * PAD;
  static constexpr int NI = cpow(PPO, DIM);
  static constexpr int NF = cpow(PPO, DIM - 1);
  static constexpr int NS = cpow(NP, DIM);
  // stencil box in shared memory: rows (last axis) of RS >= NP doubles
  // (tileprog.py box_strides() is the host copy).  Padding rows to 24 puts the
  // two 8-node z-lines of a half-warp 8 banks apart (no bank conflicts), but
  // measured no faster on cfg2 (34.2 vs 34.9 G upd/s LTS): the box stays dense
#ifndef AMR_RS
#define AMR_RS 13
#endif
  static constexpr int RS = AMR_RS > NP ? AMR_RS : NP;
  static constexpr int BOX = cpow(NP, DIM - 1) * RS;
};


// Fields are SoA, the reference's (nvars, n_nodes) zip layout: var v of node g
// at base[v*n + g]; stage j of K at K + j*2n.
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

// Launch with programmatic stream serialization (PDL): the kernel may start
// before the previous kernel on the stream has finished and must call
// griddepcontrol.wait before touching that kernel's output.  AMR_PDL=0 turns
// it off (plain stream order).
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = std::getenv("AMR_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

template <class Kern, class Params>
int pdl_launch(Kern kern, dim3 grid, dim3 block, size_t dyn, cudaStream_t st, const Params& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "cudaLaunchKernelEx");
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

}  // namespace
