// amr_kernels.cu — sm_100a kernels of the B200 LTS/GTS wave solver.
//
// Hot path: amr_stage (amr_stage_cross.cuh).  One CTA owns one leaf tile and
// computes the RHS at the zip nodes the leaf owns.  Per RK stage it
//   1. gathers the tile's stage input on its owned cross into shared memory:
//      copies of zip nodes, sorted interpolation rows (Mesh.unzip,
//      mesh.py:413-420), and at LTS level interfaces the stage sources that
//      iface_kernel formed from the transfer matrices (Engine._stage_source,
//      stepper.py:274-314);
//   2. evaluates the 4th-order RHS (biased rows and radiative overwrite at
//      physical faces; linear, sin or cubic source; wave.py:147-201) and
//      writes K_s for the owned nodes contiguously (the zip of
//      stepper.py:422-429) together with the next stage's verbatim source;
//   3. on the last stage does the RK combine u_new = u + sum dt w_s K_s into
//      the other u buffer (record rotation u_pre <- u_curr without a copy: the
//      live buffer of a leaf is the parity of its step count).
//
// Arithmetic follows the reference bit for bit: -fmad=false for the whole
// file, numpy's operation order, the reference's Fornberg weight arrays, and
// fma() only where the reference goes through OpenBLAS dgemm (np.tensordot at
// stepper.py:264,305 — an ascending-k FMA chain on the generating host).
#include "amr_common.cuh"

#include <cstddef>

namespace {

// LTS interface pass: the stage source of every (zip node, reader cadence)
// pair whose step size or time differs from the reader's (delta=0 transfer or
// virtual substep + transfer, stepper.py:256-314), once per stage, so the
// stage kernel reads it like a copy.  Pairs are sorted finest reader first:
// the eligible readers of a slice are a prefix.  The buffer holds one slab per
// stage, [stage][var][pair].  A pair whose source is not stepping at this slice
// (virtual substep, mode 2) depends on nothing the slice computes, so the
// stage-0 launch (if_phase 1) fills all its stages at once — the source's u_pre
// and K are read once instead of once per stage — and the later launches
// (if_phase 2) skip it; a slice where only one cadence steps needs no later
// launch at all.
__global__ void __launch_bounds__(256) iface_kernel(const AmrStageParams P) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // the stage kernel may fetch its tile heads meanwhile
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= P.n_iface) return;
  const int g = __ldg(P.if_gid + i);
  const int cc = __ldg(P.if_cad + i);  // reader cadence | source cadence << 8 (no dependent lookup)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");              // the fields are the previous stage kernel's output
  const int lr = cc & 0xFF, ls = cc >> 8;
  const AmrSliceCoef* C = P.coef;
  const int64_t N = P.n_iface_total;
  const int mode = C->mode[lr][ls];
  if (P.if_phase != 0 && mode == 2) {
    if (P.if_phase == 2) return;  // filled by the stage-0 launch
    const int p = P.n_stages;
    const int64_t n = P.ld;
    double2 kk[AMR_MAXP];
#pragma unroll
    for (int k = 0; k < AMR_MAXP; ++k)
      kk[k] = (k < p) ? ld_pair(P.K + (int64_t)k * 2 * n, n, g) : make_double2(0.0, 0.0);
    double2 y0 = ld_pair(C->cur[ls] ? P.U0 : P.U1, n, g);  // u_pre: the virtual substep starts there
    const double(*Mv)[AMR_MAXP] = C->Mv[lr][ls];
#pragma unroll
    for (int a = 0; a < AMR_MAXP; ++a) {
      if (a >= p) break;
      const double c = C->dtw[lr][ls][a];
      if (c == 0.0) continue;
      double ax = 0.0, ay = 0.0;
#pragma unroll
      for (int k = 0; k <= a; ++k) {
        ax = fma(Mv[a][k], kk[k].x, ax);
        ay = fma(Mv[a][k], kk[k].y, ay);
      }
      y0.x = y0.x + c * ax;
      y0.y = y0.y + c * ay;
    }
    const double(*M)[AMR_MAXP] = C->M[lr][ls];
    double2 mk[AMR_MAXP];  // (M K)_j, shared by the stages
#pragma unroll
    for (int j = 0; j < AMR_MAXP; ++j) {
      double ax = 0.0, ay = 0.0;
      if (j < p - 1) {
#pragma unroll
        for (int k = 0; k < AMR_MAXP; ++k) {
          if (k > p - 1) break;
          ax = fma(M[j][k], kk[k].x, ax);
          ay = fma(M[j][k], kk[k].y, ay);
        }
      }
      mk[j] = make_double2(ax, ay);
    }
#pragma unroll
    for (int s = 0; s < AMR_MAXP; ++s) {
      if (s >= p) break;
      double2 y = y0;
#pragma unroll
      for (int j = 0; j < AMR_MAXP; ++j) {
        if (j >= s) break;
        const double c = C->cstage[lr][s][j];
        if (c == 0.0) continue;
        y.x = y.x + c * mk[j].x;
        y.y = y.y + c * mk[j].y;
      }
      P.ibuf0[(int64_t)(2 * s) * N + i] = y.x;
      P.ibuf0[(int64_t)(2 * s + 1) * N + i] = y.y;
    }
    return;
  }
  const double2 v = lts_source(P.U0, P.U1, P.K, P.ld, P.n_stages, g, P.stage, lr, ls, C);
  P.ibuf0[(int64_t)(2 * P.stage) * N + i] = v.x;
  P.ibuf0[(int64_t)(2 * P.stage + 1) * N + i] = v.y;
}


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

// Ghost records between ranks: whole-leaf zip ranges <-> one packed buffer
// buf[row][node].  One thread per packed node; its range by binary search in
// the exclusive prefix `off`.  A range's rows come from the parity-0 or the
// parity-1 base pointers according to its cadence (the u buffers; K and Y rows
// pass the same pointer twice).
template <bool UNPACK>
__global__ void __launch_bounds__(256) ghost_move_kernel(const AmrGhostMove M, double* __restrict__ buf) {
  const int64_t node = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (node >= M.total) return;
  int64_t lo = 0, hi = M.n_ranges - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(M.off + mid) <= node) lo = mid; else hi = mid - 1;
  }
  const int64_t g = __ldg(M.start + lo) + (node - __ldg(M.off + lo));
  const int par = M.par[__ldg(M.cad + lo) & (AMR_MAXL - 1)];
  const int64_t bld = M.buf_ld > 0 ? M.buf_ld : M.total;
#pragma unroll
  for (int r = 0; r < AMR_GHOST_ROWS; ++r) {
    if (r >= M.n_rows) break;
    double* row = par ? M.row1[r] : M.row0[r];
    if (UNPACK) row[g] = buf[(int64_t)r * bld + node];
    else buf[(int64_t)r * bld + node] = row[g];
  }
}

}  // namespace

// stage-kernel instances, one translation unit each (amr_stage_inst.cu)
#define AMR_DECL(D, P)                                                       \
  int amr_stage_launch_##D##_##P##_g(const AmrStageParams*, cudaStream_t); \
  int amr_stage_launch_##D##_##P##_l(const AmrStageParams*, cudaStream_t);
AMR_DECL(2, 5) AMR_DECL(2, 7) AMR_DECL(2, 9) AMR_DECL(3, 5) AMR_DECL(3, 7) AMR_DECL(3, 9)
#undef AMR_DECL

extern "C" int amr_stage(const AmrStageParams* p, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (p->pad != 2) return AMR_EINVAL;
  if (p->n_stages < 1 || p->n_stages > AMR_MAXP || p->stage < 0 || p->stage >= p->n_stages) return AMR_EINVAL;
  if (p->n_tiles <= 0) return AMR_OK;
  int rc = AMR_EINVAL;
#define AMR_CASE(D, P)                                                                            \
  if (p->dim == D && p->ppo == P)                                                                 \
    rc = p->lts ? amr_stage_launch_##D##_##P##_l(p, st) : amr_stage_launch_##D##_##P##_g(p, st); \
  else
  AMR_CASE(2, 5) AMR_CASE(2, 7) AMR_CASE(2, 9) AMR_CASE(3, 5) AMR_CASE(3, 7) AMR_CASE(3, 9) {
    amr_set_error_internal("amr_stage: unsupported (dim, ppo)");
    return AMR_EINVAL;
  }
#undef AMR_CASE
  if (rc) return rc;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, "amr_stage launch");
}

// struct layout of AmrStageParams as compiled (checked against the ctypes
// mirror by tests/test_native_abi.py): sizeof, then the offsets of AMR_LAYOUT_FIELDS
#define AMR_LAYOUT_FIELDS(X) \
  X(n_tiles) X(heads) X(max_tail) X(probe) X(wtab) X(n_iface) X(ibuf) X(vt_j) X(Y) X(coef) X(g_cstage) \
  X(g_comb) X(max_depth) X(top_nodes) X(lo) X(h2_pow2) X(inv_h2) X(r_eps) X(f0_phi) X(d2c) X(d1e1)
extern "C" int amr_stage_params_layout(int64_t* out, int cap) {
  int i = 0;
  if (i < cap) out[i++] = (int64_t)sizeof(AmrStageParams);
#define AMR_OFF(f) \
  if (i < cap) out[i++] = (int64_t)offsetof(AmrStageParams, f);
  AMR_LAYOUT_FIELDS(AMR_OFF)
#undef AMR_OFF
  return i;
}

extern "C" int amr_iface(const AmrStageParams* p, void* stream) {
  if (p->n_iface <= 0) return AMR_OK;
  return pdl_launch(iface_kernel, dim3((unsigned)((p->n_iface + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, *p);
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

static int ghost_move(const AmrGhostMove* m, double* buf, void* stream, bool unpack) {
  if (m->total <= 0 || m->n_ranges <= 0 || m->n_rows <= 0) return AMR_OK;
  if (m->n_rows > AMR_GHOST_ROWS) return AMR_EINVAL;
  const unsigned blocks = (unsigned)((m->total + 255) / 256);
  if (unpack)
    ghost_move_kernel<true><<<blocks, 256, 0, (cudaStream_t)stream>>>(*m, buf);
  else
    ghost_move_kernel<false><<<blocks, 256, 0, (cudaStream_t)stream>>>(*m, buf);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? AMR_OK : cuda_fail(e, unpack ? "amr_ghost_unpack launch" : "amr_ghost_pack launch");
}

extern "C" int amr_ghost_pack(const AmrGhostMove* m, double* buf, void* stream) {
  return ghost_move(m, buf, stream, false);
}

extern "C" int amr_ghost_unpack(const AmrGhostMove* m, const double* buf, void* stream) {
  return ghost_move(m, const_cast<double*>(buf), stream, true);
}
