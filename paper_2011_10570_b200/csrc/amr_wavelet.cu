// amr_wavelet.cu — sm_100a kernel for the interpolation-residual ("wavelet")
// refinement coefficient of many octants at once (wavelet.py:70-144).
//
// Per octant the reference samples a field on an odd npd^D closed tensor
// grid, rebuilds it from the even-index nodes with sliding 4-point Lagrange
// windows one axis after the other (np.tensordot per axis, wavelet.py:94-97),
// and takes the max |value - reconstruction| over nodes with at least one odd
// index (wavelet.py:98-103).  The refine/keep/coarsen decision
// (wavelet.py:108-124) or the construction predicate (wavelet.py:127-144) is
// applied in the same launch.
//
// Layout: values [n][npd^D] fp64, last axis fastest (meshgrid "ij"), so one
// octant is one contiguous run that one warp streams in with coalesced loads.
// Work per octant is ~4*npd^D flops against 8*npd^D bytes: HBM-bound, so a
// warp per octant, as many warps resident per SM as shared memory allows,
// and no tensor cores.
//
// Bit parity: each reconstructed value is an np.tensordot output.  On the
// generating host that is OpenBLAS dgemm, whose outputs equal an ascending
// FMA chain from 0 over the full coarse axis (zeros included) — verified
// against the reference in tests/test_wavelet.py.  The file is compiled with
// -fmad=false; fma() appears only there.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/amr_b200.h"

extern "C" void amr_set_error_internal(const char* msg);

namespace {

constexpr int WV_MAX_NPD = 15;
#ifndef WV_MINB  // resident 256-thread CTAs per SM the 3D npd<=7 kernels are register-capped for
#define WV_MINB 2
#endif
#ifndef WV_U2  // unroll of the 3D axis-1 / axis-2 line loops
#define WV_U2 2
#endif
#ifndef WV_U3
#define WV_U3 2
#endif
constexpr int kUnroll2 = WV_U2, kUnroll3 = WV_U3;
#ifndef WV_NACC  // partial maxima per lane in the 3D residual pass
#define WV_NACC 1
#endif
#ifndef WV_SPLIT1  // 3D axis-0 pass over both half-warps when nc^2 <= 16
#define WV_SPLIT1 0
#endif
#ifndef WV_INTMAX  // 1: residual max on the |d| bit patterns; 0: fmax + a NaN flag
#define WV_INTMAX 1
#endif


// W per npd, back to back in constant memory (npd = 3, 5, ..., 15): the 3D
// path reads it with warp-uniform indices.  Filled before each launch.
constexpr int WV_CONST_TOTAL = 3 * 2 + 5 * 3 + 7 * 4 + 9 * 5 + 11 * 6 + 13 * 7 + 15 * 8;
__constant__ double cW[WV_CONST_TOTAL];
template <int NPD>
struct WvOff {
  static constexpr int value = NPD <= 3 ? 0 : WvOff<NPD - 2>::value + (NPD - 2) * ((NPD - 1) / 2);
};
template <>
struct WvOff<3> {
  static constexpr int value = 0;
};

template <int DIM, int NPD>
struct WvShape {
  static constexpr int NC = (NPD + 1) / 2;
  static constexpr int NV = DIM == 2 ? NPD * NPD : NPD * NPD * NPD;
  static constexpr int N1 = DIM == 2 ? NPD * NC : NPD * NC * NC;  // after axis 0
  static constexpr int N2 = DIM == 2 ? 0 : NPD * NPD * NC;        // after axis 1 (3D)
  static constexpr int PER_WARP = 2 * NV + N1 + N2;
  static constexpr int NW = NPD * NC;
  static constexpr int MINB = DIM == 3 && NPD <= 7 ? WV_MINB : 1;
};

// One warp per octant; the next octant's samples are copied (cp.async) into
// a second shared buffer while the current one is reduced, so each warp keeps
// one octant's HBM read in flight.  NPD is a template parameter: every index
// division is by a constant and every chain is unrolled.
template <int DIM, int NPD>
__global__ void __launch_bounds__(256, WvShape<DIM, NPD>::MINB) wavelet_kernel(int64_t n, const double* __restrict__ V,
                                                      const double* __restrict__ Wg, const int32_t* __restrict__ levels,
                                                      int mode, double tol, double coarsen_thr, int min_level,
                                                      int max_level, double* __restrict__ coeff,
                                                      int8_t* __restrict__ flags) {
  using S = WvShape<DIM, NPD>;
  constexpr int nc = S::NC, npd = NPD, nv = S::NV;
  extern __shared__ double sm[];
  const int warps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* W = sm;  // [npd][nc]
  for (int i = threadIdx.x; i < S::NW; i += blockDim.x) W[i] = Wg[i];
  double* vb = sm + S::NW + warp * S::PER_WARP;  // two sample buffers
  double* r1 = vb + 2 * nv;
  double* r2 = r1 + S::N1;
  __syncthreads();

  // Samples move HBM -> shared memory by cp.async (no register staging), one
  // octant ahead: while octant j is reduced from one buffer, octant j+stride
  // lands in the other.
  const int64_t stride = (int64_t)gridDim.x * warps;
  int64_t oct = (int64_t)blockIdx.x * warps + warp;
  auto issue = [&](int64_t o, double* dst) {
    if (o < n) {
      const double* src = V + o * nv;
      for (int i = lane; i < nv; i += 32) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + i);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src + i) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  issue(oct, vb);
  for (int cur = 0; oct < n; oct += stride, cur ^= 1) {
    issue(oct + stride, vb + (cur ^ 1) * nv);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    const double* v = vb + cur * nv;
    __syncwarp();
    // max of |v - rec| over odd nodes: every term is >= +0, so the running
    // max starts at 0 and needs no "first term" state; NaN (np.max
    // propagates it) is tracked apart so the max itself is a plain fmax
    double m = 0.0;
    bool bad = false;
    unsigned long long mb = 0ull;
    unsigned long long mbk[WV_NACC];  // independent partial maxima: short dependency chains
#pragma unroll
    for (int q = 0; q < WV_NACC; ++q) mbk[q] = 0ull;
    if (DIM == 2) {
      // r1[i][b] = sum_a W[i][a] * v[2a][2b]   (axis 0)
#pragma unroll
      for (int t0 = 0; t0 < S::N1; t0 += 32) {
        const int t = t0 + lane;
        if (t < S::N1) {
          const int i = t / nc, b = t - i * nc;
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < nc; ++a) acc = fma(W[i * nc + a], v[(2 * a) * npd + 2 * b], acc);
          r1[t] = acc;
        }
      }
      __syncwarp();
      // rec[i][j] = sum_b W[j][b] * r1[i][b]   (axis 1), odd nodes only
#pragma unroll
      for (int t0 = 0; t0 < nv; t0 += 32) {
        const int t = t0 + lane;
        const int i = t / npd, j = t - i * npd;
        if (t < nv && ((i | j) & 1)) {
          double acc = 0.0;
#pragma unroll
          for (int b = 0; b < nc; ++b) acc = fma(W[j * nc + b], r1[i * nc + b], acc);
          const double d = fabs(v[t] - acc);
          m = fmax(m, d);
          bad |= d != d;
        }
      }
    } else {
      // 3D as 1-D lines: a lane owns one line along the axis being rebuilt,
      // holds its nc coarse inputs in registers and emits the npd outputs
      // with compile-time output index, so W[i][a] is a warp-uniform
      // constant-bank operand (cW) and no index is divided at run time.
      const double* Wc = cW + WvOff<NPD>::value;
      // Lines past the end are clamped onto the last line (a duplicate
      // result, harmless for the stores and for the max), so no lane diverges.
      // axis 0: r1[i][b][c] = sum_a W[i][a] * v[2a][2b][2c]; lines (b, c)
      if (WV_SPLIT1 && 2 * nc * nc <= 32) {
        // nc^2 <= 16 lines: both half-warps take every line, each emits half
        // of the outputs (i = h*H + t); the weights differ between the halves,
        // so they come from shared memory (W) instead of the constant bank
        constexpr int H = (npd + 1) / 2;
        const int h = lane >= 16 ? 1 : 0;
        const int l = min(lane & 15, nc * nc - 1);
        const int b = l / nc, c = l - b * nc;
        double x[nc];
#pragma unroll
        for (int q = 0; q < nc; ++q) x[q] = v[((2 * q) * npd + 2 * b) * npd + 2 * c];
#pragma unroll
        for (int t = 0; t < H; ++t) {
          const int i = min(h * H + t, npd - 1);  // the upper half repeats its last output
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < nc; ++q) acc = fma(W[i * nc + q], x[q], acc);
          r1[i * nc * nc + l] = acc;
        }
      } else {
#pragma unroll
        for (int l0 = 0; l0 < nc * nc; l0 += 32) {
          const int l = min(l0 + lane, nc * nc - 1);
          const int b = l / nc, c = l - b * nc;
          double x[nc];
#pragma unroll
          for (int q = 0; q < nc; ++q) x[q] = v[((2 * q) * npd + 2 * b) * npd + 2 * c];
#pragma unroll
          for (int i = 0; i < npd; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < nc; ++q) acc = fma(Wc[i * nc + q], x[q], acc);
            r1[i * nc * nc + l] = acc;
          }
        }
      }
      __syncwarp();
      // axis 1: r2[i][j][c] = sum_b W[j][b] * r1[i][b][c]; lines (i, c)
#pragma unroll(kUnroll2)
      for (int l0 = 0; l0 < npd * nc; l0 += 32) {
        const int l = min(l0 + lane, npd * nc - 1);
        const int i = l / nc, c = l - i * nc;
        double x[nc];
#pragma unroll
        for (int q = 0; q < nc; ++q) x[q] = r1[(i * nc + q) * nc + c];
#pragma unroll
        for (int j = 0; j < npd; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < nc; ++q) acc = fma(Wc[j * nc + q], x[q], acc);
          r2[(i * npd + j) * nc + c] = acc;
        }
      }
      __syncwarp();
      // axis 2: rec[i][j][k] = sum_c W[k][c] * r2[i][j][c]; lines (i, j);
      // residual at nodes with any odd index.  |d| >= +0, so its bits order
      // like unsigned integers, and a NaN (sign cleared) sorts above +inf:
      // an integer max is np.max's result, NaN propagation included.
#pragma unroll(kUnroll3)
      for (int l0 = 0; l0 < npd * npd; l0 += 32) {
        const int l = min(l0 + lane, npd * npd - 1);
        const int i = l / npd, j = l - i * npd;
        const bool even_ij = !((i | j) & 1);
        double x[nc];
#pragma unroll
        for (int q = 0; q < nc; ++q) x[q] = r2[l * nc + q];
#pragma unroll
        for (int k = 0; k < npd; ++k) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < nc; ++q) acc = fma(Wc[k * nc + q], x[q], acc);
#if WV_INTMAX
          unsigned long long bits = (unsigned long long)__double_as_longlong(v[l * npd + k] - acc) & 0x7fffffffffffffffull;
          if (!(k & 1)) bits = even_ij ? 0ull : bits;  // k is a compile-time constant
          mbk[k % WV_NACC] = max(mbk[k % WV_NACC], bits);
#else
          double d = fabs(v[l * npd + k] - acc);
          if (!(k & 1)) d = even_ij ? 0.0 : d;
          m = fmax(m, d);
          bad |= d != d;
#endif
        }
      }
    }
    // warp max (lanes without an odd node hold 0)
#pragma unroll
    for (int q = 0; q < WV_NACC; ++q) mb = max(mb, mbk[q]);
    if (DIM == 2 || !WV_INTMAX) mb = bad ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(m);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mb = max(mb, (unsigned long long)__shfl_xor_sync(0xffffffffu, mb, off));
    m = __longlong_as_double((long long)mb);
    if (lane == 0) {
      if (coeff) coeff[oct] = m;
      if (flags) {
        const int lvl = levels[oct];
        int8_t f;
        if (mode == 0) {  // refine_flags (wavelet.py:118-123)
          if (m > tol && lvl < max_level) f = 1;
          else if (m < coarsen_thr && lvl > min_level) f = -1;
          else f = 0;
        } else {  // refinement_predicate (wavelet.py:137-142)
          f = lvl < min_level ? 1 : (lvl >= max_level ? 0 : (m > tol ? 1 : 0));
        }
        flags[oct] = f;
      }
    }
    __syncwarp();
  }
}

using WvKernel = void (*)(int64_t, const double*, const double*, const int32_t*, int, double, double, int, int,
                          double*, int8_t*);

template <int DIM>
WvKernel pick(int npd, int* per_warp) {
#define WV_CASE(N)                         \
  case N:                                  \
    *per_warp = WvShape<DIM, N>::PER_WARP; \
    return wavelet_kernel<DIM, N>;
  switch (npd) {
    WV_CASE(3) WV_CASE(5) WV_CASE(7) WV_CASE(9) WV_CASE(11) WV_CASE(13) WV_CASE(15)
  }
#undef WV_CASE
  return nullptr;
}

int fail(const char* msg) {
  amr_set_error_internal(msg);
  return AMR_EINVAL;
}

}  // namespace

extern "C" int amr_wavelet_coeff(int dim, int npd, int64_t n, const double* values, const double* W,
                                 const int32_t* levels, int mode, double tol, double coarsen_thr, int min_level,
                                 int max_level, double* coeff, int8_t* flags, void* stream) {
  if (dim != 2 && dim != 3) return fail("amr_wavelet_coeff: dim must be 2 or 3");
  if (npd < 3 || npd % 2 == 0 || npd > WV_MAX_NPD) return fail("amr_wavelet_coeff: nodes_per_dim must be odd, 3..15");
  if (n < 0 || mode < 0 || mode > 1) return fail("amr_wavelet_coeff: bad n or mode");
  if (flags && !levels) return fail("amr_wavelet_coeff: flags need levels");
  if (n == 0) return AMR_OK;
  const int nc = (npd + 1) / 2;
  int per_warp = 0;
  WvKernel kern = dim == 2 ? pick<2>(npd, &per_warp) : pick<3>(npd, &per_warp);
  int woff = 0;
  for (int q = 3; q < npd; q += 2) woff += q * ((q + 1) / 2);
  const size_t budget = 72 * 1024;  // per CTA: several CTAs resident per SM
  int warps = (int)((budget / sizeof(double) - npd * nc) / per_warp);
  warps = warps < 1 ? 1 : (warps > 8 ? 8 : warps);
  const size_t smem = sizeof(double) * (npd * nc + (size_t)warps * per_warp);
  int dev = 0;
  cudaGetDevice(&dev);
  // per (device, dim, npd): SM count and resident CTAs, set up once
  static int cache_sms[16][2][WV_MAX_NPD + 1] = {};
  static int cache_per_sm[16][2][WV_MAX_NPD + 1] = {};
  const int slot = dev & 15;
  int& sms = cache_sms[slot][dim - 2][npd];
  int& per_sm = cache_per_sm[slot][dim - 2][npd];
  cudaError_t e = cudaMemcpyToSymbolAsync(cW, W, sizeof(double) * npd * nc, sizeof(double) * woff,
                                          cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  if (e == cudaSuccess && per_sm == 0) {
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int b = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, warps * 32, smem);
    if (e == cudaSuccess) per_sm = b < 1 ? 1 : b;
  }
  if (e != cudaSuccess) {
    amr_set_error_internal((std::string("amr_wavelet_coeff: ") + cudaGetErrorString(e)).c_str());
    return AMR_ECUDA;
  }
  const int64_t need = (n + warps - 1) / warps;
  const int64_t cap = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
  const int grid = (int)(need < cap ? need : cap);
  kern<<<grid, warps * 32, smem, (cudaStream_t)stream>>>(n, values, W, levels, mode, tol, coarsen_thr,
                                                          min_level, max_level, coeff, flags);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    amr_set_error_internal((std::string("amr_wavelet_coeff launch: ") + cudaGetErrorString(e)).c_str());
    return AMR_ECUDA;
  }
  return AMR_OK;
}
