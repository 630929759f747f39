// amr_stage_blob.cuh — the per-tile stage kernel with the compact blob
// front-end (included by amr_kernels.cu inside its anonymous namespace, after
// amr_stage_pipe.cuh, whose async-copy helpers it uses).
//
// One CTA per leaf tile, several resident per SM (their phases interleave).
// Per tile:
//   1. one thread bulk-copies the blob head (tileprog.py: header, source
//      bases, copy runs, slot codes) into shared memory (one DRAM round trip
//      for every table the tile needs), and bulk-prefetches the tail (rows,
//      taps) into L2;
//   2. every field gather is an 8-byte cp.async along the copy runs straight
//      into the stencil box (chi; phi at owned nodes, or on the whole cross of
//      a face tile) and per interpolation source; u at the owned nodes is
//      loaded into registers for the epilogue;
//   3. hanging rows (0 + sum w*src in ascending-gid order), then the RHS at
//      the owned nodes and the epilogue of stage_kernel.
// Arithmetic is stage_kernel's except that copies land unmodified (no
// "0 + src"): only the sign of a zero can differ, which no later operation
// turns into a nonzero difference.

template <int DIM, int PPO>
struct BlobK {
  using T = Tile<DIM, PPO>;
#ifndef AMR_BLOB_THREADS
#define AMR_BLOB_THREADS 256
#endif
  static constexpr int THREADS = DIM == 3 ? AMR_BLOB_THREADS : 128;
  static constexpr int HEAD = 16 + 64 * 8;                  // mbarrier, interpolation weights
  static constexpr int BOXB = (T::NS * 8 + 15) / 16 * 16;   // one stencil box
  static constexpr int OWNC = (T::NI * 4 + 15) / 16 * 16;   // owned node -> box cell
  __host__ __device__ static int slot_bytes(int max_slots) { return ((max_slots + 1) * 8 + 15) / 16 * 16; }
  __host__ __device__ static size_t smem_bytes(int max_slots, int max_head) {
    return HEAD + (size_t)max_head + 2 * BOXB + 2 * slot_bytes(max_slots) + OWNC;
  }
};

#ifndef AMR_BLOB_MIN_BLOCKS
#define AMR_BLOB_MIN_BLOCKS 4
#endif
// u at the owned nodes is read at the RHS (L2-warm) rather than held in
// registers from the start (-DAMR_BLOB_UO_EARLY): fewer live registers
// (cfg2: LTS 27.0 vs 26.9, GTS 29.7 vs 28.5 G upd/s)
#ifndef AMR_BLOB_UO_EARLY
#define AMR_BLOB_UO_LATE
#endif

template <int DIM, int PPO, bool LTS, int NT>
__global__ void __launch_bounds__(BlobK<DIM, PPO>::THREADS, AMR_BLOB_MIN_BLOCKS)
    stage_blob(const __grid_constant__ AmrStageParams P) {
  using T = Tile<DIM, PPO>;
  using BK = BlobK<DIM, PPO>;
  constexpr int NTH = BK::THREADS;
  constexpr int OPT = (T::NI + NTH - 1) / NTH;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* s_w = reinterpret_cast<double*>(smem + 16);
  unsigned char* head = smem + BK::HEAD;
  double* s_chi = reinterpret_cast<double*>(head + P.max_blob);
  double* s_phi = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(s_chi) + BK::BOXB);
  const int sb = BK::slot_bytes(P.max_slots);
  double* slc = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(s_phi) + BK::BOXB);
  double* slp = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(slc) + sb);
  int* own = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(slp) + sb);
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int64_t n = P.ld;
  const int s = P.stage;
  const bool last = (s == P.n_stages - 1);
  const double* IB = P.ibuf;
  const int64_t nib = P.n_iface_total;
  const AmrSliceCoef* C = P.coef;
  const uint16_t* blob = P.blob;

  // ---- 1: the blob head (one bulk copy), weights meanwhile
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // heads live at a fixed stride (no dependent offset load before the copy)
    const uint32_t hb = (uint32_t)P.max_blob;
    mbar_expect_tx(bar, hb);
    bulk_g2s(head, reinterpret_cast<const unsigned char*>(P.heads) + tile * (int64_t)hb, hb, bar);
    // the tile that takes this CTA slot one wave later: its head into L2
    const int64_t nt = tile + P.prefetch_dist;
    if (P.prefetch_dist > 0 && nt < P.n_tiles)
      bulk_prefetch_l2(P.heads + nt * (int64_t)hb, hb);
  }
  for (int i = tid; i < P.n_wtab; i += NTH) s_w[i] = __ldg(P.wtab + i);
  __syncthreads();  // mbarrier initialised before anyone waits on it
  mbar_wait(bar, 0);
  const int* h = reinterpret_cast<const int*>(head);
  const int g0 = h[0], n_own = h[1], lmeta = h[2], nrun = h[3], nslot = h[4], nrow = h[5], nbase = h[6];
  const int* bases = h + 16;
  const uint32_t* runs = reinterpret_cast<const uint32_t*>(bases + ((nbase + 3) & ~3));
  const uint16_t* sl = reinterpret_cast<const uint16_t*>(head) + h[12];
  const uint16_t* gblob = blob + (int64_t)h[15] * 8;
  const int lvl = lmeta & 0xFF;
  const int cad = (lmeta >> 8) & 0xFF;
  const int faces = (lmeta >> 16) & 0x3F;
  const bool face = faces != 0;
  const int cur = LTS ? C->cur[cad] : P.gts_cur;
  const double* Ucur = cur ? P.U1 : P.U0;
  const double* V = (s == 0) ? Ucur : P.Y + (int64_t)(s & 1) * 2 * n;
  if (tid == 0) {
    const uint32_t tail = 2u * (uint32_t)(h[7] - h[11]);
    if (tail) bulk_prefetch_l2(gblob + h[11], tail);
    if (last) {  // the combine's K_j over the owned range
      const int64_t a16 = g0 & ~1, e16 = (g0 + n_own + 1) & ~1;
      const uint32_t bytes = (uint32_t)(e16 - a16) * 8;
      for (int jj = 0; jj < s; ++jj) {
        bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + a16, bytes);
        bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + n + a16, bytes);
      }
    }
  }
#ifndef AMR_BLOB_UO_LATE
  // u at this thread's owned nodes, for the epilogue (in flight during the
  // gathers and the rows)
  double2 uo[OPT];
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = tid + r * NTH;
    const int64_t g = g0 + (k < n_own ? k : 0);
    uo[r] = make_double2(__ldg(Ucur + g), __ldg(Ucur + n + g));
  }
#else
  if (tid == 0) {  // u over the owned range into L2; read at the RHS (fewer live registers)
    const int64_t a16 = g0 & ~1, e16 = (g0 + n_own + 1) & ~1;
    bulk_prefetch_l2(Ucur + a16, (uint32_t)(e16 - a16) * 8);
    bulk_prefetch_l2(Ucur + n + a16, (uint32_t)(e16 - a16) * 8);
  }
#endif

  // ---- 2: gathers
#ifdef AMR_ABLATE
  const bool gather = !(P.dbg_skip & 1);  // ablation (tools/ablate.py): no copy gathers
#else
  constexpr bool gather = true;
#endif
  for (int r = tid; r < nrun; r += NTH) {
    const uint32_t w = runs[r];
    const int cell = w & 0xFFF, len = ((w >> 12) & 15) + 1;
    const int bi = w >> 26, off = (w >> 16) & 1023;
    if (bi == 63) {  // outside the domain: zero rows
      for (int i = 0; i < len; ++i) {
        s_chi[cell + i] = 0.0;
        s_phi[cell + i] = 0.0;
      }
      continue;
    }
    const int base = bases[bi];
    if (!LTS || base >= 0) {
      const double* src = V + base + off;
      if (gather)
        for (int i = 0; i < len; ++i) cp_async8(s_chi + cell + i, src + i);
      const bool mine = base == g0;
      if (gather && (face || mine))
        for (int i = 0; i < len; ++i) cp_async8(s_phi + cell + i, src + n + i);
      if (mine)
        for (int i = 0; i < len; ++i) own[off + i] = cell + i;
    } else {
      const double* src = IB + (-base - 1 + off);
      for (int i = 0; i < len; ++i) cp_async8(s_chi + cell + i, src + i);
      if (face)
        for (int i = 0; i < len; ++i) cp_async8(s_phi + cell + i, src + nib + i);
    }
  }
  for (int k = tid; k < nslot; k += NTH) {
    const int code = sl[k];
    const int base = bases[code >> 10], off = code & 1023;
    if (!LTS || base >= 0) {
      cp_async8(&slc[k], V + base + off);
      if (face) cp_async8(&slp[k], V + n + base + off);
    } else {
      cp_async8(&slc[k], IB + (-base - 1 + off));
      if (face) cp_async8(&slp[k], IB + nib + (-base - 1 + off));
    }
  }
  if (tid == 0) {
    slc[nslot] = 0.0;  // zero slot of the padding taps
    slp[nslot] = 0.0;
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // ---- 3a: hanging rows, 0 + sum_k w_k src(g_k) in ascending-gid order
  //      (mesh.py:316-351); row words and taps read through L2
  {
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(gblob + h[13]);
    const uint2* taps = reinterpret_cast<const uint2*>(gblob + h[14]);
#ifdef AMR_ABLATE
    const int nrow_ = (P.dbg_skip & 2) ? 0 : nrow;  // ablation: no hanging-row sums
#else
    const int nrow_ = nrow;
#endif
    if (!face) {
      // two quads per step: their 8 products are formed before the 8 ordered
      // adds, and the next two tap words are in flight meanwhile
      for (int r = tid; r < nrow_; r += NTH) {
        const uint32_t w = __ldg(rows + r);
        const int nq = (w >> 12) & 31;
        const uint2* tq = taps + (w >> 17);
        double ax = 0.0;
        uint2 a = nq > 0 ? __ldg(tq) : make_uint2(0u, 0u);
        uint2 b = nq > 1 ? __ldg(tq + 1) : make_uint2(0u, 0u);
        int q = 0;
        for (; q + 2 <= nq; q += 2) {
          const uint32_t t8[8] = {a.x & 0xFFFF, a.x >> 16, a.y & 0xFFFF, a.y >> 16,
                                  b.x & 0xFFFF, b.x >> 16, b.y & 0xFFFF, b.y >> 16};
          if (q + 2 < nq) a = __ldg(tq + q + 2);
          if (q + 3 < nq) b = __ldg(tq + q + 3);
          double pr[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pr[u] = s_w[t8[u] & 63] * slc[t8[u] >> 6];
#pragma unroll
          for (int u = 0; u < 8; ++u) ax = ax + pr[u];
        }
        if (q < nq) {  // odd quad count: the last quad is in a
          const uint32_t t4[4] = {a.x & 0xFFFF, a.x >> 16, a.y & 0xFFFF, a.y >> 16};
          double pr[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) pr[u] = s_w[t4[u] & 63] * slc[t4[u] >> 6];
#pragma unroll
          for (int u = 0; u < 4; ++u) ax = ax + pr[u];
        }
        s_chi[w & 0xFFF] = ax;
      }
    } else
    for (int r = tid; r < nrow_; r += NTH) {
      const uint32_t w = __ldg(rows + r);
      const int nq = (w >> 12) & 31;
      const uint2* tq = taps + (w >> 17);
      double ax = 0.0, ay = 0.0;
      uint2 vn = nq > 0 ? __ldg(tq) : make_uint2(0u, 0u);
      for (int q = 0; q < nq; ++q) {
        const uint2 v = vn;
        if (q + 1 < nq) vn = __ldg(tq + q + 1);  // next tap word in flight during this quad
        const uint32_t t4[4] = {v.x & 0xFFFF, v.x >> 16, v.y & 0xFFFF, v.y >> 16};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double wt = s_w[t4[u] & 63];
          ax = ax + wt * slc[t4[u] >> 6];
          if (face) ay = ay + wt * slp[t4[u] >> 6];
        }
      }
      s_chi[w & 0xFFF] = ax;
      if (face) s_phi[w & 0xFFF] = ay;
    }
  }
  __syncthreads();

  // ---- 3b: RHS at the owned nodes, K_s (and the RK combine) out
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
  const bool need_x = face || P.nonlinear == 1;
  double* Unew = cur ? P.U0 : P.U1;
  double* Ks = P.K + (int64_t)s * 2 * n;
#ifdef AMR_ABLATE
  const int n_own_ = (P.dbg_skip & 4) ? 0 : n_own;  // ablation: no RHS / epilogue
#else
  const int n_own_ = n_own;
#endif
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = tid + r * NTH;
    if (k >= n_own_) break;
    const int cell = own[k];
#ifdef AMR_BLOB_UO_LATE
    const double2 uor = make_double2(__ldg(Ucur + g0 + k), __ldg(Ucur + n + g0 + k));
#else
    const double2 uor = uo[r];
#endif
    SmemAcc<DIM, PPO> acc{s_chi, s_phi, cell};
    double2 ks;
    if (!need_x) {
      ks = rhs_interior<DIM>(acc, W, R);
    } else {
      int pos[3];
      {
        int c = cell;
#pragma unroll
        for (int d = DIM - 1; d >= 0; --d) {
          pos[d] = c % T::NP - T::PAD;
          c /= T::NP;
        }
      }
      double x[3] = {0.0, 0.0, 0.0};
      const int64_t side_len = (int64_t)1 << (P.max_depth - lvl);
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const int64_t lat = (int64_t)h[8 + d] * (PPO - 1) + side_len * pos[d];
        x[d] = P.lo[d] + ((double)lat / (double)P.top_nodes) * P.extent[d];
      }
      ks = rhs_point<DIM>(acc, pos, PPO, faces, x, W, R);
    }
    const int64_t g = g0 + k;
    if (!last || LTS) {
      Ks[g] = ks.x;
      Ks[n + g] = ks.y;
    }
    if (!last) {  // next stage's verbatim source of this owned node
      double yx = 0.0 + uor.x, yy = 0.0 + uor.y;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const int jv = P.vt_j[t];
        const double c = LTS ? C->cstage[cad][s + 1][jv] : P.g_cstage[s + 1][jv];
        const double kx = (jv == s) ? ks.x : __ldg(P.K + (int64_t)jv * 2 * n + g);
        const double ky = (jv == s) ? ks.y : __ldg(P.K + (int64_t)jv * 2 * n + n + g);
        yx = yx + c * kx;
        yy = yy + c * ky;
      }
      double* Yout = P.Y + (int64_t)((s + 1) & 1) * 2 * n;
      Yout[g] = yx;
      Yout[n + g] = yy;
    } else {
      double ux = 0.0 + uor.x, uy = 0.0 + uor.y;
      for (int jj = 0; jj < P.n_stages; ++jj) {
        const double c = LTS ? C->comb[cad][jj] : P.g_comb[jj];
        if (c == 0.0) continue;
        const double kx = (jj == s) ? ks.x : __ldg(P.K + (int64_t)jj * 2 * n + g);
        const double ky = (jj == s) ? ks.y : __ldg(P.K + (int64_t)jj * 2 * n + n + g);
        ux = ux + c * kx;
        uy = uy + c * ky;
      }
      Unew[g] = ux;
      Unew[n + g] = uy;
    }
  }
}
