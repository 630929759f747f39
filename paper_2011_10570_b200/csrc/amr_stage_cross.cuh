// amr_stage_cross.cuh — the stage kernel on the owned cross (included by
// amr_kernels.cu inside its anonymous namespace).
//
// One CTA per leaf tile, many resident per SM (small footprint: one stencil
// box).  The tile's program (tileprog.py) has a head — header, source bases,
// copy runs, slot codes — that one thread bulk-copies into shared memory, and
// a tail — hanging rows and taps — read through L2.  Per tile:
//   1. head (cp.async.bulk + mbarrier); L2 prefetch of the tail and of the
//      owned ranges the epilogue reads;
//   2. chi on the owned cross: 8-byte cp.async along the copy runs, a warp
//      covering 32 nodes per instruction (runs bucketed by length: 8, 4, 2 or
//      1 lanes per run, so lanes walk along runs — coalesced and balanced);
//      one cp.async per interpolation source ("slot");
//   3. hanging rows 0 + sum w*src(slot) in ascending-gid order (mesh.py:316-351);
//   4. RHS at the owned nodes (wave.py:147-201; phi at an owned node is read
//      from the stage source row directly — only physical-face rows need phi
//      derivatives), then K_s, the next stage's verbatim source Y, or on the
//      last stage the RK combine (stepper.py:422-453);
//   5. tiles on a physical face only: phi on the owned cross into the same box
//      (steps 2-3 again) and the radiative rows' phi part (wave.py:173-201)
//      for the on-face nodes, whose epilogue was deferred.
// Arithmetic is bit-identical to the reference (see amr_kernels.cu): numpy's
// operation order, no FMA contraction; copies land unmodified (only the sign
// of a zero can differ from the reference's "0 + 1.0*src", and no later
// operation turns that into a nonzero difference).

template <int DIM, int PPO>
struct CrossK {
  using T = Tile<DIM, PPO>;
  static constexpr int HEAD = 16 + 64 * 8;                 // mbarrier, interpolation weights
  static constexpr int BOXB = (T::NS * 8 + 15) / 16 * 16;  // the stencil box (chi; phi in step 5)
  static constexpr int OWNB = (T::NI * 2 + 15) / 16 * 16;  // owned node -> box cell (uint16)
  __host__ __device__ static int slot_bytes(int max_slots) { return ((max_slots + 1) * 8 + 15) / 16 * 16; }
  __host__ __device__ static size_t smem_bytes(int max_slots, int max_head) {
    return HEAD + (size_t)max_head + BOXB + slot_bytes(max_slots) + OWNB;
  }
};

// step 2 for one variable (vo = row offset of the variable in the field
// arrays, ibo in the interface buffer)
template <bool LTS, int NTH>
__device__ __forceinline__ void cross_gather(const int* __restrict__ h, double* box, double* slot, uint16_t* own,
                                             const double* __restrict__ V, const double* __restrict__ IB,
                                             int64_t vo, int64_t ibo, int g0, bool own_map) {
  constexpr int NW = NTH / 32;
  const int nrun = h[3], nslot = h[4], nbase = h[6];
  const int* bases = h + 16;
  const uint32_t* runs = reinterpret_cast<const uint32_t*>(bases + ((nbase + 3) & ~3));
  const uint16_t* sl = reinterpret_cast<const uint16_t*>(runs + ((nrun + 3) & ~3));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cnt4[4] = {h[11] & 0xFFFF, h[11] >> 16, h[12] & 0xFFFF, h[12] >> 16};
  int r0 = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int lg = 3 - b;        // log2 lanes per run: 8, 4, 2, 1
    const int rpi = 32 >> lg;    // runs per warp instruction
    const int i = lane & ((1 << lg) - 1);
    const int cnt = cnt4[b];
    for (int r = warp * rpi + (lane >> lg); r < cnt; r += NW * rpi) {
      const uint32_t w = runs[r0 + r];
      if (i <= (int)((w >> 12) & 7)) {
        const int cell = (int)(w & 0xFFF) + i;
        const int off = (int)((w >> 16) & 1023) + i;
        const int base = bases[w >> 26];
        if (!LTS || base >= 0) {
          cp_async8(box + cell, V + vo + base + off);
          if (own_map && base == g0) own[off] = (uint16_t)cell;
        } else {
          cp_async8(box + cell, IB + ibo + (-base - 1 + off));
        }
      }
    }
    r0 += cnt;
  }
  for (int k = threadIdx.x; k < nslot; k += NTH) {
    const int code = sl[k];
    const int base = bases[code >> 10], off = code & 1023;
    if (!LTS || base >= 0)
      cp_async8(slot + k, V + vo + base + off);
    else
      cp_async8(slot + k, IB + ibo + (-base - 1 + off));
  }
  if (threadIdx.x == 0) slot[nslot] = 0.0;  // zero slot of the padding taps
}

// step 3: hanging rows into the box.  Two quads of taps per step: their 8
// products first, then the 8 ordered adds; the next tap words in flight.
template <int NTH>
__device__ __forceinline__ void cross_rows(const uint16_t* __restrict__ tl, int nrow, int taps_off,
                                           const double* s_w, const double* slot, double* box) {
  const uint32_t* rows = reinterpret_cast<const uint32_t*>(tl);
  const uint2* taps = reinterpret_cast<const uint2*>(tl + taps_off);
  for (int r = threadIdx.x; r < nrow; r += NTH) {
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
      for (int u = 0; u < 8; ++u) pr[u] = s_w[t8[u] & 63] * slot[t8[u] >> 6];
#pragma unroll
      for (int u = 0; u < 8; ++u) ax = ax + pr[u];
    }
    if (q < nq) {  // odd quad count: the last quad is in a
      const uint32_t t4[4] = {a.x & 0xFFFF, a.x >> 16, a.y & 0xFFFF, a.y >> 16};
      double pr[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) pr[u] = s_w[t4[u] & 63] * slot[t4[u] >> 6];
#pragma unroll
      for (int u = 0; u < 4; ++u) ax = ax + pr[u];
    }
    box[w & 0xFFF] = ax;
  }
}

// box accessor of deriv(): value at offset o along axis d of the current cell
template <int DIM, int PPO>
struct BoxLine {
  const double* b;
  int cell, stride;
  __device__ __forceinline__ double operator()(int o) const { return b[cell + o * stride]; }
};

template <int DIM, int PPO>
__device__ __forceinline__ int box_stride(int d) {
  constexpr int NP = Tile<DIM, PPO>::NP;
  return (DIM == 3) ? (d == 0 ? NP * NP : (d == 1 ? NP : 1)) : (d == 0 ? NP : 1);
}

template <int DIM, int PPO>
__device__ __forceinline__ void cell_pos(int cell, int* pos) {
  constexpr int NP = Tile<DIM, PPO>::NP;
  int c = cell;
#pragma unroll
  for (int d = DIM - 1; d >= 0; --d) {
    pos[d] = c % NP - 2;
    c /= NP;
  }
}

template <int DIM>
__device__ __forceinline__ bool on_face_of(const int* pos, int n, int faces) {
  bool f = false;
#pragma unroll
  for (int d = 0; d < DIM; ++d)
    f |= (((faces >> (2 * d)) & 1) && pos[d] == 0) || (((faces >> (2 * d + 1)) & 1) && pos[d] == n - 1);
  return f;
}

template <int DIM, int PPO, bool LTS, int NT, int NTH>
__global__ void __launch_bounds__(NTH, (NTH <= 128 ? 8 : 4)) stage_cross(const __grid_constant__ AmrStageParams P) {
  using T = Tile<DIM, PPO>;
  using CK = CrossK<DIM, PPO>;
  constexpr int OPT = (T::NI + NTH - 1) / NTH;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  double* s_w = reinterpret_cast<double*>(smem + 16);
  unsigned char* head = smem + CK::HEAD;
  double* box = reinterpret_cast<double*>(head + P.max_blob);
  double* slot = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(box) + CK::BOXB);
  uint16_t* own = reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(slot) + CK::slot_bytes(P.max_slots));
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;
  const int64_t n = P.ld;
  const int s = P.stage;
  const bool last = (s == P.n_stages - 1);
  const AmrSliceCoef* C = P.coef;

  // ---- 1: the head (one bulk copy at a fixed stride), weights meanwhile
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    const uint32_t hb = (uint32_t)P.max_blob;
    mbar_expect_tx(bar, hb);
    bulk_g2s(head, P.heads + tile * (int64_t)hb, hb, bar);
  }
  for (int i = tid; i < P.n_wtab; i += NTH) s_w[i] = __ldg(P.wtab + i);
  __syncthreads();  // mbarrier initialised before anyone waits on it
  mbar_wait(bar, 0);
  const int* h = reinterpret_cast<const int*>(head);
  const int g0 = h[0], n_own = h[1], lmeta = h[2], nrow = h[5];
  const int lvl = lmeta & 0xFF;
  const int cad = (lmeta >> 8) & 0xFF;
  const int faces = (lmeta >> 16) & 0x3F;
  const uint16_t* tl = P.tail + (int64_t)h[14] * 8;
  const int taps_off = h[15];
  const int cur = LTS ? C->cur[cad] : P.gts_cur;
  const double* Ucur = cur ? P.U1 : P.U0;
  const double* V = (s == 0) ? Ucur : P.Y + (int64_t)(s & 1) * 2 * n;
  if (tid == 0) {
    if (h[7]) bulk_prefetch_l2(tl, (uint32_t)h[7]);
    // owned ranges the RHS and epilogue read: u (chi, phi), the stage
    // source's phi row, and on the last stage the combine's K_j
    const int64_t a16 = g0 & ~1, e16 = (g0 + n_own + 1) & ~1;
    const uint32_t bytes = (uint32_t)(e16 - a16) * 8;
    bulk_prefetch_l2(Ucur + a16, bytes);
    bulk_prefetch_l2(Ucur + n + a16, bytes);
    if (s) bulk_prefetch_l2(V + n + a16, bytes);
    if (last)
      for (int jj = 0; jj < s; ++jj) {
        bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + a16, bytes);
        bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + n + a16, bytes);
      }
  }

  // ---- 2, 3: chi on the owned cross
  cross_gather<LTS, NTH>(h, box, slot, own, V, P.ibuf, 0, 0, g0, true);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cross_rows<NTH>(tl, nrow, taps_off, s_w, slot, box);
  __syncthreads();

  // ---- 4: RHS at the owned nodes
  const Weights& W = P;
  const double h_l = P.h[lvl], h2 = P.h2[lvl], inv_h2 = P.inv_h2[lvl];
  const bool pow2 = P.h2_pow2[lvl] != 0;
  const bool face = faces != 0;
  const bool need_x = face || P.nonlinear == 1;
  double* Unew = cur ? P.U0 : P.U1;
  double* Ks = P.K + (int64_t)s * 2 * n;
  const int64_t side_len = (int64_t)1 << (P.max_depth - lvl);

  // K_s, the next stage's verbatim source, or the RK combine of owned node k
  auto epilogue = [&](int k, double2 ks) {
    const int64_t g = g0 + k;
    const double2 uor = make_double2(__ldg(Ucur + g), __ldg(Ucur + n + g));
    if (!last || LTS) {
      Ks[g] = ks.x;
      Ks[n + g] = ks.y;
    }
    if (!last) {
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
  };
  auto coords = [&](const int* pos, double* x) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const int64_t lat = (int64_t)h[8 + d] * (PPO - 1) + side_len * pos[d];
      x[d] = P.lo[d] + ((double)lat / (double)P.top_nodes) * P.extent[d];
    }
  };
  auto radius = [&](const double* x) {
    double r2 = x[0] * x[0];
#pragma unroll
    for (int d = 1; d < DIM; ++d) r2 = r2 + x[d] * x[d];
    const double r = sqrt(r2);
    return r > P.r_eps ? r : P.r_eps;
  };

#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = tid + r * NTH;
    if (k >= n_own) break;
    const int cell = own[k];
    const double phi_c = __ldg(V + n + g0 + k);
    if (!need_x) {  // centred 4th-order Laplacian (+ cubic), dchi = phi (wave.py:147-170)
      double lap = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const int S = box_stride<DIM, PPO>(d);
        double t = W.d2c[0] * box[cell - 2 * S];
#pragma unroll
        for (int q = 1; q < 5; ++q) t = t + W.d2c[q] * box[cell + (q - 2) * S];
        t = pow2 ? t * inv_h2 : t / h2;
        lap = (d == 0) ? t : lap + t;
      }
      double dphi = lap;
      if (P.nonlinear == 2) {
        const double chi = box[cell];
        dphi = dphi - (chi * chi) * chi;
      }
      epilogue(k, make_double2(phi_c, dphi));
      continue;
    }
    int pos[3] = {0, 0, 0};
    cell_pos<DIM, PPO>(cell, pos);
    double x[3] = {0.0, 0.0, 0.0};
    coords(pos, x);
    const bool of = on_face_of<DIM>(pos, PPO, faces);
    const double chi = box[cell];
    if (!of) {
      double lap = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        BoxLine<DIM, PPO> get{box, cell, box_stride<DIM, PPO>(d)};
        const double t = deriv(get, 2, pos[d], PPO, faces & (1 << (2 * d)), faces & (2 << (2 * d)), W, h2, pow2,
                               inv_h2);
        lap = (d == 0) ? t : lap + t;
      }
      double dphi = lap;
      if (P.nonlinear == 1) {
        double r2 = x[0] * x[0];
#pragma unroll
        for (int d = 1; d < DIM; ++d) r2 = r2 + x[d] * x[d];
        const double r2_reg = r2 > P.r_eps2 ? r2 : P.r_eps2;
        dphi = dphi - sin(2.0 * chi) / r2_reg;
      } else if (P.nonlinear == 2) {
        dphi = dphi - (chi * chi) * chi;
      }
      epilogue(k, make_double2(phi_c, dphi));
    } else {  // radiative row, chi part (wave.py:173-201); phi part in step 5
      double a = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        BoxLine<DIM, PPO> get{box, cell, box_stride<DIM, PPO>(d)};
        const double gd = deriv(get, 1, pos[d], PPO, faces & (1 << (2 * d)), faces & (2 << (2 * d)), W, h_l, false,
                                0.0);
        const double term = x[d] * gd;
        a = (d == 0) ? term : a + term;
      }
      Ks[g0 + k] = a / radius(x) - P.k_chi * (chi - P.f0_chi);
    }
  }
  if (!face) return;

  // ---- 5: physical-face tiles: phi on the owned cross, radiative phi rows
  __syncthreads();  // everyone is done reading chi from the box
  cross_gather<LTS, NTH>(h, box, slot, own, V, P.ibuf, n, P.n_iface_total, g0, false);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  cross_rows<NTH>(tl, nrow, taps_off, s_w, slot, box);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = tid + r * NTH;
    if (k >= n_own) break;
    const int cell = own[k];
    int pos[3] = {0, 0, 0};
    cell_pos<DIM, PPO>(cell, pos);
    if (!on_face_of<DIM>(pos, PPO, faces)) continue;
    double x[3] = {0.0, 0.0, 0.0};
    coords(pos, x);
    double a = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      BoxLine<DIM, PPO> get{box, cell, box_stride<DIM, PPO>(d)};
      const double gd = deriv(get, 1, pos[d], PPO, faces & (1 << (2 * d)), faces & (2 << (2 * d)), W, h_l, false,
                              0.0);
      const double term = x[d] * gd;
      a = (d == 0) ? term : a + term;
    }
    const double phi_c = box[cell];
    const double dphi = a / radius(x) - P.k_phi * (phi_c - P.f0_phi);
    const double dchi = *(volatile const double*)(Ks + g0 + k);  // written by this thread in step 4
    epilogue(k, make_double2(dchi, dphi));
  }
}
