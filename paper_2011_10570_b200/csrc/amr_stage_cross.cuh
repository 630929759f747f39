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
  static constexpr int BARS = 64;                          // mbarriers: one per head and per tail of the CTA's tiles
  static constexpr int HEAD = BARS + 64 * 8;               // + interpolation weights
  static constexpr int BOXB = (T::BOX * 8 + 15) / 16 * 16;  // the stencil box (chi; phi in step 5)
  static constexpr int OWNB = (T::NI * 2 + 15) / 16 * 16;  // owned node -> box cell (uint16)
  __host__ __device__ static int slot_bytes(int max_slots) { return ((max_slots + 1) * 8 + 15) / 16 * 16; }
  __host__ __device__ static size_t smem_bytes(int max_slots, int max_head, int max_tail, int tiles_per_cta) {
    return HEAD + (size_t)tiles_per_cta * max_head + (size_t)max_tail + BOXB + slot_bytes(max_slots) + OWNB;
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
  // the interpolation sources first, as their own cp.async group: the hanging
  // rows start when these have landed, while the copy runs are still in flight
  for (int k = threadIdx.x; k < nslot; k += NTH) {
    const int code = sl[k];
    const int base = bases[code >> 10], off = code & 1023;
    if (!LTS || base >= 0)
      cp_async8(slot + k, V + vo + base + off);
    else
      cp_async8(slot + k, IB + ibo + (-base - 1 + off));
  }
  if (threadIdx.x == 0) slot[nslot] = 0.0;  // zero slot of the padding taps
  cp_async_commit();
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
  cp_async_commit();
}

// step 3: hanging rows into the box, from the tile's tail in shared memory.
// Two quads of taps per step: their 8 products first, then the 8 ordered adds.
template <int NTH>
__device__ __forceinline__ void cross_rows(const uint16_t* tl, int nrow, int taps_off, const double* s_w,
                                           const double* slot, double* box) {
  const uint32_t* rows = reinterpret_cast<const uint32_t*>(tl);
  const uint2* taps = reinterpret_cast<const uint2*>(tl + taps_off);
  for (int r = threadIdx.x; r < nrow; r += NTH) {
    const uint32_t w = rows[r];
    const int nq = (w >> 12) & 31;
    const uint2* tq = taps + (w >> 17);
    double ax = 0.0;
    uint2 a = nq > 0 ? tq[0] : make_uint2(0u, 0u);
    uint2 b = nq > 1 ? tq[1] : make_uint2(0u, 0u);
    int q = 0;
    for (; q + 2 <= nq; q += 2) {
      const uint32_t t8[8] = {a.x & 0xFFFF, a.x >> 16, a.y & 0xFFFF, a.y >> 16,
                              b.x & 0xFFFF, b.x >> 16, b.y & 0xFFFF, b.y >> 16};
      if (q + 2 < nq) a = tq[q + 2];
      if (q + 3 < nq) b = tq[q + 3];
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
  using T = Tile<DIM, PPO>;
  return (DIM == 3) ? (d == 0 ? T::NP * T::RS : (d == 1 ? T::RS : 1)) : (d == 0 ? T::RS : 1);
}

template <int DIM, int PPO>
__device__ __forceinline__ void cell_pos(int cell, int* pos) {
  using T = Tile<DIM, PPO>;
  pos[DIM - 1] = cell % T::RS - 2;
  int c = cell / T::RS;
#pragma unroll
  for (int d = DIM - 2; d >= 0; --d) {
    pos[d] = c % T::NP - 2;
    c /= T::NP;
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

// A tile's decoded header and stage context.
struct TileCtx {
  const int* h;           // head in shared memory
  const uint16_t* tl;     // tail in global memory
  int g0, n_own, nrow, taps_off, lvl, cad, faces;
  const double* Ucur;     // u_curr buffer of the tile's cadence
  const double* V;        // verbatim stage source (u at stage 0, Y after)
  double* Unew;           // the other u buffer (RK combine target)
};

__device__ __forceinline__ TileCtx tile_ctx(const AmrStageParams& P, const unsigned char* head, bool lts) {
  TileCtx c;
  c.h = reinterpret_cast<const int*>(head);
  c.g0 = c.h[0];
  c.n_own = c.h[1];
  const int lmeta = c.h[2];
  c.nrow = c.h[5];
  c.lvl = lmeta & 0xFF;
  c.cad = (lmeta >> 8) & 0xFF;
  c.faces = (lmeta >> 16) & 0x3F;
  c.tl = P.tail + (int64_t)c.h[14] * 8;
  c.taps_off = c.h[15];
  const int cur = lts ? (int)((P.l_cur_mask >> c.cad) & 1u) : P.gts_cur;
  c.Ucur = cur ? P.U1 : P.U0;
  c.Unew = cur ? P.U0 : P.U1;
  c.V = (P.stage == 0) ? c.Ucur : P.Y + (int64_t)(P.stage & 1) * 2 * P.ld;
  return c;
}

// one thread: on the last stage, L2 prefetch of the combine's K_j over the
// owned range
__device__ __forceinline__ void tile_prefetch(const AmrStageParams& P, const TileCtx& c) {
  if (P.stage == P.n_stages - 1) {
    const int64_t n = P.ld;
    const int64_t a16 = c.g0 & ~1, e16 = (c.g0 + c.n_own + 1) & ~1;
    const uint32_t bytes = (uint32_t)(e16 - a16) * 8;
    for (int jj = 0; jj < P.stage; ++jj) {
      bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + a16, bytes);
      bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + n + a16, bytes);
    }
  }
}

// this thread's owned nodes (k = tid + r*NTH): phi of the stage source and u
template <int OPT, int NTH>
__device__ __forceinline__ void owned_loads(const AmrStageParams& P, const TileCtx& c, double* pc, double* u0,
                                            double* u1) {
  const int64_t n = P.ld;
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = threadIdx.x + r * NTH;
    const int64_t g = c.g0 + (k < c.n_own ? k : 0);
    pc[r] = __ldg(c.V + n + g);
    u0[r] = __ldg(c.Ucur + g);
    u1[r] = __ldg(c.Ucur + n + g);
  }
}

// K_s, the next stage's verbatim source, or the RK combine of owned node k
template <bool LTS, int NT>
__device__ __forceinline__ void tile_epilogue(const AmrStageParams& P, const TileCtx& c, int k, double2 ks,
                                              double2 uor) {
  const int64_t n = P.ld;
  const int s = P.stage;
  const bool last = (s == P.n_stages - 1);
  const int64_t g = c.g0 + k;
  double* Ks = P.K + (int64_t)s * 2 * n;
  if (!last || LTS) {
    Ks[g] = ks.x;
    Ks[n + g] = ks.y;
  }
  if (!last) {
    double yx = 0.0 + uor.x, yy = 0.0 + uor.y;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int jv = P.vt_j[t];
      const double cf = LTS ? P.l_cnext[c.cad][jv] : P.g_cstage[s + 1][jv];
      const double kx = (jv == s) ? ks.x : __ldg(P.K + (int64_t)jv * 2 * n + g);
      const double ky = (jv == s) ? ks.y : __ldg(P.K + (int64_t)jv * 2 * n + n + g);
      yx = yx + cf * kx;
      yy = yy + cf * ky;
    }
    double* Yout = P.Y + (int64_t)((s + 1) & 1) * 2 * n;
    Yout[g] = yx;
    Yout[n + g] = yy;
  } else {
    // every K_j (j < s) in flight at once, then the ordered combine
    double kx[AMR_MAXP], ky[AMR_MAXP];
#pragma unroll
    for (int jj = 0; jj < AMR_MAXP; ++jj) {
      if (jj < s) {
        kx[jj] = __ldg(P.K + (int64_t)jj * 2 * n + g);
        ky[jj] = __ldg(P.K + (int64_t)jj * 2 * n + n + g);
      } else {
        kx[jj] = ks.x;
        ky[jj] = ks.y;
      }
    }
    double ux = 0.0 + uor.x, uy = 0.0 + uor.y;
#pragma unroll
    for (int jj = 0; jj < AMR_MAXP; ++jj) {
      if (jj >= P.n_stages) break;
      const double cf = LTS ? P.l_comb[c.cad][jj] : P.g_comb[jj];
      if (cf == 0.0) continue;
      ux = ux + cf * kx[jj];
      uy = uy + cf * ky[jj];
    }
    c.Unew[g] = ux;
    c.Unew[n + g] = uy;
  }
}

template <int DIM, int PPO>
__device__ __forceinline__ void tile_coords(const AmrStageParams& P, const TileCtx& c, const int* pos, double* x) {
  const int64_t side_len = (int64_t)1 << (P.max_depth - c.lvl);
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const int64_t lat = (int64_t)c.h[8 + d] * (PPO - 1) + side_len * pos[d];
    x[d] = P.lo[d] + ((double)lat / (double)P.top_nodes) * P.extent[d];
  }
}

template <int DIM>
__device__ __forceinline__ double face_radius(const AmrStageParams& P, const double* x) {
  double r2 = x[0] * x[0];
#pragma unroll
  for (int d = 1; d < DIM; ++d) r2 = r2 + x[d] * x[d];
  const double r = sqrt(r2);
  return r > P.r_eps ? r : P.r_eps;
}

// radiative row of one variable at an on-face node (wave.py:173-201):
// (sum_d x_d * d1_d f) / max(r, r_eps), from the box holding that variable
template <int DIM, int PPO>
__device__ __forceinline__ double radial_term(const AmrStageParams& P, const double* box, int cell, const int* pos,
                                              int faces, const double* x, double h_l) {
  double a = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    BoxLine<DIM, PPO> get{box, cell, box_stride<DIM, PPO>(d)};
    const double gd = deriv(get, 1, pos[d], PPO, faces & (1 << (2 * d)), faces & (2 << (2 * d)), P, h_l, false, 0.0);
    const double term = x[d] * gd;
    a = (d == 0) ? term : a + term;
  }
  return a / face_radius<DIM>(P, x);
}

// step 4: RHS at the owned nodes from the chi box; on-face nodes of a
// physical-face tile store their dchi in K_s and defer the rest to step 5
template <int DIM, int PPO, bool LTS, int NT, int NTH, int OPT, bool FULL>
__device__ __forceinline__ void rhs_pass1(const AmrStageParams& P, const TileCtx& c, const double* box,
                                          const uint16_t* own, const double* pc, const double* u0, const double* u1) {
  const double h2 = P.h2[c.lvl], inv_h2 = P.inv_h2[c.lvl];
  const bool pow2 = P.h2_pow2[c.lvl] != 0;
  // lean instance (FULL = false): tiles off the physical faces, no coordinate-dependent source
  const bool need_x = FULL && (c.faces != 0 || P.nonlinear == 1);
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = threadIdx.x + r * NTH;
    if (k >= c.n_own) break;
    const int cell = own[k];
    const double phi_c = pc[r];
    if (!need_x) {  // centred 4th-order Laplacian (+ cubic), dchi = phi (wave.py:147-170)
      double lap = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const int S = box_stride<DIM, PPO>(d);
        double t = P.d2c[0] * box[cell - 2 * S];
#pragma unroll
        for (int q = 1; q < 5; ++q) t = t + P.d2c[q] * box[cell + (q - 2) * S];
        t = pow2 ? t * inv_h2 : t / h2;
        lap = (d == 0) ? t : lap + t;
      }
      double dphi = lap;
      if (P.nonlinear == 2) {
        const double chi = box[cell];
        dphi = dphi - (chi * chi) * chi;
      }
      tile_epilogue<LTS, NT>(P, c, k, make_double2(phi_c, dphi), make_double2(u0[r], u1[r]));
      continue;
    }
    int pos[3] = {0, 0, 0};
    cell_pos<DIM, PPO>(cell, pos);
    double x[3] = {0.0, 0.0, 0.0};
    tile_coords<DIM, PPO>(P, c, pos, x);
    const double chi = box[cell];
    if (!on_face_of<DIM>(pos, PPO, c.faces)) {
      double lap = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        BoxLine<DIM, PPO> get{box, cell, box_stride<DIM, PPO>(d)};
        const double t = deriv(get, 2, pos[d], PPO, c.faces & (1 << (2 * d)), c.faces & (2 << (2 * d)), P, h2, pow2,
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
      tile_epilogue<LTS, NT>(P, c, k, make_double2(phi_c, dphi), make_double2(u0[r], u1[r]));
    } else {  // radiative row, chi part; the phi part in step 5
      P.K[(int64_t)P.stage * 2 * P.ld + c.g0 + k] =
          radial_term<DIM, PPO>(P, box, cell, pos, c.faces, x, P.h[c.lvl]) - P.k_chi * (chi - P.f0_chi);
    }
  }
}

// step 5 (after phi replaced chi in the box): radiative phi rows of the
// on-face nodes and their deferred epilogue
template <int DIM, int PPO, bool LTS, int NT, int NTH, int OPT>
__device__ __forceinline__ void rhs_pass2(const AmrStageParams& P, const TileCtx& c, const double* box,
                                          const uint16_t* own, const double* u0, const double* u1) {
#pragma unroll
  for (int r = 0; r < OPT; ++r) {
    const int k = threadIdx.x + r * NTH;
    if (k >= c.n_own) break;
    const int cell = own[k];
    int pos[3] = {0, 0, 0};
    cell_pos<DIM, PPO>(cell, pos);
    if (!on_face_of<DIM>(pos, PPO, c.faces)) continue;
    double x[3] = {0.0, 0.0, 0.0};
    tile_coords<DIM, PPO>(P, c, pos, x);
    const double phi_c = box[cell];
    const double dphi = radial_term<DIM, PPO>(P, box, cell, pos, c.faces, x, P.h[c.lvl]) - P.k_phi * (phi_c - P.f0_phi);
    // dchi was written by this thread in step 4
    const double dchi = *(volatile const double*)(P.K + (int64_t)P.stage * 2 * P.ld + c.g0 + k);
    tile_epilogue<LTS, NT>(P, c, k, make_double2(dchi, dphi), make_double2(u0[r], u1[r]));
  }
}

#ifndef AMR_CROSS_MINB
#define AMR_CROSS_MINB 4  // resident 256-thread CTAs per SM the register budget is sized for
#endif
#ifndef AMR_ALT_NTH
#define AMR_ALT_NTH 128  // the second CTA size compiled in (AmrStageParams.threads selects it)
#endif

#ifdef AMR_PHASE_PROBE
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define AMR_PROBE(i) \
  if (P.probe && threadIdx.x == 0) P.probe[tile * 8 + (i)] = gtimer()
#else
#define AMR_PROBE(i)
#endif

#ifndef AMR_TPC
#define AMR_TPC 1  // consecutive tiles per CTA (2 and 3 measured slower: the unrolled tile bodies thrash the instruction cache)
#endif

// Two instances: FULL handles every tile; the lean one (FULL = false) is for
// tiles off the physical faces with a coordinate-free source.  It is a quarter
// of the code (no biased rows, radiative rows, coordinates or second cross
// gather) and runs the common tiles about 3 % faster; the engine launches it on
// those tiles and the full instance on the rest.
// One CTA runs AMR_TPC consecutive tiles, one after the other.  All their
// heads are requested up front (one bulk copy each, own mbarrier), so only the
// first head fetch is exposed; many CTAs stay resident per SM, so tiles in
// different phases interleave.
template <int DIM, int PPO, bool LTS, int NT, int NTH, bool FULL>
__global__ void __launch_bounds__(NTH, (AMR_CROSS_MINB * 256) / NTH)
    stage_cross(const __grid_constant__ AmrStageParams P) {
  using T = Tile<DIM, PPO>;
  using CK = CrossK<DIM, PPO>;
  constexpr int OPT = (T::NI + NTH - 1) / NTH;
  constexpr int TPC = AMR_TPC;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // [0, TPC): heads; [TPC, 2 TPC): tails
  double* s_w = reinterpret_cast<double*>(smem + CK::BARS);
  unsigned char* head0 = smem + CK::HEAD;
  const uint32_t hb = (uint32_t)P.max_head;
  uint16_t* s_tail = reinterpret_cast<uint16_t*>(head0 + (size_t)TPC * hb);
  double* box = reinterpret_cast<double*>(head0 + (size_t)TPC * hb + P.max_tail);
  double* slot = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(box) + CK::BOXB);
  uint16_t* own = reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(slot) + CK::slot_bytes(P.max_slots));
  const int tid = threadIdx.x;
  const int64_t tile0 = (int64_t)blockIdx.x * TPC;
  // programmatic dependent launch: the next kernel on the stream may start its
  // CTAs (and fetch its static tables) while this grid drains
  pdl_launch_dependents();

  // ---- 1: the heads (one bulk copy each at a fixed stride), weights meanwhile
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < 2 * TPC; ++j) mbar_init(bar + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
#pragma unroll
    for (int j = 0; j < TPC; ++j) {
      if (tile0 + j < P.n_tiles) {
        mbar_expect_tx(bar + j, hb);
        bulk_g2s(head0 + (size_t)j * hb, P.heads + (tile0 + j) * hb, hb, bar + j);
      }
    }
  }
  // interpolation weights: in flight with the gathers (waited for with them)
  for (int i = tid; i < P.n_wtab; i += NTH) cp_async8(s_w + i, P.wtab + i);
  __syncthreads();  // mbarriers initialised before anyone waits on them

#pragma unroll
  for (int j = 0; j < TPC; ++j) {
    const int64_t tile = tile0 + j;
    if (tile >= P.n_tiles) break;
    AMR_PROBE(0);
    const unsigned char* head = head0 + (size_t)j * hb;
    mbar_wait(bar + j, 0);
    // everything above reads static tables only; the fields (and the interface
    // buffer) are the previous kernels' output
    if (j == 0) pdl_wait();
    AMR_PROBE(1);
    const TileCtx c = tile_ctx(P, head, LTS);
    const uint32_t tail_bytes = (uint32_t)c.h[7];
    if (tid == 0) {
      // the tail (hanging rows, taps): one bulk copy, lands during the gathers
      if (tail_bytes) {
        mbar_expect_tx(bar + TPC + j, tail_bytes);
        bulk_g2s(s_tail, c.tl, tail_bytes, bar + TPC + j);
      }
      tile_prefetch(P, c);
    }

    // ---- 2, 3: chi on the owned cross; owned-node loads in flight meanwhile
    cross_gather<LTS, NTH>(c.h, box, slot, own, c.V, P.ibuf, 0, 0, c.g0, true);
    AMR_PROBE(2);
    double pc[OPT], u0[OPT], u1[OPT];
    owned_loads<OPT, NTH>(P, c, pc, u0, u1);
    if (c.nrow) {  // tile-uniform: the rows overlap the copy runs still in flight
      cp_async_wait<1>();  // slots (and weights) landed
      __syncthreads();
      AMR_PROBE(3);
      if (tail_bytes) mbar_wait(bar + TPC + j, 0);
      cross_rows<NTH>(s_tail, c.nrow, c.taps_off, s_w, slot, box);
    }
    cp_async_wait<0>();
    __syncthreads();
    AMR_PROBE(4);

    // ---- 4: RHS at the owned nodes
    rhs_pass1<DIM, PPO, LTS, NT, NTH, OPT, FULL>(P, c, box, own, pc, u0, u1);
    AMR_PROBE(5);
    if (FULL && c.faces != 0) {
      // ---- 5: physical-face tiles: phi on the owned cross, radiative phi rows
      __syncthreads();  // everyone is done reading chi from the box
      cross_gather<LTS, NTH>(c.h, box, slot, own, c.V, P.ibuf, P.ld, P.n_iface_total, c.g0, false);
      cp_async_wait<0>();
      __syncthreads();
      cross_rows<NTH>(s_tail, c.nrow, c.taps_off, s_w, slot, box);
      __syncthreads();
      rhs_pass2<DIM, PPO, LTS, NT, NTH, OPT>(P, c, box, own, u0, u1);
    }
    if (j + 1 < TPC) __syncthreads();  // box, slots, own map and tail are free for the next tile
    AMR_PROBE(6);
  }
}
