// amr_stage_pipe.cuh — the persistent, software-pipelined stage kernel
// (included by amr_kernels.cu inside its anonymous namespace).
//
// Each CTA walks the tiles blockIdx.x, +gridDim.x, ... (2 CTAs per SM).  For
// tile j it
//   * bulk-copies the head of the tile's program blob (tileprog.py: header,
//     source bases, entry and slot codes) into a 3-slot smem ring two tiles
//     ahead (one thread, mbarrier completion), and bulk-prefetches the rows
//     and taps of the blob into L2;
//   * two tiles ahead, issues every field gather of the tile: 8-byte cp.async
//     copies along the tile's copy runs (z-consecutive box cells from
//     consecutive source nodes) straight into the stencil box (no register
//     staging) and per interpolation source, plus bulk copies of the
//     contiguous owned ranges (u chi/phi, stage-source phi) and of the blob's
//     rows and taps — so the loads of tile j+2 are in flight while tiles j+1
//     (rows) and j (RHS) compute;
//   * computes tile j: hanging rows from the slot values (rows/taps read
//     through L2), RHS at the owned nodes, K_s / next-stage sources / RK
//     combine out.
// Arithmetic is that of stage_kernel (same operation order; a copy row's
// "0 + src" only changes the sign of a zero, which no later operation turns
// into a nonzero difference).
//
// Field arrays have an even row stride P.ld (16-byte aligned rows), so a
// tile's owned range can be bulk-copied from the 16-byte aligned superset
// [g0 & ~1, (g0 + n_own + 1) & ~1).

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}

template <int DIM, int PPO>
struct Pipe {
  using T = Tile<DIM, PPO>;
  static constexpr int THREADS = DIM == 3 ? 256 : 128;
  static constexpr int MIN_CTAS = 2;  // two independent CTAs per SM: their phases interleave
  static constexpr int NG = 3;  // gather buffers: tile landing, tile in its row phase, tile in its RHS phase
  static constexpr int NB = 2;  // blob-head ring slots (a head is consumed when its tile's gathers issue)
  static constexpr int HEAD = 64 + 64 * 8;  // mbarriers, interpolation weights
  static constexpr int BOXB = (T::NS * 8 + 15) / 16 * 16;     // the stencil box
  static constexpr int HPHB = (T::NI * 8 + 15) / 16 * 16;     // face tiles: phi of the hanging rows
  static constexpr int OWNC = (T::NI * 4 + 15) / 16 * 16;     // owned node -> box cell
  static constexpr int HDRB = (16 + 64) * 4;                   // the tile's header + source bases
  // gather buffer: box chi | hanging-row phi | slot chi, slot phi | owned cells | header
  __host__ __device__ static int slot_bytes(int max_slots) { return ((max_slots + 1) * 8 + 15) / 16 * 16; }
  __host__ __device__ static int gbuf_bytes(int max_slots) {
    return BOXB + HPHB + 2 * slot_bytes(max_slots) + OWNC + HDRB;
  }
  __host__ __device__ static size_t smem_bytes(int max_slots, int max_head) {
    return HEAD + (size_t)NG * gbuf_bytes(max_slots) + (size_t)NB * max_head;
  }
};

template <int DIM, int PPO>
struct AccI {  // interior fast path: chi from the box, phi of the node
  const double* chi;
  double phi;
  int cell;
  __device__ __forceinline__ double at(int v, int d, int o) const {
    constexpr int NP = Tile<DIM, PPO>::NP;
    const int stride = (DIM == 3) ? (d == 0 ? NP * NP : (d == 1 ? NP : 1)) : (d == 0 ? NP : 1);
    return v == 0 ? chi[cell + o * stride] : phi;
  }
};

// general path (physical faces, coordinate-dependent sources).  Face tiles read
// phi through the tile's entry codes: copies / interface sources from global
// memory, hanging rows from hph, outside = 0.
template <int DIM, int PPO>
struct AccF {
  const double* chi;
  const double* hph;
  const uint16_t* ent;
  const int* bases;
  const uint16_t* cell_ent;
  const double* V;
  const double* IB;
  int64_t n, nib;
  double phi;  // phi of the node (non-face tiles)
  int cell;
  bool face;
  __device__ __forceinline__ double phi_at(int c) const {
    const int e = __ldg(cell_ent + c);
    const int code = ent[e];
    const int bi = code >> 10, off = code & 1023;
    if (bi == 63) return off == 0 ? 0.0 : hph[off - 1];
    const int base = bases[bi];
    return base >= 0 ? __ldg(V + n + base + off) : __ldg(IB + nib + (-base - 1 + off));
  }
  __device__ __forceinline__ double at(int v, int d, int o) const {
    constexpr int NP = Tile<DIM, PPO>::NP;
    const int stride = (DIM == 3) ? (d == 0 ? NP * NP : (d == 1 ? NP : 1)) : (d == 0 ? NP : 1);
    if (v == 0) return chi[cell + o * stride];
    return face ? phi_at(cell + o * stride) : phi;
  }
};

// RHS at one owned node of a tile on a physical face or with a
// coordinate-dependent source (rare): out of line, so its registers do not
// weigh on the fast path.  h = the tile's header + bases.
template <int DIM, int PPO>
__device__ __noinline__ double2 rhs_general(const AmrStageParams* Pp, const double* box, const double* hph,
                                            const uint16_t* ent, const int* h, const double* V, int cell,
                                            double ph) {
  using T = Tile<DIM, PPO>;
  const AmrStageParams& P = *Pp;
  const int lmeta = h[2];
  const int lvl = lmeta & 0xFF;
  const int faces = (lmeta >> 16) & 0x3F;
  RhsConst R;
  R.h = P.h[lvl];
  R.h2 = P.h2[lvl];
  R.inv_h2 = P.inv_h2[lvl];
  R.pow2 = P.h2_pow2[lvl] != 0;
  R.nonlinear = P.nonlinear;
  R.r_eps = P.r_eps;
  R.r_eps2 = P.r_eps2;
  R.k_chi = P.k_chi;
  R.k_phi = P.k_phi;
  R.f0_chi = P.f0_chi;
  R.f0_phi = P.f0_phi;
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
  AccF<DIM, PPO> acc{box, hph, ent, h + 16, P.cell_ent, V, P.ibuf, P.ld, P.n_iface_total, ph, cell, faces != 0};
  return rhs_point<DIM>(acc, pos, PPO, faces, x, P, R);
}

template <int DIM, int PPO, bool LTS, int NT>
__global__ void __launch_bounds__(Pipe<DIM, PPO>::THREADS, Pipe<DIM, PPO>::MIN_CTAS)
    stage_pipe(const __grid_constant__ AmrStageParams P) {
  using T = Tile<DIM, PPO>;
  using PP = Pipe<DIM, PPO>;
  constexpr int NTH = PP::THREADS;
  constexpr int NG = PP::NG;
  constexpr int NB = PP::NB;
  constexpr int OPT = (T::NI + NTH - 1) / NTH;
  constexpr int NW = NTH / 32;
  constexpr int PROD = NTH - 32;  // the producer lane (bulk copies, prefetches): lane 0 of the last warp
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* bbar = reinterpret_cast<uint64_t*>(smem);  // [NB] blob heads
  double* s_w = reinterpret_cast<double*>(smem + 64);
  const int sb = PP::slot_bytes(P.max_slots);
  const int gstride = PP::gbuf_bytes(P.max_slots);
  unsigned char* const gbase = smem + PP::HEAD;
  unsigned char* const bbase = gbase + NG * gstride;
  const int bstride = P.max_blob;
  // gather-buffer section offsets
  const int o_hph = PP::BOXB, o_slc = o_hph + PP::HPHB, o_slp = o_slc + sb, o_own = o_slp + sb;
  const int o_hdr = o_own + PP::OWNC;
  const int tid = threadIdx.x;
  const int64_t n = P.ld;
  const int s = P.stage;
  const bool last = (s == P.n_stages - 1);
  const double* IB = P.ibuf;
  const int64_t nib = P.n_iface_total;
  const AmrSliceCoef* C = P.coef;
  const uint16_t* blob = P.blob;
  const double* Ys = P.Y + (int64_t)(s & 1) * 2 * n;  // this stage's verbatim sources (s > 0)
  const int n_my = (int)((P.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
  if (n_my <= 0) return;

  for (int i = tid; i < P.n_wtab; i += NTH) s_w[i] = P.wtab[i];
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&bbar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---- producer lane: bulk copy of blob head j into ring slot j % NB -----------
  auto issue_blob = [&](int j, int64_t off, int head) {
    const int b = j % NB;
    mbar_expect_tx(&bbar[b], (uint32_t)head);
    bulk_g2s(bbase + b * bstride, reinterpret_cast<const unsigned char*>(blob) + off, (uint32_t)head, &bbar[b]);
  };

  // ---- all threads: every gather of tile j (its head has landed) ----------------
  auto issue_gathers = [&](int j) {
    const unsigned char* B = bbase + (j % NB) * bstride;
    const int* h = reinterpret_cast<const int*>(B);
    const int g0 = h[0], n_own = h[1], lmeta = h[2], nrun = h[3], nslot = h[4], nbase = h[6];
    const int* bases = h + 16;
    const uint16_t* sl = reinterpret_cast<const uint16_t*>(B) + h[12];
    const int cad = (lmeta >> 8) & 0xFF;
    const bool face = ((lmeta >> 16) & 0x3F) != 0;
    const int cur = LTS ? C->cur[cad] : P.gts_cur;
    const double* Ucur = cur ? P.U1 : P.U0;
    const double* V = (s == 0) ? Ucur : Ys;
    unsigned char* G = gbase + (j % NG) * gstride;
    double* box = reinterpret_cast<double*>(G);
    double* slc = reinterpret_cast<double*>(G + o_slc);
    double* slp = reinterpret_cast<double*>(G + o_slp);
    int* own = reinterpret_cast<int*>(G + o_own);
    int* hdr = reinterpret_cast<int*>(G + o_hdr);
    // the header and bases stay with the gather buffer (the head slot is reused)
    if (tid < 16 + nbase) hdr[tid] = h[tid];
    if (tid == PROD) {
      // warm L2 for what the later phases read from global memory: the blob
      // tail (face entry codes, rows, taps), the owned ranges of u and of the
      // stage-source phi, and (last stage) the K_j of the combine
      const int64_t a16 = g0 & ~1, e16 = (g0 + n_own + 1) & ~1;
      const uint32_t bytes = (uint32_t)(e16 - a16) * 8;
      const uint32_t tail = 2u * (uint32_t)(h[7] - h[11]);
      if (tail) bulk_prefetch_l2(blob + (int64_t)h[15] * 8 + h[11], tail);
      bulk_prefetch_l2(Ucur + a16, bytes);
      bulk_prefetch_l2(Ucur + n + a16, bytes);
      if (s != 0) bulk_prefetch_l2(V + n + a16, bytes);
      if (last)
        for (int jj = 0; jj < s; ++jj) {
          bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + a16, bytes);
          bulk_prefetch_l2(P.K + (int64_t)jj * 2 * n + n + a16, bytes);
        }
    }
    if (P.dbg_skip & 1) return;
    // copy runs: z-consecutive box cells from consecutive source nodes
    const uint32_t* runs = reinterpret_cast<const uint32_t*>(bases + ((nbase + 3) & ~3));
    for (int r = tid; r < nrun; r += NTH) {
      const uint32_t w = runs[r];
      const int cell = w & 0xFFF, len = ((w >> 12) & 15) + 1;
      const int bi = w >> 26, off = (w >> 16) & 1023;
      double* dst = box + cell;
      if (bi == 63) {  // outside the domain: zero rows
        for (int i = 0; i < len; ++i) dst[i] = 0.0;
        continue;
      }
      const int base = bases[bi];
      if (!LTS || base >= 0) {
        const double* src = V + base + off;
        for (int i = 0; i < len; ++i) cp_async8(dst + i, src + i);
        if (base == g0)
          for (int i = 0; i < len; ++i) own[off + i] = cell + i;
      } else {
        const double* src = IB + (-base - 1 + off);
        for (int i = 0; i < len; ++i) cp_async8(dst + i, src + i);
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
  };

  // ---- row phase of tile j: hanging rows, 0 + sum_k w_k src(g_k) in
  //      ascending-gid order (mesh.py:316-351).  Rows are stored longest first
  //      and dealt round-robin over the warps (row lane*NW + warp, + NTH); the
  //      row words and taps are read through L2.
  auto rows_phase = [&](int j) {
    unsigned char* G = gbase + (j % NG) * gstride;
    const int* h = reinterpret_cast<const int*>(G + o_hdr);
    const int nrow = h[5];
    const int r0 = (tid & 31) * NW + (tid >> 5);
    if (r0 >= nrow) return;
    const bool face = ((h[2] >> 16) & 0x3F) != 0;
    double* box = reinterpret_cast<double*>(G);
    double* hph = reinterpret_cast<double*>(G + o_hph);
    const double* slc = reinterpret_cast<const double*>(G + o_slc);
    const double* slp = reinterpret_cast<const double*>(G + o_slp);
    const uint16_t* gblob = blob + (int64_t)h[15] * 8;
    const uint32_t* rows = reinterpret_cast<const uint32_t*>(gblob + h[13]);
    const uint2* taps = reinterpret_cast<const uint2*>(gblob + h[14]);
    for (int r = r0; r < nrow; r += NTH) {
      const uint32_t w = __ldg(rows + r);
      const int nq = (w >> 12) & 31;
      const uint2* tq = taps + (w >> 17);
      double ax = 0.0, ay = 0.0;
      uint2 v = nq > 0 ? __ldg(tq) : make_uint2(0u, 0u);
      for (int q = 0; q < nq; ++q) {
        const uint2 vn = q + 1 < nq ? __ldg(tq + q + 1) : v;  // next tap word in flight
        const uint32_t t4[4] = {v.x & 0xFFFF, v.x >> 16, v.y & 0xFFFF, v.y >> 16};
        double pc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pc[u] = s_w[t4[u] & 63] * slc[t4[u] >> 6];
#pragma unroll
        for (int u = 0; u < 4; ++u) ax = ax + pc[u];
        if (face) {
#pragma unroll
          for (int u = 0; u < 4; ++u) ay = ay + s_w[t4[u] & 63] * slp[t4[u] >> 6];
        }
        v = vn;
      }
      box[w & 0xFFF] = ax;
      if (face) hph[r] = ay;
    }
  };

  // ---- RHS phase of tile j: owned nodes k = tid (+ NTH); u and the stage-source
  //      phi of the node come from global memory (L2-warm); K_s / next-stage
  //      source / RK combine out
  const Weights& W = P;
  auto rhs_phase = [&](int j) {
    unsigned char* G = gbase + (j % NG) * gstride;
    const int* h = reinterpret_cast<const int*>(G + o_hdr);
    const int g0 = h[0], n_own = h[1], lmeta = h[2];
    const int lvl = lmeta & 0xFF;
    const int cad = (lmeta >> 8) & 0xFF;
    const int faces = (lmeta >> 16) & 0x3F;
    const bool face = faces != 0;
    const int cur = LTS ? C->cur[cad] : P.gts_cur;
    const double* box = reinterpret_cast<const double*>(G);
    const int* own = reinterpret_cast<const int*>(G + o_own);
    const double* Ucur = cur ? P.U1 : P.U0;
    const double* V = (s == 0) ? Ucur : Ys;
    double* Unew = cur ? P.U0 : P.U1;
    double* Ks = P.K + (int64_t)s * 2 * n;
    RhsConst R;
    R.h2 = P.h2[lvl];
    R.inv_h2 = P.inv_h2[lvl];
    R.pow2 = P.h2_pow2[lvl] != 0;
    R.nonlinear = P.nonlinear;
    const bool need_x = face || P.nonlinear == 1;
#pragma unroll 1
    for (int r = 0; r < OPT; ++r) {
      const int k = tid + r * NTH;
      if (k >= n_own) break;
      const int64_t g = g0 + k;
      const int cell = own[k];
      // node values from global memory (L2-warm), issued before the stencil
      const double uc = __ldg(Ucur + g), up = __ldg(Ucur + n + g);
      const double ph = __ldg(V + n + g);
      double2 ks;
      if (!need_x && R.pow2) {
        const double* b = box + cell;
        double dphi = lap_pow2<DIM, PPO>(b, W, R.inv_h2);
        if (P.nonlinear == 2) {
          const double chi = b[0];
          dphi = dphi - (chi * chi) * chi;
        }
        ks = make_double2(ph, dphi);
      } else if (!need_x) {
        ks = rhs_interior<DIM>(AccI<DIM, PPO>{box, ph, cell}, W, R);
      } else {
        ks = rhs_general<DIM, PPO>(&P, box, reinterpret_cast<const double*>(G + o_hph),
                                   blob + (int64_t)h[15] * 8 + h[11], h, V, cell, face ? 0.0 : ph);
      }
      if (!last || LTS) {
        Ks[g] = ks.x;
        Ks[n + g] = ks.y;
      }
      if (!last) {  // next stage's verbatim source of this owned node
        double yx = 0.0 + uc, yy = 0.0 + up;
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
        double ux = 0.0 + uc, uy = 0.0 + up;
#pragma unroll
        for (int jj = 0; jj < AMR_MAXP; ++jj) {
          if (jj > s) break;
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
  };

  // ---- the pipeline -------------------------------------------------------------
  // iteration j: head of j+3 issued; gathers of j+2 issued; rows of j+1 and RHS
  // of j computed together (different buffers: no barrier between them)
  const int64_t* boff = P.blob_off;
  const int* bhead = P.blob_head;
  auto tile_of = [&](int j) { return (int64_t)blockIdx.x + (int64_t)j * gridDim.x; };
  auto wait_head = [&](int j) { mbar_wait(&bbar[j % NB], (j / NB) & 1); };
  int64_t nx_off = 0;  // producer lane: blob head of the tile issued next, loaded one iteration early
  int nx_head = 0;
  if (tid == PROD) {
    for (int j = 0; j < 2 && j < n_my; ++j) issue_blob(j, __ldg(boff + tile_of(j)), __ldg(bhead + tile_of(j)));
    if (n_my > 2) {
      nx_off = __ldg(boff + tile_of(2));
      nx_head = __ldg(bhead + tile_of(2));
    }
  }
  wait_head(0);
  issue_gathers(0);
  cp_async_commit();
  if (n_my > 1) {
    wait_head(1);
    issue_gathers(1);
  }
  cp_async_commit();
  cp_async_wait<1>();
  __syncthreads();  // gathers of tile 0 visible; head slots 0 and 1 consumed
  if (tid == PROD && n_my > 2) {
    issue_blob(2, nx_off, nx_head);
    if (n_my > 3) {
      nx_off = __ldg(boff + tile_of(3));
      nx_head = __ldg(bhead + tile_of(3));
    }
  }
  rows_phase(0);
  __syncthreads();
  long long ph[6] = {0, 0, 0, 0, 0, 0};
  const bool dbg = P.dbg != nullptr;
  for (int j = 0; j < n_my; ++j) {
    long long c0 = dbg ? clock64() : 0;
    if (tid == PROD && j + 3 < n_my) {  // slot (j+3)%2 held head j+1, consumed last iteration
      issue_blob(j + 3, nx_off, nx_head);
      if (j + 4 < n_my) {
        nx_off = __ldg(boff + tile_of(j + 4));
        nx_head = __ldg(bhead + tile_of(j + 4));
      }
    }
    if (j + 2 < n_my) {
      wait_head(j + 2);
      issue_gathers(j + 2);
    }
    cp_async_commit();
    long long c1 = dbg ? clock64() : 0;
    cp_async_wait<1>();
    long long c2 = dbg ? clock64() : 0;
    __syncthreads();
    long long c3 = dbg ? clock64() : 0;
    if (j + 1 < n_my && !(P.dbg_skip & 2)) rows_phase(j + 1);
    long long c4 = dbg ? clock64() : 0;
    if (!(P.dbg_skip & 4)) rhs_phase(j);
    long long c5 = dbg ? clock64() : 0;
    __syncthreads();
    if (dbg) {
      const long long c6 = clock64();
      ph[0] += c1 - c0;
      ph[1] += c2 - c1;
      ph[2] += c3 - c2;
      ph[3] += c4 - c3;
      ph[4] += c5 - c4;
      ph[5] += c6 - c5;
    }
  }
  if (dbg && (tid & 31) == 0) {
    long long* o = P.dbg + ((int64_t)blockIdx.x * NW + tid / 32) * 8;
#pragma unroll
    for (int i = 0; i < 6; ++i) o[i] += ph[i];  // summed over the launches of a slice
    o[6] += n_my;
  }
}
