// amr_stage_inst.cu — one instance of the stage kernel launcher per
// (dimension, points per octant, LTS) triple: build.py compiles this file once
// per triple with -DAMR_INST_DIM/-DAMR_INST_PPO/-DAMR_INST_LTS, in parallel.
#include "amr_common.cuh"

namespace {
#include "amr_async.cuh"
#include "amr_stage_cross.cuh"

// per-device launch state (a process may drive several GPUs)
constexpr int kMaxDev = 64;

template <int DIM, int PPO, bool LTS, int NT, int NTH, bool FULL>
int launch_cross_one(const AmrStageParams* p, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= kMaxDev) return AMR_EINVAL;
  using CK = CrossK<DIM, PPO>;
  const size_t dyn = CK::smem_bytes(p->max_slots, p->max_head, p->max_tail, AMR_TPC);
  static size_t configured[kMaxDev] = {0};
  if (dyn > configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(stage_cross<DIM, PPO, LTS, NT, NTH, FULL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(stage_cross)");
    configured[dev] = dyn;
  }
  return pdl_launch(stage_cross<DIM, PPO, LTS, NT, NTH, FULL>, dim3((unsigned)((p->n_tiles + AMR_TPC - 1) / AMR_TPC)), dim3(NTH), dyn, st, *p);
}

template <int DIM, int PPO, bool LTS, int NTH, bool FULL>
int launch_cross_nt(const AmrStageParams* p, cudaStream_t st) {
  switch (p->n_vt) {
    case 0: return launch_cross_one<DIM, PPO, LTS, 0, NTH, FULL>(p, st);
    case 1: return launch_cross_one<DIM, PPO, LTS, 1, NTH, FULL>(p, st);
    case 2: return launch_cross_one<DIM, PPO, LTS, 2, NTH, FULL>(p, st);
    case 3: return launch_cross_one<DIM, PPO, LTS, 3, NTH, FULL>(p, st);
    default: return AMR_EINVAL;
  }
}

template <int DIM, int PPO, bool LTS>
int launch_stage_nt(const AmrStageParams* p, cudaStream_t st) {
  if (p->lean) {  // the caller vouches: no physical face, no coordinate-dependent source
    if (p->nonlinear == 1) return AMR_EINVAL;
    if (p->threads == 256) return launch_cross_nt<DIM, PPO, LTS, 256, false>(p, st);
    return launch_cross_nt<DIM, PPO, LTS, AMR_ALT_NTH, false>(p, st);
  }
  if (p->threads == 256) return launch_cross_nt<DIM, PPO, LTS, 256, true>(p, st);
  return launch_cross_nt<DIM, PPO, LTS, AMR_ALT_NTH, true>(p, st);
}

}  // namespace

#define AMR_CAT(a, b, c) amr_stage_launch_##a##_##b##_##c
#define AMR_NAME(a, b, c) AMR_CAT(a, b, c)
#if AMR_INST_LTS
#define AMR_SUFFIX l
#else
#define AMR_SUFFIX g
#endif
int AMR_NAME(AMR_INST_DIM, AMR_INST_PPO, AMR_SUFFIX)(const AmrStageParams* p, cudaStream_t st) {
  return launch_stage_nt<AMR_INST_DIM, AMR_INST_PPO, (AMR_INST_LTS != 0)>(p, st);
}
