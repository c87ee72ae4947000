// kernels_nomedium.cu — K1 for scenes without a medium (render_emitters with
// kField = 0 and its per-ray replay), compiled apart from kernels.cu so its
// code-size choices (rolled off-tile spot rows and thick-lens surfaces,
// RB_COMPACT_*: the no-medium kernel is instruction-cache bound) cannot perturb
// the register allocation of the RK4 loop the field instantiations carry.
// Both units use the FP64 reciprocal normalisations (RB_FAST_DIV, stages.cuh)
// and the branch-free spot erf (RB_FAST_ERF, render.cuh: piv +5%, optics +8.5%).
#define RB_FAST_DIV 1
#define RB_FAST_ERF 1
#define RB_COMPACT_SLOW_ROWS 1
#define RB_COMPACT_OPTICS 1
#include "kernels.h"
#include "render.cuh"

namespace rbk {

int render_occupancy_nomedium(int blocks_per_sm[2]) {
  set_smem<false, 0>();
  set_smem<true, 0>();
  blocks_per_sm[0] = occupancy<false, 0>();
  blocks_per_sm[1] = occupancy<true, 0>();
  return (int)cudaGetLastError();
}

cudaError_t launch_render_nomedium(const KScene& s, int grid, cudaStream_t stream) {
  const size_t sm = render_smem();
  if (s.pair)
    render_emitters<true, 0><<<grid, kBlock, sm, stream>>>(s);
  else
    render_emitters<false, 0><<<grid, kBlock, sm, stream>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_trace_rays_nomedium(const KScene& s, int64_t n, const int64_t* src,
                                       const int32_t* ray, double* uv, int32_t* status,
                                       int32_t* steps, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int bs = 128;
  trace_rays_kernel<0><<<(unsigned)((n + bs - 1) / bs), bs, 0, stream>>>(s, n, src, ray, uv,
                                                                        status, steps);
  return cudaGetLastError();
}

}  // namespace rbk
