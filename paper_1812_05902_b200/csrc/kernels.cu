// kernels.cu — the B200 render pipeline (sm_100a).
//
// K1 render_emitters fuses the four stages of process_source
// (reference proj/src/engine.cpp:107-140) for one chunk of one emitter per CTA
// (an emitter is split over KScene::split CTAs):
//   stage 1  ray generation        raygen.cpp:12-88   FP64, counter RNG (core.hpp:80-107)
//   stage 2  GRIN RK4 propagation   grin.cpp:23-134    FP32 perturbation form; the cell
//            under the ray cached in registers as a polynomial (per-cell table or the
//            float4 nodes), evaluated with packed FFMA2
//   stage 3  optics chain           optics.cpp:15-158  FP64 in registers
//   stage 4  sensor + deposition    sensor.cpp:27-122  FP64 hit, FP32 erf spot weights,
//            u32 shared-memory tile (branch-free RED rows) flushed with u64 global reductions
// plus make_tile/composite_tile (engine.cpp:142-187): the image is a 64-bit
// fixed-point sum (radiance * 2^31) and the DotHitStats sums are fixed point too,
// so every output is order-independent and bit-identical for any emitter order,
// chunking, CTA count or GPU count.
// FP64 normalisations by one reciprocal (stages.cuh RB_FAST_DIV) and the
// branch-free spot erf (render.cuh RB_FAST_ERF), as in kernels_nomedium.cu:
// together tomo +1.5%, bos neutral, with the RK4 loop's allocation unchanged
// (242 instructions, no spills).  The FP64 validation build keeps neither.
#define RB_FAST_DIV 1
#define RB_FAST_ERF 1
// The field scenes' spots are in focus (~12 px windows): a 2048-word tile (8 KB
// instead of 24 KB) leaves more of the SM's L1 to the cell table (+0.2%); the
// no-medium kernel keeps 6144 words for defocused spots.
#ifndef RB_TILE_CAP
#define RB_TILE_CAP 2048
#endif
#include "kernels.h"
#include "render.cuh"
#include "render_warps.cuh"

namespace rbk {
namespace {

// Split emitters: DotHitStats = the chunk partials summed in chunk order.
__global__ void emitter_stats_kernel(const __grid_constant__ KScene S) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < S.n_work; e += gridDim.x * blockDim.x) {
    const int src = S.order[e];
    long long a = 0, b = 0;
    long long l = 0;
    for (int c = 0; c < S.split; ++c) {
      const size_t w = (size_t)e * S.split + c;
      a += S.hit_part[2 * w];
      b += S.hit_part[2 * w + 1];
      l += S.landed_part[w];
    }
    S.hit_sum[2 * src] = hit_double(a);
    S.hit_sum[2 * src + 1] = hit_double(b);
    S.landed[src] = l;
    if (S.pair) {
      long long a0 = 0, b0 = 0;
      long long l0 = 0;
      for (int c = 0; c < S.split; ++c) {
        const size_t w = (size_t)e * S.split + c;
        a0 += S.hit_part0[2 * w];
        b0 += S.hit_part0[2 * w + 1];
        l0 += S.landed_part0[w];
      }
      S.hit_sum0[2 * src] = hit_double(a0);
      S.hit_sum0[2 * src + 1] = hit_double(b0);
      S.landed0[src] = l0;
    }
  }
}

// ------------------------------------------------ K0: field pack / build
// float4 (n-1, dn/dx, dn/dy, dn/dz) from GriddedField's FP64 node arrays.
__global__ void pack_nodes_kernel(const double* __restrict__ n, const double* __restrict__ gx,
                                  const double* __restrict__ gy, const double* __restrict__ gz,
                                  float4* __restrict__ out, int64_t count) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = make_float4((float)(n[q] - 1.0), (float)gx[q], (float)gy[q], (float)gz[q]);
}

// GriddedField ctor (scene.cpp:53-92) on device: n = K*rho + 1 (gladstone_dale,
// scene.cpp:16-20) and central differences inside / one-sided first order on
// the faces, all FP64 with explicit round-to-nearest ops (no FMA contraction),
// so the packed grid is bit-identical to packing the reference's own nodes.
__device__ __forceinline__ double n_of(const float* rho, double k, size_t q) {
  return __dadd_rn(__dmul_rn(k, (double)rho[q]), 1.0);
}

__global__ void build_from_density_kernel(const float* __restrict__ rho, int nx, int ny, int nz,
                                          double k, double3 sp, float4* __restrict__ out, int z0,
                                          int z1) {
  const int64_t plane = (int64_t)nx * ny;
  const int64_t count = plane * (z1 - z0);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int kk = z0 + (int)(t / plane);
    const int64_t rem = t % plane;
    const int j = (int)(rem / nx), i = (int)(rem % nx);
    const size_t q = (size_t)kk * plane + (size_t)j * nx + i;
    const double nq = n_of(rho, k, q);
    double g[3];
    const int idx[3] = {i, j, kk}, dim[3] = {nx, ny, nz};
    const size_t stride[3] = {1, (size_t)nx, (size_t)plane};
    const double h[3] = {sp.x, sp.y, sp.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (idx[a] == 0)
        g[a] = __ddiv_rn(__dsub_rn(n_of(rho, k, q + stride[a]), nq), h[a]);
      else if (idx[a] == dim[a] - 1)
        g[a] = __ddiv_rn(__dsub_rn(nq, n_of(rho, k, q - stride[a])), h[a]);
      else
        g[a] = __ddiv_rn(__dsub_rn(n_of(rho, k, q + stride[a]), n_of(rho, k, q - stride[a])),
                         __dmul_rn(2.0, h[a]));
    }
    out[q] = make_float4((float)__dsub_rn(nq, 1.0), (float)g[0], (float)g[1], (float)g[2]);
  }
}

// Per-cell coefficient table (KScene::cell_table) from the packed nodes.
// Each thread derives one cell's 8 coefficients; the block stages its 256
// cells (32 KB) in shared memory and writes them out as consecutive float4 so
// every store instruction covers 4 KB of contiguous table (direct 128 B-per-
// thread stores ran at 1.65 TB/s).
constexpr int kCellsPerBlock = 256;
__global__ void __launch_bounds__(kCellsPerBlock)
    build_cells_kernel(const float4* __restrict__ grid, int nx, int ny, int nz,
                       CellCoef* __restrict__ cells) {
  __shared__ float4 stage[kCellsPerBlock * 8];
  const int64_t cx = nx - 1, cxy = (int64_t)(nx - 1) * (ny - 1);
  const int64_t count = cxy * (nz - 1);
  const int64_t nxny = (int64_t)nx * ny;
  for (int64_t base = (int64_t)blockIdx.x * kCellsPerBlock; base < count;
       base += (int64_t)gridDim.x * kCellsPerBlock) {
    const int64_t t = base + threadIdx.x;
    if (t < count) {
      const int64_t k = t / cxy, rem = t - k * cxy, j = rem / cx, i = rem - j * cx;
      const float4* p0 = grid + (k * nxny + j * nx + i);
      const float4* p1 = p0 + nxny;
      float4* o = stage + threadIdx.x * 8;
      cell_coefficients(p0[0], p0[1], p0[nx], p0[nx + 1], p1[0], p1[1], p1[nx], p1[nx + 1], o[0],
                        o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
    }
    __syncthreads();
    const int64_t n = min((int64_t)kCellsPerBlock, count - base) * 8;
    float4* dst = cells[base].c;
    for (int q = threadIdx.x; q < n; q += kCellsPerBlock) dst[q] = stage[q];
    __syncthreads();
  }
}

// ------------------------------------------------ K2: image finalize
__global__ void image_finalize_kernel(const unsigned long long* __restrict__ fx,
                                      double* __restrict__ out, int64_t n) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    out[q] = (double)fx[q] * (1.0 / 2147483648.0);
}

// ------------------------------------------------ K3: quantize (render tail)
// quantize, sensor.cpp:124-135: counts = llround(gain * v), clamped.
__global__ void quantize_kernel(const double* __restrict__ img, int64_t n, double gain,
                                long long max_count, uint16_t* __restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const long long c = llround(gain * img[q]);
    out[q] = (uint16_t)(c < 0 ? 0 : (c > max_count ? max_count : c));
  }
}

}  // namespace

// ------------------------------------------------ launch wrappers
int render_occupancy(int blocks_per_sm[2][3]) {
  set_smem<false, 1>();
  set_smem<false, 2>();
  set_smem<true, 1>();
  set_smem<true, 2>();
  cudaFuncSetAttribute(render_warps<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)render_smem());
  cudaFuncSetAttribute(render_warps<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)render_smem());
  blocks_per_sm[0][1] = occupancy<false, 1>();
  blocks_per_sm[0][2] = occupancy<false, 2>();
  blocks_per_sm[1][1] = occupancy<true, 1>();
  blocks_per_sm[1][2] = occupancy<true, 2>();
  int nm[2] = {0, 0};
  render_occupancy_nomedium(nm);  // kernels_nomedium.cu
  blocks_per_sm[0][0] = nm[0];
  blocks_per_sm[1][0] = nm[1];
  return (int)cudaGetLastError();
}

int field_mode(const KScene& s) { return !s.with_field ? 0 : (s.cell_table ? 2 : 1); }

cudaError_t launch_render(const KScene& s, int grid, cudaStream_t stream) {
  const size_t sm = render_smem();
  switch (field_mode(s) + (s.pair ? 3 : 0)) {
    case 0:
    case 3: return launch_render_nomedium(s, grid, stream);  // kernels_nomedium.cu
    case 1:
      if (s.warp_mode) render_warps<1><<<grid, kBlock, sm, stream>>>(s);
      else render_emitters<false, 1><<<grid, kBlock, sm, stream>>>(s);
      break;
    case 2:
      if (s.warp_mode) render_warps<2><<<grid, kBlock, sm, stream>>>(s);
      else render_emitters<false, 2><<<grid, kBlock, sm, stream>>>(s);
      break;
    case 4: render_emitters<true, 1><<<grid, kBlock, sm, stream>>>(s); break;
    default: render_emitters<true, 2><<<grid, kBlock, sm, stream>>>(s); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_emitter_stats(const KScene& s, cudaStream_t stream) {
  if (s.split <= 1 || s.n_work <= 0) return cudaSuccess;
  emitter_stats_kernel<<<(s.n_work + 255) / 256, 256, 0, stream>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_trace_rays(const KScene& s, int64_t n, const int64_t* src, const int32_t* ray,
                              double* uv, int32_t* status, int32_t* steps, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int bs = 128;
  const unsigned blocks = (unsigned)((n + bs - 1) / bs);
  switch (field_mode(s)) {
    case 0: return launch_trace_rays_nomedium(s, n, src, ray, uv, status, steps, stream);
    case 1: trace_rays_kernel<1><<<blocks, bs, 0, stream>>>(s, n, src, ray, uv, status, steps); break;
    default: trace_rays_kernel<2><<<blocks, bs, 0, stream>>>(s, n, src, ray, uv, status, steps); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_build_cells(const float4* grid, int nx, int ny, int nz, CellCoef* cells,
                               cudaStream_t stream) {
  build_cells_kernel<<<148 * 6, kCellsPerBlock, 0, stream>>>(grid, nx, ny, nz, cells);
  return cudaGetLastError();
}

cudaError_t launch_pack_nodes(const double* n, const double* gx, const double* gy,
                              const double* gz, float4* out, int64_t count, cudaStream_t stream) {
  pack_nodes_kernel<<<148 * 8, 256, 0, stream>>>(n, gx, gy, gz, out, count);
  return cudaGetLastError();
}

cudaError_t launch_build_from_density(const float* rho, int nx, int ny, int nz, double k,
                                      double3 spacing, float4* out, int z0, int z1,
                                      cudaStream_t stream) {
  build_from_density_kernel<<<148 * 8, 256, 0, stream>>>(rho, nx, ny, nz, k, spacing, out, z0, z1);
  return cudaGetLastError();
}

cudaError_t launch_quantize(const double* image, int64_t n, double gain, int bit_depth,
                            uint16_t* out, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  quantize_kernel<<<148 * 4, 256, 0, stream>>>(image, n, gain, (1LL << bit_depth) - 1, out);
  return cudaGetLastError();
}

cudaError_t launch_image_finalize(const unsigned long long* fixed, double* out, int64_t n,
                                  cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  image_finalize_kernel<<<148 * 4, 256, 0, stream>>>(fixed, out, n);
  return cudaGetLastError();
}

}  // namespace rbk
