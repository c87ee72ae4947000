// kernels.h — device-side scene layout and launch entry points of the
// B200 render pipeline (K0 field_pack/field_build, K1 render_emitters,
// K2 image_finalize, plus the per-ray replay kernel).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rbk {

constexpr int kMaxElements = 8;
#ifndef RB_BLOCK
#define RB_BLOCK 256
#endif
#ifndef RB_MINB
#define RB_MINB 2
#endif
constexpr int kBlock = RB_BLOCK;     // threads per CTA (one emitter chunk at a time)
constexpr int kMinBlocks = RB_MINB;  // resident CTAs per SM the register budget targets
#ifndef RB_MINB_NOFIELD
#define RB_MINB_NOFIELD 4  // measured: 2 -> 4 CTAs/SM is +24% optics, +15% piv
#endif
constexpr int kMinBlocksNoField = RB_MINB_NOFIELD;  // the same for scenes without a medium
#ifndef RB_MINB_CELLS
#define RB_MINB_CELLS 3  // cell-table GRIN loop fits 80 registers: bos +3.5%, 1024^3 +5% (not pair mode)
#endif
constexpr int kMinBlocksCells = RB_MINB_CELLS;  // ... and for fields read from the cell table
#ifndef RB_TILE_CAP
#define RB_TILE_CAP 6144
#endif
constexpr int kTileCap = RB_TILE_CAP;  // u32 entries of the per-emitter shared tile (24 KB)
#ifndef RB_MAX_SPOT
#define RB_MAX_SPOT 12  // 16 measured 10-40% slower (code size); bench spots are <= 11 wide
#endif
constexpr int kMaxSpot = RB_MAX_SPOT;  // register fast path: spot windows up to this many columns

// raybos::SphericalSurface with the derived quantities intersect_sphere
// recomputes on every call (optics.cpp:34-57) hoisted to the host.
struct DSurface {
  double3 vertex, axis, center;  // center = vertex + axis * R   (optics.hpp:35)
  double R, absR, aperture, n_before, n_after;
  int planar;                    // !isfinite(R)                  (optics.hpp:34)
  int pad;
};

// One grid cell's trilinear interpolant in polynomial form (grin.cuh CellPoly):
// coefficients a..h of a + b fx + c fy + d fz + e fx fy + f fx fz + g fy fz +
// h fx fy fz for the four channels.  128 B = one L1/L2 line per cell.
struct __align__(128) CellCoef {
  float4 c[8];
};

struct DElement {
  int kind, pad;
  double3 center, axis;
  double radius, focal, half_diameter;
  DSurface front, back;
};

// Everything K1 reads, passed by value (param space / constant bank).
struct KScene {
  // sources and work list
  const double* sources;         // 3 * n_sources
  const int64_t* source_ids;     // RNG stream per source (may be null = index)
  const int32_t* order;          // queue position -> source index (owned sources only)
  int64_t n_sources;
  int32_t n_work;                // entries in order[]
  int32_t pad0;
  // ray generation (raygen.cpp:27-88)
  double3 pupil_center, e1, e2;
  double pupil_radius;
  double radiance;               // 1/N exactly (raygen.cpp:86)
  uint64_t key_seed;             // mix_bits(seed ^ 0xa93c0de5) (core.hpp:93-94)
  int32_t rays;                  // N
  int32_t cells;                 // ceil(sqrt(N))
  int32_t sampling;
  int32_t with_field;
  // warp patches: the pupil lattice (cells x rows, ray i = cy * cells + cx) is
  // cut into bands of band_h rows (the last one band_tail rows), each
  // enumerated column-major, so 32 consecutive band positions are a compact
  // (32 / band_h) x band_h block whose rays gather from the same few grid cells,
  // and no lane idles where cells is not a multiple of the block width (only
  // the warps that straddle two bands are split); see make_kscene for the
  // patch order.
  int32_t band_rays;             // band_h * cells
  int32_t patch_count;
  int32_t patch_stride;          // coprime to patch_count (1 with a medium)
  int32_t band_h;                // rows per band: 4, 8 or 16
  int32_t band_sh;               // log2(band_h)
  int32_t band_full;             // bands of band_h rows
  int32_t band_tail;             // rows of the last, partial band (0: none)
  int32_t pad_band;
  // density grid (float4: n-1, dn/dx, dn/dy, dn/dz)
  const float4* grid;
  // optional per-cell coefficient table (nullptr = derive from the nodes)
  const CellCoef* cell_table;
  unsigned c_nx, c_nxny;         // cell strides: nx - 1, (nx - 1) * (ny - 1)
  int32_t nx, ny, nz, max_steps;
  double3 origin, spacing, box_lo, box_hi;
  double h;
  // scene-uniform GRIN constants (host-computed; read as constant-bank operands
  // so they take no registers in the RK4 loop)
  unsigned g_nx, g_nxny, g_ix, g_iy, g_iz;  // strides, last cell index per axis
  float g_mx, g_my, g_mz;                   // n - 1 per axis (box in grid coordinates)
  float hx, hy, hz;                         // h / spacing          (dt -> dr)
  float hhx, hhy, hhz;                      // h / spacing / 2
  float kbx, kby, kbz;                      // h^2 / spacing / 8    (a/8 h)
  float kcx, kcy, kcz;                      // h^2 / spacing / 2    (b/2 h)
  float krx, kry, krz;                      // h^2 / spacing / 6    ((a+2b)/6 h)
  float kt;                                 // h / 6                ((a+4b+c)/6)
  float pad_g;
  // optics (optics.cpp:143-158)
  int32_t n_elem, pad1;
  DElement elem[kMaxElements];
  // sensor (sensor.cpp:27-122)
  double3 s_center, s_normal, s_eu, s_ev;
  int32_t W, H;
  double pitch, sigma, half_width, inv_s;
  double hit_limit;                 // |u|, |v| bound keeping a bundle's fixed-point hit sum in int64
  float inv_s_f;                    // inv_s in FP32 (render.cuh spot_erf)
  float pad_s;
  int32_t accumulate, degenerate;   // degenerate: sigma < 1e-3 * pitch
  // outputs
  unsigned long long* image;        // W*H fixed point (radiance * 2^31)
  double* hit_sum;                  // 2 * n_sources
  long long* landed;                // n_sources
  unsigned long long* counters;     // [0..4] lost, aperture, miss, tir, sensor_miss; [5] steps
  int* queue;                       // work counter
  int* err_flag;
  unsigned* check_fail;             // checked build (RB_CHECKED): [0] violations, [1] last site
  unsigned n_cells;                 // cells of the table (checked build's index bound)
  // bos_run pair mode: also follow every emitted ray without the field and
  // accumulate that leg's DotHitStats / counters here (no image)
  int32_t pair, pad_pair;
  double* hit_sum0;
  long long* landed0;
  unsigned long long* counters0;
  // emitter split: `split` CTAs share one emitter's rays (fewer distinct cones
  // in flight -> a smaller L2 working set); each writes its DotHitStats partial
  // to part[work * split + chunk] and emitter_stats_kernel sums them in chunk
  // order (deterministic).  split == 1 writes hit_sum / landed directly.
  int32_t split;
  int32_t warp_mode;                // 1: render_warps (warp-level items; split = items per emitter)
  long long* hit_part;              // 2 * n_work * split, fixed point (render.cuh kHitScale)
  long long* landed_part;
  long long* hit_part0;
  long long* landed_part0;
};

// FP64 GriddedField nodes for the validation build (kernels_fp64.cu).
struct Field64 {
  const double *n, *gx, *gy, *gz;
  int nx, ny, nz, pad;
  double3 origin, spacing, lo, hi;
};

// ---- launches (all on `stream`) ----
cudaError_t launch_trace_rays_fp64(const KScene& s, const Field64& f, int64_t n, const int64_t* src,
                                   const int32_t* ray, double* uv, int32_t* status,
                                   int32_t* steps, cudaStream_t stream);
cudaError_t launch_source_stats_fp64(const KScene& s, const Field64& f, cudaStream_t stream);
cudaError_t launch_trace_debug(const KScene& s, const Field64& f, int64_t src, int ray,
                               double* rec, int64_t cap, int64_t* n_rec, cudaStream_t stream);
cudaError_t launch_quantize(const double* image, int64_t n, double gain, int bit_depth,
                            uint16_t* out, cudaStream_t stream);
cudaError_t launch_build_fp64(const float* rho, int nx, int ny, int nz, double k, double3 spacing,
                              double* n, double* gx, double* gy, double* gz, cudaStream_t stream);
cudaError_t launch_render(const KScene& s, int grid, cudaStream_t stream);
cudaError_t launch_emitter_stats(const KScene& s, cudaStream_t stream);
// the no-medium instantiations, compiled in their own translation unit
// (kernels_nomedium.cu); launch_render / launch_trace_rays dispatch to them
int render_occupancy_nomedium(int blocks_per_sm[2]);
cudaError_t launch_render_nomedium(const KScene& s, int grid, cudaStream_t stream);
cudaError_t launch_trace_rays_nomedium(const KScene& s, int64_t n, const int64_t* src,
                                       const int32_t* ray, double* uv, int32_t* status,
                                       int32_t* steps, cudaStream_t stream);
// resident CTAs per SM of each render_emitters instantiation, [pair][field mode]
int render_occupancy(int blocks_per_sm[2][3]);
int field_mode(const KScene& s);  // 0 no medium, 1 nodes, 2 cell table
cudaError_t launch_trace_rays(const KScene& s, int64_t n, const int64_t* src, const int32_t* ray,
                              double* uv, int32_t* status, int32_t* steps, cudaStream_t stream);
cudaError_t launch_pack_nodes(const double* n, const double* gx, const double* gy,
                              const double* gz, float4* out, int64_t count, cudaStream_t stream);
cudaError_t launch_build_from_density(const float* rho, int nx, int ny, int nz, double k,
                                      double3 spacing, float4* out, int z0, int z1,
                                      cudaStream_t stream);
cudaError_t launch_build_cells(const float4* grid, int nx, int ny, int nz, CellCoef* cells,
                               cudaStream_t stream);
cudaError_t launch_image_finalize(const unsigned long long* fixed, double* out, int64_t n,
                                  cudaStream_t stream);

}  // namespace rbk
