// render.cuh — K1 render_emitters and the per-ray replay kernel, with every
// device helper they use, in an anonymous namespace: included by kernels.cu
// (field instantiations) and kernels_nomedium.cu (the no-medium instantiation,
// compiled on its own so its FP64 arithmetic choices cannot perturb the
// register allocation of the RK4 loop).  Not a public header.
#pragma once

#include <math.h>

#ifndef RB_CHECKED
#define RB_CHECKED 0
#endif
// Checked build (RB_CHECKED=1 -> libraybos_gpu_checked.so): every shared- and
// global-memory index K1 computes is range-checked; a violation is counted in
// check_fail[0] with its site code in check_fail[1] (no trap, the kernel
// finishes and rb_trace reports it).  compute-sanitizer is closed on this pool;
// this is the out-of-bounds half of its memcheck, run by tests/test_gpu_checked.py.
#if RB_CHECKED
#define RB_CHECK(S, cond, code)                  \
  do {                                           \
    if (!(cond)) {                               \
      atomicAdd((S).check_fail, 1u);             \
      atomicMax((S).check_fail + 1, (unsigned)(code)); \
    }                                            \
  } while (0)
#else
#define RB_CHECK(S, cond, code) \
  do {                          \
  } while (0)
#endif

namespace rbk {
namespace {

#include "stages.cuh"
#include "grin.cuh"

struct RayResult {
  double u, v;
  int status;
};

// process_source's per-ray body, engine.cpp:112-137.
// emit_rays (raygen.cpp:74-80) for one ray: false when the source coincides
// with its aperture point (the reference throws).
__device__ __forceinline__ bool emit_ray(const KScene& S, uint64_t ekey, double3 src, int i,
                                         double3& d) {
  const double3 p = aperture_point(S, ekey, i);
  const double3 to = p - src;
  const double len = norm(to);
  if (!(len > 0.0)) {
    atomicOr(S.err_flag, 1);
    return false;
  }
  d = to / len;
  return true;
}

// Stages 2-4 of process_source (engine.cpp:112-137) for an emitted ray.
// kField: 0 = the scene has no medium (no GRIN code at all), 1 = field read
// from the float4 nodes, 2 = from the per-cell coefficient table.
// The ray's RK4 steps are added to *steps_acc (a per-thread shared counter,
// folded into the 64-bit per-unit count after every ray).
template <int kField>
__device__ __forceinline__ RayResult finish_ray(const KScene& S, double3 o, double3 d, bool field,
                                                double* scratch, unsigned* steps_acc) {
  RayResult r;
  r.u = r.v = 0.0;
  if (kField != 0 && field) {
    const int st = grin_trace<kField == 2>(S, o, d, steps_acc, scratch);
    if (st == kLost || st == kInvalid) {
      r.status = 1;  // RB_RAY_LOST
      return r;
    }
  }
  const int br = optics_chain(S, o, d);
  if (br != kBrNone) {
    r.status = br == kBrAperture ? 2 : (br == kBrTir ? 4 : 3);
    return r;
  }
  if (!sensor_hit(S, o, d, r.u, r.v)) {
    r.status = 5;
    return r;
  }
  r.status = 0;
  return r;
}

// process_source's per-ray body, engine.cpp:112-137.
template <int kField>
__device__ __forceinline__ RayResult trace_ray(const KScene& S, uint64_t ekey, double3 src, int i,
                                               double* scratch, unsigned* steps_acc) {
  double3 d;
  if (!emit_ray(S, ekey, src, i, d)) {
    RayResult r;
    r.u = r.v = 0.0;
    r.status = 1;
    return r;
  }
  return finish_ray<kField>(S, src, d, S.with_field, scratch, steps_acc);
}

// Tile-or-global fixed-point add of one pixel contribution.
__device__ __forceinline__ void add_px(const KScene& S, uint32_t* tile, int tc0, int tr0, int tw,
                                       int th, int c, int r, uint32_t f) {
  const int tx = c - tc0, ty = r - tr0;
  if ((unsigned)tx < (unsigned)tw && (unsigned)ty < (unsigned)th) {
    RB_CHECK(S, ty * tw + tx < kTileCap, 1);
    atomicAdd(&tile[ty * tw + tx], f);
  } else {
    RB_CHECK(S, r >= 0 && r < S.H && c >= 0 && c < S.W, 2);
    atomicAdd(&S.image[(size_t)r * S.W + c], (unsigned long long)f);
  }
}

__device__ __forceinline__ float erf_arg(const KScene& S, int pix, double center) {
  return (float)(((double)pix - center) * S.inv_s);
}

#ifndef RB_FAST_ERF
#define RB_FAST_ERF 0  // kernels_nomedium.cu turns it on
#endif
// erf for the spot weights (RB_FAST_ERF): the branch-free Chebyshev fit of erfc (Numerical
// Recipes' erfcc, fractional error < 1.2e-7) on the MUFU reciprocal and exp2,
// with the polynomial pre-scaled by log2(e) — about 16 instructions and no
// divergence between lanes whose arguments fall in different ranges, against
// erff's ~30 in several branches (erff was 27% of a no-medium ray's
// instructions).  The weights are differences of these values normalised by
// their own sum (sensor.cpp:106-111), so a spot's energy stays exact; a
// per-pixel weight moves by < 1e-6 absolute.
__device__ __forceinline__ float fast_erf(float x) {
  const float z = fabsf(x);
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.5f, z, 1.0f)));
  constexpr float L = 1.4426950408889634f;  // log2(e)
  float p = 0.17087277f * L;
  p = fmaf(p, t, -0.82215223f * L);
  p = fmaf(p, t, 1.48851587f * L);
  p = fmaf(p, t, -1.13520398f * L);
  p = fmaf(p, t, 0.27886807f * L);
  p = fmaf(p, t, -0.18628806f * L);
  p = fmaf(p, t, 0.09678418f * L);
  p = fmaf(p, t, 0.37409196f * L);
  p = fmaf(p, t, 1.00002368f * L);
  p = fmaf(p, t, -1.26551223f * L);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(fmaf(z * -L, z, p)));
  const float erfc = t * e;  // erfc(|x|)
  return copysignf(1.0f - erfc, x);
}

// One axis of a spot window: the erf argument (pix - centre) / (sqrt2 sigma /
// pitch) of sensor.cpp:86-95 is evaluated in FP64 once, at the window's first
// pixel p0, and stepped by inv_s in FP32 from there.
struct SpotAxis {
  double center;  // spot centre in pixels (cc or rc)
  int p0;         // first pixel of the window
  float base;     // argument at p0
};
__device__ __forceinline__ SpotAxis spot_axis(const KScene& S, double center, int p0) {
  SpotAxis a;
  a.center = center;
  a.p0 = p0;
  a.base = (float)(((double)p0 - center) * S.inv_s);
  return a;
}
__device__ __forceinline__ float spot_erf(const KScene& S, const SpotAxis& a, int pix) {
#if RB_FAST_ERF
  return fast_erf(fmaf((float)(pix - a.p0), S.inv_s_f, a.base));
#else
  return erff(erf_arg(S, pix, a.center));
#endif
}

// Unbiased deterministic rounding of a fixed-point contribution: floor(x + u)
// with a dither offset u in [0, 1) per (ray, spot row): a Weyl step of the
// ray's counter-RNG key by the absolute row index.  Over the rays that hit a
// pixel the u are independent and uniform, so E[f] = x and the rounding errors
// of coherent rays (which all see nearly the same weights) do not accumulate
// into a bias (round-to-nearest left 5e-5 relative L2 on 1e4-ray bundles; this
// leaves < 1e-6); a fresh u per row keeps one ray's rounding errors from all
// moving together.  u depends only on the ray and the pixel row, never on
// scheduling, so images stay bit-reproducible.
__device__ __forceinline__ float row_dither(uint32_t seed, int row) {
  return __uint_as_float(0x3f800000u | ((seed + (uint32_t)row * 0x9E3779B9u) >> 9)) - 1.0f;
}
#ifndef RB_DITHER
#define RB_DITHER 1
#endif
__device__ __forceinline__ uint32_t dround(float x, float u) {
  return RB_DITHER ? __float2uint_rd(x + u) : __float2uint_rn(x);
}

// Shared-memory add without a return value (RED) — adding 0 is harmless, so
// callers need no per-pixel branch.
__device__ __forceinline__ void red_shared(uint32_t addr, uint32_t f) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(f) : "memory");
}

// Reloads chunks [0, n) of the column weights (volatile: must not be hoisted
// out of the row loop, or they would stay in registers again).
__device__ __forceinline__ void lds_weights(const float4* wsh, float (&wr)[kMaxSpot], int n) {
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < n)
      asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w)
                   : "r"((uint32_t)__cvta_generic_to_shared(wsh + j * kBlock)));
    wr[4 * j] = q.x;
    wr[4 * j + 1] = q.y;
    wr[4 * j + 2] = q.z;
    wr[4 * j + 3] = q.w;
  }
}

template <int W>
__device__ __forceinline__ void red_row(uint32_t trow, const float (&wu)[kMaxSpot], float row_w,
                                        float u) {
#pragma unroll
  for (int k = 0; k < W; ++k) red_shared(trow + 4 * k, dround(wu[k] * row_w, u));
}

// accumulate_spot (sensor.cpp:57-122): separable erf-difference Gaussian,
// normalized over the full window, in-frame pixels only.
// wsh: this thread's 3 float4 slots (stride kBlock) of shared memory for the
// column weights; the row loop re-reads them (3 LDS.128 per row) instead of
// holding 12 registers across it, which at 80 registers spilled them.
__device__ __forceinline__ void deposit(const KScene& S, double u, double v, uint32_t* tile, int tc0,
                                     int tr0, int tw, int th, uint32_t seed, float4* wsh) {
  const double cc = u / S.pitch + 0.5 * S.W;
  const double rc = 0.5 * S.H - v / S.pitch;
  const float energy_fx = (float)(S.radiance * 2147483648.0);
  if (S.degenerate) {  // sensor.cpp:71-77
    const int col = (int)floor(cc), row = (int)floor(rc);
    if (col >= 0 && col < S.W && row >= 0 && row < S.H)
      add_px(S, tile, tc0, tr0, tw, th, col, row, dround(energy_fx, row_dither(seed, row)));
    return;
  }
  const int c0 = (int)floor(cc - S.half_width), c1 = (int)floor(cc + S.half_width);
  const int r0 = (int)floor(rc - S.half_width), r1 = (int)floor(rc + S.half_width);
  const int cb = max(c0, 0), ce = min(c1, S.W - 1), rb = max(r0, 0), re = min(r1, S.H - 1);
  if (cb > ce || rb > re) return;
  const int ncol = c1 - c0 + 1;
  const SpotAxis ca = spot_axis(S, cc, c0), ra = spot_axis(S, rc, r0);
  const float eu0 = spot_erf(S, ca, c0);
  const float ev0 = spot_erf(S, ra, r0);
  const float ev1 = spot_erf(S, ra, r1 + 1);
  const float mass_v = 0.5f * (ev1 - ev0);
  if (ncol <= kMaxSpot) {
    // column weights straight to shared memory, one column at a time (an
    // unrolled erff chain held every weight in registers and spilled);
    // columns past the window stay 0 and deposit floor(0 + u) = 0
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    wsh[0] = z4;
    wsh[kBlock] = z4;
    wsh[2 * kBlock] = z4;
    float e = eu0;
#pragma unroll 1
    for (int k = 0; k < ncol; ++k) {
      RB_CHECK(S, (k >> 2) < 3, 11);
      const float en = spot_erf(S, ca, c0 + k + 1);
      reinterpret_cast<float*>(wsh + (k >> 2) * kBlock)[k & 3] = 0.5f * (en - e);
      e = en;
    }
    const float mass_u = 0.5f * (e - eu0);
    const float scale = energy_fx / (mass_u * mass_v);
    const bool cols_in_tile = c0 >= tc0 && c1 < tc0 + tw;
    const int width = __reduce_max_sync(__activemask(), ncol);  // warp-uniform row width
    // Rows are visited starting at a lane-dependent row (wrapping once), so the
    // lanes of a coherent warp, whose spots coincide, add to different rows at
    // the same time instead of serialising on the same shared-memory words.
    const int nr = re - rb + 1;
    int r = rb + (int)(threadIdx.x & 31) % nr;
    float er = r == r0 ? ev0 : spot_erf(S, ra, r);
    for (int jr = 0; jr < nr; ++jr, ++r) {
      if (r > re) {
        r = rb;
        er = rb == r0 ? ev0 : spot_erf(S, ra, rb);
      }
      const float er1 = r == r1 ? ev1 : spot_erf(S, ra, r + 1);
      const float row_w = 0.5f * (er1 - er) * scale;
      const float w = row_dither(seed, r);
      er = er1;
      // Fast path when every active lane's current row lies in the shared tile
      // (which lies in the frame): no per-pixel bounds checks.  The choice is
      // warp-uniform, so the warp never executes both loops for one row.
      if (__all_sync(__activemask(), cols_in_tile && (unsigned)(r - tr0) < (unsigned)th)) {
        // The row is `width` unconditional REDs, no branch per pixel: columns
        // past the window have wu = 0, so they add floor(0 + u) = 0 to a word
        // further along the tile (the allocation has kMaxSpot words of slack).
        RB_CHECK(S, (r - tr0) * tw + (c0 - tc0) >= 0 &&
                        (r - tr0) * tw + (c0 - tc0) + (width <= 4 ? 4 : (width <= 8 ? 8 : kMaxSpot)) <=
                            tw * th + kMaxSpot, 3);
        const uint32_t trow = (uint32_t)__cvta_generic_to_shared(tile + (r - tr0) * tw + (c0 - tc0));
        float wr[kMaxSpot];
        lds_weights(wsh, wr, width <= 4 ? 1 : (width <= 8 ? 2 : 3));
        if (width <= 4) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t f = dround(wr[k] * row_w, w);
            if (f) red_shared(trow + 4 * k, f);
          }
        } else if (width <= 8) {
          red_row<8>(trow, wr, row_w, w);
        } else {
          red_row<kMaxSpot>(trow, wr, row_w, w);
        }
      } else {
#if RB_COMPACT_SLOW_ROWS
        // rolled: rows off the tile are rare, and a smaller kernel misses the
        // instruction cache less (the no-medium kernel's main stall; the field
        // kernels measured 1% slower rolled, so they keep the unrolled row)
#pragma unroll 1
        for (int k = 0; k < ncol; ++k) {
          const int c = c0 + k;
          if (c >= 0 && c < S.W) {
            const float wk = reinterpret_cast<const float*>(wsh + (k >> 2) * kBlock)[k & 3];
            const uint32_t f = dround(wk * row_w, w);
            if (f) add_px(S, tile, tc0, tr0, tw, th, c, r, f);
          }
        }
#else
        float wr[kMaxSpot];
        lds_weights(wsh, wr, 3);
#pragma unroll
        for (int k = 0; k < kMaxSpot; ++k) {
          const int c = c0 + k;
          if (k < ncol && c >= 0 && c < S.W) {
            const uint32_t f = dround(wr[k] * row_w, w);
            if (f) add_px(S, tile, tc0, tr0, tw, th, c, r, f);
          }
        }
#endif
      }
    }
  } else {  // wide spots: recompute column weights per pixel
    const float eu1 = spot_erf(S, ca, c1 + 1);
    const float mass_u = 0.5f * (eu1 - eu0);
    const float scale = energy_fx / (mass_u * mass_v);
    float er = rb == r0 ? ev0 : spot_erf(S, ra, rb);
    for (int r = rb; r <= re; ++r) {
      const float er1 = r == r1 ? ev1 : spot_erf(S, ra, r + 1);
      const float row_w = 0.5f * (er1 - er) * scale;
      const float w = row_dither(seed, r);
      er = er1;
      float ec = cb == c0 ? eu0 : spot_erf(S, ca, cb);
      for (int c = cb; c <= ce; ++c) {
        const float ec1 = c == c1 ? eu1 : spot_erf(S, ca, c + 1);
        const uint32_t f = dround(0.5f * (ec1 - ec) * row_w, w);
        ec = ec1;
        if (f) add_px(S, tile, tc0, tr0, tw, th, c, r, f);
      }
    }
  }
}

// DotHitStats::hit_sum is accumulated in fixed point, 2^-40 m per unit
// (9.1e-13 m, 1e-7 of a 10 um pixel; a sensor-plane coordinate is < 2^36 units,
// so 2^27 rays fit an int64): integer sums are exact, so the statistic is the
// same for any assignment of rays to threads, chunks, CTAs or GPUs.
constexpr double kHitScale = 1099511627776.0;  // 2^40
__device__ __forceinline__ long long hit_fixed(double u) { return __double2ll_rn(u * kHitScale); }
__device__ __forceinline__ double hit_double(long long s) { return (double)s * (1.0 / kHitScale); }
// Adds a landed ray's (u, v) to its thread's fixed-point sums.  The reference
// does not clip hits to the sensor (sensor.cpp:27-34), so a grazing ray can land
// arbitrarily far out; past S.hit_limit (2^22 m / rays per emitter) a bundle's
// sum could wrap int64, and the call reports that (err_flag bit 2) instead of a
// wrong DotHitStats.
__device__ __forceinline__ void add_hit(const KScene& S, long long& su, long long& sv, double u,
                                        double v) {
  if (fabs(u) > S.hit_limit || fabs(v) > S.hit_limit) atomicOr(S.err_flag, 2);
  su += hit_fixed(u);
  sv += hit_fixed(v);
}

// Deterministic block sum (fixed shuffle tree, fixed warp order).
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

#ifndef RB_STRAIGHT_PILOT
#define RB_STRAIGHT_PILOT 1
#endif

// Ray index of this lane in patch slot `slot` (k * warps + warp) of the strided
// patch order, or -1 past the lattice (kernels.h KScene::band_rays).
// Ray index of `lane` in patch p of the band order (consecutive p are
// neighbouring patches of the pupil lattice), or -1 past the lattice.
__device__ __forceinline__ int patch_ray_at(const KScene& S, int p, int lane, int N) {
  const int j = p * 32 + lane;  // position in the bands (kernels.h)
  const int band = j / S.band_rays;
  int cx, cy;
  if (band < S.band_full) {
    const int rem = j - band * S.band_rays;
    cx = rem >> S.band_sh;
    cy = band * S.band_h + (rem & (S.band_h - 1));
  } else {
    if (S.band_tail == 0) return -1;
    const int rem = j - S.band_full * S.band_rays;
    cx = rem / S.band_tail;
    cy = S.band_full * S.band_h + (rem - cx * S.band_tail);
  }
  return cx < S.cells && cy * S.cells + cx < N ? cy * S.cells + cx : -1;
}

// render_emitters' slot order: slot k kWarps + w (warp w, patch iteration k)
// visits patch slot * patch_stride mod patch_count, so the 8 patches of one
// iteration lie across the whole pupil.
__device__ __forceinline__ int patch_ray(const KScene& S, int slot, int lane, int N) {
  if (slot >= S.patch_count) return -1;
  return patch_ray_at(S, (int)(((long long)slot * S.patch_stride) % S.patch_count), lane, N);
}

// Grows the unit's pilot bounding box by a landed ray's spot_pixel_window
// (sensor.cpp:44-55), clipped to the frame.
__device__ __forceinline__ void pilot_box(const KScene& S, double u, double v, int* sh_box) {
  const double cc = u / S.pitch + 0.5 * S.W;
  const double rc = 0.5 * S.H - v / S.pitch;
  const int c0 = max((int)floor(cc - S.half_width), 0);
  const int c1 = min((int)floor(cc + S.half_width), S.W - 1);
  const int r0 = max((int)floor(rc - S.half_width), 0);
  const int r1 = min((int)floor(rc + S.half_width), S.H - 1);
  if (c0 <= c1 && r0 <= r1) {
    atomicMin(&sh_box[0], c0);
    atomicMin(&sh_box[1], r0);
    atomicMax(&sh_box[2], c1);
    atomicMax(&sh_box[3], r1);
  }
}

#ifndef RB_TILE_COPIES
#define RB_TILE_COPIES 8
#endif
// Places the unit's shared tile over the pilot box (+2 px margin, at most
// kTileCap words) and zeroes it.  Called by the whole CTA.  When the tile is
// small it is replicated (up to RB_TILE_COPIES copies at an odd word stride)
// and lane L deposits into copy L mod copies: the 32 rays of a coherent warp
// land on the same pixels, so with one copy the lanes that visit the same spot
// row at the same time hit the same words (PIV: 3.6 shared wavefronts per
// RED), while the copies put them on different words in different banks.
// The flush sums the copies, so the image is unchanged.
// sh_tile: tc0, tr0, tw, th, copies, stride.
__device__ __forceinline__ void place_tile(const KScene& S, int tid, int* sh_box, int* sh_tile,
                                           uint32_t* tile) {
  __syncthreads();
  if (tid == 0 && sh_box[2] >= 0) {
    const int m = 2;
    const int bw = sh_box[2] - sh_box[0] + 1 + 2 * m, bh = sh_box[3] - sh_box[1] + 1 + 2 * m;
    int tw = min(bw, S.W), th = min(bh, S.H);
    if (tw * th > kTileCap) {
      const float f = sqrtf((float)kTileCap / (float)(tw * th));
      tw = max(1, min(tw, (int)(tw * f)));
      th = max(1, min(th, kTileCap / tw));
    }
    const int ccen = (sh_box[0] + sh_box[2]) / 2, rcen = (sh_box[1] + sh_box[3]) / 2;
    sh_tile[0] = min(max(ccen - tw / 2, 0), S.W - tw);
    sh_tile[1] = min(max(rcen - th / 2, 0), S.H - th);
    sh_tile[2] = tw;
    sh_tile[3] = th;
    const int stride = (tw * th + kMaxSpot) | 1;
    int copies = 1;
    while (copies < RB_TILE_COPIES && 2 * copies * stride <= kTileCap + kMaxSpot) copies *= 2;
    sh_tile[4] = copies;
    sh_tile[5] = copies > 1 ? stride : 0;
    RB_CHECK(S, tw * th <= kTileCap && sh_tile[0] >= 0 && sh_tile[1] >= 0 &&
                    sh_tile[0] + tw <= S.W && sh_tile[1] + th <= S.H &&
                    (copies == 1 || copies * stride <= kTileCap + kMaxSpot), 4);
  }
  __syncthreads();
  const int words = sh_tile[4] > 1 ? sh_tile[4] * sh_tile[5] : sh_tile[2] * sh_tile[3];
  for (int q = tid; q < words; q += kBlock) tile[q] = 0u;
  __syncthreads();
}

// ------------------------------------------------ K1: render_emitters
// Persistent CTAs pull work units from a queue: a unit is one chunk (KScene::
// split) of one emitter's bundle, i.e. a range of patch iterations, each of
// which gives every warp one compact 8x4 patch of the pupil lattice (KScene::
// band_rays).  The unit's first iteration is the pilot: its spots' bounding box
// places the unit's shared-memory tile before any deposit; deposits outside
// the tile go straight to global.  Every accumulator is an integer, so the
// queue order, the split and the CTA count never change a result bit.
// kPair: bos_run pair mode (rb_trace_bos_pair), a separate instantiation so the
// default kernel carries none of its code or registers.
// kField: see finish_ray (a scene without a medium gets a kernel without the
// GRIN loop, which keeps its instruction footprint small).
template <bool kPair, int kField>
__global__ void __launch_bounds__(kBlock, kField == 0 ? kMinBlocksNoField
                                                     : (kField == 2 && !kPair ? kMinBlocksCells
                                                                              : kMinBlocks))
    render_emitters(const __grid_constant__ KScene S) {
  extern __shared__ uint32_t tile[];  // [kTileCap + kMaxSpot slack] then the deposit weights
  float4* const wsh = reinterpret_cast<float4*>(tile + kTileCap + kMaxSpot) + threadIdx.x;
  constexpr int kWarps = kBlock / 32;
  __shared__ int sh_work, sh_src;
  __shared__ int sh_box[4];
  __shared__ int sh_tile[6];                 // tc0, tr0, tw, th, copies, stride (place_tile)
  __shared__ double sh_so[3];                // emitter position
  __shared__ unsigned long long sh_ekey;     // per-emitter RNG key
  // Per-thread emitter accumulators and the GRIN entry state live in shared
  // memory, not registers: they change once per ray, and keeping them out of
  // the register file during the RK4 loop is what lets K1 fit its budget.
  __shared__ long long sh_uv[2][kBlock];      // hit sums, fixed point (kHitScale)
  __shared__ unsigned sh_cnt[6][kBlock];     // landed, lost, aperture, miss, tir, smiss
  __shared__ unsigned long long sh_steps[kBlock];  // RK4 steps (64-bit: rays x max_steps)
  __shared__ unsigned sh_st32[kBlock];             // the ray in flight's steps
  __shared__ double sh_rt[kBlock][7];        // R0, T0 of the ray in flight (grin.cuh)
  __shared__ long long sh_d[2][kWarps];
  __shared__ unsigned long long sh_l[7][kWarps];
  // bos_run pair mode (rb_trace_bos_pair): the no-field leg's accumulators
  __shared__ long long sh_uv0[2][kBlock];
  __shared__ unsigned sh_cnt0[7][kBlock];
  __shared__ long long sh_d0[2][kWarps];
  __shared__ unsigned long long sh_l0[7][kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int N = S.rays;
  const int K = (S.patch_count + kWarps - 1) / kWarps;
  const int Kc = (K + S.split - 1) / S.split;  // patch iterations per chunk
  const int n_units = S.n_work * S.split;
  volatile double* vso = sh_so;
  volatile unsigned long long* vkey = &sh_ekey;
  volatile int* vtile = sh_tile;
  for (;;) {
    if (tid == 0) {
      const int w = atomicAdd(S.queue, 1);
      sh_work = w;
      if (w < n_units) {
        RB_CHECK(S, w / S.split < S.n_work, 8);
        const int src = S.order[w / S.split];
        RB_CHECK(S, src >= 0 && src < S.n_sources, 9);
        sh_src = src;
        const uint64_t sid = S.source_ids ? (uint64_t)S.source_ids[src] : (uint64_t)src;
        sh_ekey = mix_bits(S.key_seed + sid);
        sh_so[0] = S.sources[3 * src];
        sh_so[1] = S.sources[3 * src + 1];
        sh_so[2] = S.sources[3 * src + 2];
      }
      sh_box[0] = sh_box[1] = 0x7fffffff;
      sh_box[2] = sh_box[3] = -1;
      sh_tile[0] = sh_tile[1] = sh_tile[2] = sh_tile[3] = sh_tile[5] = 0;
      sh_tile[4] = 1;
    }
    sh_uv[0][tid] = sh_uv[1][tid] = 0ll;
    sh_uv0[0][tid] = sh_uv0[1][tid] = 0ll;
#pragma unroll
    for (int j = 0; j < 6; ++j) sh_cnt[j][tid] = 0u;
#pragma unroll
    for (int j = 0; j < 7; ++j) sh_cnt0[j][tid] = 0u;
    sh_steps[tid] = 0ull;
    sh_st32[tid] = 0u;
    __syncthreads();
    if (sh_work >= n_units) break;
    const int kb = (sh_work % S.split) * Kc, ke = min(K, kb + Kc);

    // One loop, one trace_ray call site: without a medium iteration kb is the
    // pilot, after which the CTA places the tile (with one, the straight pilot
    // below places it first).  __syncwarp() reconverges the lanes after every
    // ray so a warp never splits into groups running different rays' RK4 loops.
    // (Taking the patches after the pilot from a shared counter instead, so
    // warps with short rays take more, measured no gain: the unit-end barrier
    // waits on the last ray's length, not on the patch count.)
    // Straight pilot (field kernels): the unit's shared tile is placed from one
    // patch per warp, spread over the unit's iterations, traced WITHOUT the medium
    // (raygen + optics + sensor, ~1% of a ray through the field), so the CTA synchronises right
    // after the unit starts instead of after its slowest warp's first ray has
    // crossed the volume (BOS: 2 patch iterations per unit, ~10% of warp time
    // was spent waiting at that barrier).  The medium only shifts spots by the
    // deflection (~1 px, inside the tile margin); a spot that leaves the tile
    // anyway is added to the global image directly, so the image is the same.
    constexpr bool kStraightPilot = RB_STRAIGHT_PILOT && kField != 0;
    if (kStraightPilot && S.accumulate) {
      // warp w pilots its patch of iteration kb + w (ke - kb) / kWarps, so the box
      // spans the unit's iterations, not only its first
      const int i = patch_ray(S, (kb + (warp * (ke - kb)) / kWarps) * kWarps + warp, lane, N);
      if (i >= 0) {
        const double3 so = make_double3(vso[0], vso[1], vso[2]);
        double3 d;
        if (emit_ray(S, *vkey, so, i, d)) {
          const RayResult p = finish_ray<kField>(S, so, d, false, sh_rt[tid], &sh_st32[tid]);
          if (p.status == 0) pilot_box(S, p.u, p.v, sh_box);
        }
      }
      place_tile(S, tid, sh_box, sh_tile, tile);
    }
    for (int k = kb; k < ke; ++k) {
      const int i = patch_ray(S, k * kWarps + warp, lane, N);
      const uint64_t ekey = *vkey;
      RayResult r;
      r.status = -1;
      if (i >= 0) {
        if (kPair) {  // one emitted ray, both legs: no field first (cheap), then the field
          const double3 so = make_double3(vso[0], vso[1], vso[2]);
          double3 d;
          if (emit_ray(S, ekey, so, i, d)) {
            const RayResult r0 = finish_ray<kField>(S, so, d, false, sh_rt[tid], &sh_st32[tid]);
            sh_cnt0[r0.status][tid] += 1u;
            if (r0.status == 0) add_hit(S, sh_uv0[0][tid], sh_uv0[1][tid], r0.u, r0.v);
            r = finish_ray<kField>(S, so, d, true, sh_rt[tid], &sh_st32[tid]);
          } else {
            r.status = 1;
          }
        } else {
          r = trace_ray<kField>(S, ekey, make_double3(vso[0], vso[1], vso[2]), i, sh_rt[tid],
                                &sh_st32[tid]);
        }
        sh_steps[tid] += sh_st32[tid];
        sh_st32[tid] = 0u;
      }
      if (!kStraightPilot && k == kb && S.accumulate) {  // block-uniform branch
        if (r.status == 0) pilot_box(S, r.u, r.v, sh_box);
        place_tile(S, tid, sh_box, sh_tile, tile);
      }
      if (r.status >= 0) {
        RB_CHECK(S, r.status < 6, 10);
        sh_cnt[r.status][tid] += 1u;
        if (r.status == 0) {
          add_hit(S, sh_uv[0][tid], sh_uv[1][tid], r.u, r.v);
          if (S.accumulate)
            deposit(S, r.u, r.v, tile + (lane & (vtile[4] - 1)) * vtile[5], vtile[0], vtile[1],
                    vtile[2], vtile[3],
                    (uint32_t)(mix_bits(ekey + (uint64_t)i) >> 32), wsh);
        }
      }
      __syncwarp();
    }

    // per-emitter stats: DotHitStats (bos.hpp:71-74) + counters, fixed order
    const long long su = warp_sum(sh_uv[0][tid]);
    const long long sv = warp_sum(sh_uv[1][tid]);
    unsigned long long cnt[7];
#pragma unroll
    for (int j = 0; j < 6; ++j) cnt[j] = warp_sum((unsigned long long)sh_cnt[j][tid]);
    cnt[6] = warp_sum(sh_steps[tid]);
    if (lane == 0) {
      sh_d[0][warp] = su;
      sh_d[1][warp] = sv;
#pragma unroll
      for (int j = 0; j < 7; ++j) sh_l[j][warp] = cnt[j];
    }
    if (kPair) {
      const long long su0 = warp_sum(sh_uv0[0][tid]);
      const long long sv0 = warp_sum(sh_uv0[1][tid]);
      unsigned long long c0[7];
#pragma unroll
      for (int j = 0; j < 7; ++j) c0[j] = warp_sum((unsigned long long)sh_cnt0[j][tid]);
      if (lane == 0) {
        sh_d0[0][warp] = su0;
        sh_d0[1][warp] = sv0;
#pragma unroll
        for (int j = 0; j < 7; ++j) sh_l0[j][warp] = c0[j];
      }
    }
    __syncthreads();
    if (S.accumulate) {  // flush the tile (composite_tile, engine.cpp:181-187)
      const int tc0 = sh_tile[0], tr0 = sh_tile[1], tw = sh_tile[2], th = sh_tile[3];
      const int copies = sh_tile[4], stride = sh_tile[5];
      for (int q = tid; q < tw * th; q += kBlock) {
        uint32_t f = tile[q];
        for (int c = 1; c < copies; ++c) f += tile[c * stride + q];
        if (f) {
          const int y = q / tw, x = q - y * tw;
          RB_CHECK(S, tr0 + y < S.H && tc0 + x < S.W && tr0 >= 0 && tc0 >= 0, 5);
          atomicAdd(&S.image[(size_t)(tr0 + y) * S.W + (tc0 + x)], (unsigned long long)f);
        }
      }
    }
    if (tid == 0) {
      long long a = 0, b = 0;
      unsigned long long l[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int k = 0; k < kWarps; ++k) {
        a += sh_d[0][k];
        b += sh_d[1][k];
#pragma unroll
        for (int j = 0; j < 7; ++j) l[j] += sh_l[j][k];
      }
      const int src = sh_src;
      RB_CHECK(S, sh_work < S.n_work * S.split, 12);
      if (S.split > 1) {
        S.hit_part[2 * (size_t)sh_work] = a;
        S.hit_part[2 * (size_t)sh_work + 1] = b;
      } else {
        S.hit_sum[2 * src] = hit_double(a);
        S.hit_sum[2 * src + 1] = hit_double(b);
      }
      *(S.split > 1 ? S.landed_part + sh_work : S.landed + src) = (long long)l[0];
#pragma unroll
      for (int j = 1; j < 7; ++j)
        if (l[j]) atomicAdd(&S.counters[j - 1], l[j]);
      if (kPair) {
        long long a0 = 0, b0 = 0;
        unsigned long long m[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int k = 0; k < kWarps; ++k) {
          a0 += sh_d0[0][k];
          b0 += sh_d0[1][k];
#pragma unroll
          for (int j = 0; j < 7; ++j) m[j] += sh_l0[j][k];
        }
        if (S.split > 1) {
          S.hit_part0[2 * (size_t)sh_work] = a0;
          S.hit_part0[2 * (size_t)sh_work + 1] = b0;
        } else {
          S.hit_sum0[2 * src] = hit_double(a0);
          S.hit_sum0[2 * src + 1] = hit_double(b0);
        }
        *(S.split > 1 ? S.landed_part0 + sh_work : S.landed0 + src) = (long long)m[0];
#pragma unroll
        for (int j = 1; j < 6; ++j)
          if (m[j]) atomicAdd(&S.counters0[j - 1], m[j]);
      }
    }
    __syncthreads();
  }
}

// Per-ray replay (rb_trace_rays).
template <int kField>
__global__ void trace_rays_kernel(const __grid_constant__ KScene S, int64_t n,
                                  const int64_t* __restrict__ srcs, const int32_t* __restrict__ rays,
                                  double* uv, int32_t* status, int32_t* steps) {
  __shared__ double sh_rt[128][7];
  __shared__ unsigned sh_st[128];
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  sh_st[threadIdx.x] = 0u;
  const int64_t src = srcs[q];
  const uint64_t sid = S.source_ids ? (uint64_t)S.source_ids[src] : (uint64_t)src;
  const double3 so = make_double3(S.sources[3 * src], S.sources[3 * src + 1], S.sources[3 * src + 2]);
  const RayResult r = trace_ray<kField>(S, mix_bits(S.key_seed + sid), so, rays[q], sh_rt[threadIdx.x],
                                        &sh_st[threadIdx.x]);
  uv[2 * q] = r.status == 0 ? r.u : nan("");
  uv[2 * q + 1] = r.status == 0 ? r.v : nan("");
  status[q] = r.status;
  steps[q] = (int32_t)sh_st[threadIdx.x];
}

// launch helpers
static size_t render_smem() {
  static_assert(((kTileCap + kMaxSpot) * sizeof(uint32_t)) % 16 == 0, "weights must be 16 B aligned");
  return (size_t)(kTileCap + kMaxSpot) * sizeof(uint32_t) + 3 * kBlock * sizeof(float4);
}

template <bool kPair, int kField>
static void set_smem() {
  cudaFuncSetAttribute(render_emitters<kPair, kField>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)render_smem());
}

template <bool kPair, int kField>
static int occupancy() {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, render_emitters<kPair, kField>, kBlock,
                                                    render_smem()) != cudaSuccess)
    return 0;
  return n;
}

}  // namespace
}  // namespace rbk
