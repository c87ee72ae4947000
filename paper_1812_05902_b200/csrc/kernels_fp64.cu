// kernels_fp64.cu — the FP64 validation build of the per-ray pipeline.
//
// Compiled with -fmad=false (build.py), so every FP64 add/mul/div/sqrt rounds
// exactly like the reference's x86-64 build (which has no FMA).
// The GRIN stage is a literal FP64 restatement of trace_through_volume
// (grin.cpp:74-134) sampling the FP64 GriddedField nodes (scene.cpp:99-135) in
// the reference's operation order, instead of K1's FP32 perturbation form; the
// FP64 raygen / optics / sensor stages are the same source as K1's (stages.cuh).
// Per-ray results are therefore bit-identical to the reference except where the
// device sin/cos (raygen.cpp:24) differ from glibc's by an ulp.
//
// Two kernels: a per-ray replay (rb_trace_rays_fp64) and the per-source
// statistics with rays summed in the reference's order (rb_trace_stats_fp64),
// which makes DotHitStats bit-identical too.  Validation only: one thread per
// ray / per source, FP64 SoA field copy (32 B/node) kept on device.
#include "kernels.h"

#include <math.h>

namespace rbk {
namespace {

// ---- correctly rounded sin/cos for concentric_disk_map's angle --------------
// glibc's sin/cos (raygen.cpp:24) return the correctly rounded result in
// practice; the device sincos may be 1-2 ulp off, which flipped ~5% of the
// aperture points' last bits.  The angle lies in [-pi/4, 3pi/4]; reduce by
// pi/2 in double-double, evaluate the Taylor series in double-double (15 terms
// reach 1e-36 at |r| <= pi/4) and round once.  Explicit __fma_rn / __d*_rn
// keep this exact under -fmad=false.
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd dd_fast2sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  const double s = __dadd_rn(a.hi, b.hi);
  const double bb = __dsub_rn(s, a.hi);
  const double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b.hi, bb));
  return dd_fast2sum(s, __dadd_rn(e, __dadd_rn(a.lo, b.lo)));
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  const double p = __dmul_rn(a.hi, b.hi);
  const double e = __fma_rn(a.hi, b.hi, -p);
  return dd_fast2sum(p, __fma_rn(a.hi, b.lo, __fma_rn(a.lo, b.hi, e)));
}
__device__ __forceinline__ dd dd_div_small(dd a, double b) {  // b a small integer
  const double q1 = __ddiv_rn(a.hi, b);
  const double p = __dmul_rn(q1, b);
  const double e = __fma_rn(q1, b, -p);
  const double r = __dadd_rn(__dsub_rn(__dsub_rn(a.hi, p), e), a.lo);
  return dd_fast2sum(q1, __ddiv_rn(r, b));
}
__device__ void cr_sincos(double x, double& s, double& c) {
  const dd kPio2 = {1.5707963267948966192e+00, 6.1232339957367658e-17};
  const bool shift = x > 0.78539816339744830962;
  // r = x - pi/2 exactly in double-double when shifting
  dd r = shift ? dd_add(dd{x, 0.0}, dd{-kPio2.hi, -kPio2.lo}) : dd{x, 0.0};
  const dd r2 = dd_mul(r, r);
  // sin r = r (1 - r2/(2*3) (1 - r2/(4*5) (...))),  cos r = 1 - r2/(1*2) (1 - r2/(3*4) (...))
  dd ps = {1.0, 0.0}, pc = {1.0, 0.0};
  for (int k = 15; k >= 1; --k) {
    const dd ts = dd_div_small(dd_mul(r2, ps), (double)(2 * k) * (double)(2 * k + 1));
    ps = dd_add(dd{1.0, 0.0}, dd{-ts.hi, -ts.lo});
    const dd tc = dd_div_small(dd_mul(r2, pc), (double)(2 * k - 1) * (double)(2 * k));
    pc = dd_add(dd{1.0, 0.0}, dd{-tc.hi, -tc.lo});
  }
  const dd sr = dd_mul(r, ps);
  if (shift) {  // sin(x) = cos(r), cos(x) = -sin(r)
    s = __dadd_rn(pc.hi, pc.lo);
    c = -__dadd_rn(sr.hi, sr.lo);
  } else {
    s = __dadd_rn(sr.hi, sr.lo);
    c = __dadd_rn(pc.hi, pc.lo);
  }
}
#define RB_CORRECTLY_ROUNDED_SINCOS 1

#include "stages.cuh"

// GriddedField::sample, scene.cpp:99-135 (bounds recomputed, true divisions,
// weights and 8-term sums left to right).
__device__ bool sample64(const Field64& F, double3 p, double& n, double3& g) {
  if (!(p.x >= F.lo.x && p.x <= F.hi.x && p.y >= F.lo.y && p.y <= F.hi.y && p.z >= F.lo.z &&
        p.z <= F.hi.z))
    return false;
  const double qx = (p.x - F.origin.x) / F.spacing.x;
  const double qy = (p.y - F.origin.y) / F.spacing.y;
  const double qz = (p.z - F.origin.z) / F.spacing.z;
  int i = (int)qx, j = (int)qy, k = (int)qz;
  if (i > F.nx - 2) i = F.nx - 2;
  if (j > F.ny - 2) j = F.ny - 2;
  if (k > F.nz - 2) k = F.nz - 2;
  const double fx = qx - i, fy = qy - j, fz = qz - k;
  const size_t q000 = ((size_t)k * F.ny + j) * F.nx + i;
  const size_t q100 = q000 + 1, q010 = q000 + F.nx, q110 = q010 + 1;
  const size_t q001 = q000 + (size_t)F.nx * F.ny, q101 = q001 + 1, q011 = q001 + F.nx,
               q111 = q011 + 1;
  const double w000 = (1 - fx) * (1 - fy) * (1 - fz);
  const double w100 = fx * (1 - fy) * (1 - fz);
  const double w010 = (1 - fx) * fy * (1 - fz);
  const double w110 = fx * fy * (1 - fz);
  const double w001 = (1 - fx) * (1 - fy) * fz;
  const double w101 = fx * (1 - fy) * fz;
  const double w011 = (1 - fx) * fy * fz;
  const double w111 = fx * fy * fz;
#define RB_L(a)                                                                             \
  (w000 * a[q000] + w100 * a[q100] + w010 * a[q010] + w110 * a[q110] + w001 * a[q001] +     \
   w101 * a[q101] + w011 * a[q011] + w111 * a[q111])
  n = RB_L(F.n);
  g = make_double3(RB_L(F.gx), RB_L(F.gy), RB_L(F.gz));
#undef RB_L
  return true;
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// ClampedD, grin.cpp:23-33
__device__ double3 clamped_d(const Field64& F, double3 r) {
  const double3 q = make_double3(clampd(r.x, F.lo.x, F.hi.x), clampd(r.y, F.lo.y, F.hi.y),
                                 clampd(r.z, F.lo.z, F.hi.z));
  double n;
  double3 g;
  if (!sample64(F, q, n, g)) return make_double3(0.0, 0.0, 0.0);
  return g * n;
}

// aabb_intersect, grin.cpp:52-72
__device__ bool aabb64(const Field64& F, double3 o, double3 d, double& tn) {
  double t_near = -INFINITY, t_far = INFINITY;
  const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
  const double lo[3] = {F.lo.x, F.lo.y, F.lo.z}, hi[3] = {F.hi.x, F.hi.y, F.hi.z};
  for (int a = 0; a < 3; ++a) {
    if (dd[a] == 0.0) {
      if (oo[a] < lo[a] || oo[a] > hi[a]) return false;
      continue;
    }
    double t0 = (lo[a] - oo[a]) / dd[a], t1 = (hi[a] - oo[a]) / dd[a];
    if (t0 > t1) {
      const double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    t_near = t_near < t0 ? t0 : t_near;
    t_far = t1 < t_far ? t1 : t_far;
  }
  if (t_far < t_near || t_far < 0.0) return false;
  tn = t_near < 0.0 ? 0.0 : t_near;
  return true;
}

__device__ __forceinline__ bool contains64(const Field64& F, double3 p) {
  return p.x >= F.lo.x && p.x <= F.hi.x && p.y >= F.lo.y && p.y <= F.hi.y && p.z >= F.lo.z &&
         p.z <= F.hi.z;
}

// StepObserver (grin.hpp:64-66) sink for trace_debug: (xi, r, t) records.
struct Recorder {
  double* rec;
  int64_t cap;
  int64_t n;
  __device__ void operator()(double xi, double3 r, double3 t) {
    if (rec && n < cap) {
      double* q = rec + 7 * n;
      q[0] = xi;
      q[1] = r.x;
      q[2] = r.y;
      q[3] = r.z;
      q[4] = t.x;
      q[5] = t.y;
      q[6] = t.z;
    }
    ++n;
  }
};

// trace_through_volume, grin.cpp:74-134, with rk4_step_impl (grin.cpp:35-44).
__device__ int grin64(const Field64& F, double h, int max_steps, double3& o, double3& d,
                      int& steps, Recorder* obs = nullptr) {
  steps = 0;
  double tn;
  if (!aabb64(F, o, d, tn)) return kMissed;
  if (!(h > 0.0)) return kInvalid;
  double3 r = o + d * (tn + 1e-9);
  if (!contains64(F, r)) return kMissed;
  double ne;
  double3 ge;
  double3 t = d * (sample64(F, r, ne, ge) ? ne : 1.0);
  double xi = 0.0;
  if (obs) (*obs)(xi, r, t);
  for (int step = 0; step < max_steps; ++step) {
    const double3 a = clamped_d(F, r) * h;
    const double3 b = clamped_d(F, r + (t * 0.5 + a * 0.125) * h) * h;
    const double3 c = clamped_d(F, r + (t + b * 0.5) * h) * h;
    const double3 nr = r + (t + (a + b * 2.0) * (1.0 / 6.0)) * h;
    const double3 nt = t + (a + b * 4.0 + c) * (1.0 / 6.0);
    if (!(isfinite(nr.x) && isfinite(nr.y) && isfinite(nr.z) && isfinite(nt.x) &&
          isfinite(nt.y) && isfinite(nt.z))) {
      steps = step;
      return kInvalid;
    }
    if (contains64(F, nr)) {
      r = nr;
      t = nt;
      xi += h;
      if (obs) (*obs)(xi, r, t);
      continue;
    }
    double s = 1.0;
    const double r0[3] = {r.x, r.y, r.z}, r1[3] = {nr.x, nr.y, nr.z};
    const double lo[3] = {F.lo.x, F.lo.y, F.lo.z}, hi[3] = {F.hi.x, F.hi.y, F.hi.z};
    for (int ax = 0; ax < 3; ++ax) {
      const double delta = r1[ax] - r0[ax];
      if (r1[ax] < lo[ax]) s = fmin(s, (lo[ax] - r0[ax]) / delta);
      if (r1[ax] > hi[ax]) s = fmin(s, (hi[ax] - r0[ax]) / delta);
    }
    s = clampd(s, 0.0, 1.0);
    const double3 er = r + (nr - r) * s;
    const double3 et = t + (nt - t) * s;
    xi += s * h;
    if (obs) (*obs)(xi, er, et);
    o = er;
    d = normalized(et);
    steps = step + 1;
    return kTraced;
  }
  steps = max_steps;
  return kLost;
}

// process_source's per-ray body (engine.cpp:112-137) in FP64.
__device__ int trace_ray64(const KScene& S, const Field64& F, uint64_t ekey, double3 src, int i,
                           double& u, double& v, int& steps) {
  steps = 0;
  const double3 p = aperture_point(S, ekey, i);
  const double3 to = p - src;
  const double len = norm(to);
  if (!(len > 0.0)) {
    atomicOr(S.err_flag, 1);
    return 1;
  }
  double3 o = src, d = to / len;
  if (S.with_field) {
    const int st = grin64(F, S.h, S.max_steps, o, d, steps);
    if (st == kLost || st == kInvalid) return 1;
  }
  const int br = optics_chain(S, o, d);
  if (br != kBrNone) return br == kBrAperture ? 2 : (br == kBrTir ? 4 : 3);
  if (!sensor_hit(S, o, d, u, v)) return 5;
  return 0;
}

__global__ void trace_rays_fp64_kernel(const __grid_constant__ KScene S, const Field64 F, int64_t n,
                                       const int64_t* __restrict__ srcs,
                                       const int32_t* __restrict__ rays, double* uv,
                                       int32_t* status, int32_t* steps) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t src = srcs[q];
  const uint64_t sid = S.source_ids ? (uint64_t)S.source_ids[src] : (uint64_t)src;
  const double3 so = make_double3(S.sources[3 * src], S.sources[3 * src + 1], S.sources[3 * src + 2]);
  double u = nan(""), v = nan("");
  int st_steps = 0;
  const int st = trace_ray64(S, F, mix_bits(S.key_seed + sid), so, rays[q], u, v, st_steps);
  uv[2 * q] = st == 0 ? u : nan("");
  uv[2 * q + 1] = st == 0 ? v : nan("");
  status[q] = st;
  steps[q] = st_steps;
}

// One thread per source, rays in the reference's order: DotHitStats summed
// exactly as process_source sums them (engine.cpp:136-137).
__global__ void source_stats_fp64_kernel(const __grid_constant__ KScene S, const Field64 F) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S.n_sources) return;
  const uint64_t sid = S.source_ids ? (uint64_t)S.source_ids[s] : (uint64_t)s;
  const double3 so = make_double3(S.sources[3 * s], S.sources[3 * s + 1], S.sources[3 * s + 2]);
  const uint64_t ekey = mix_bits(S.key_seed + sid);
  double hx = 0.0, hy = 0.0;
  long long landed = 0;
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  for (int i = 0; i < S.rays; ++i) {
    double u = 0.0, v = 0.0;
    int steps = 0;
    const int st = trace_ray64(S, F, ekey, so, i, u, v, steps);
    c[5] += (unsigned long long)steps;
    if (st == 0) {
      hx += u;
      hy += v;
      ++landed;
    } else {
      c[st - 1] += 1;
    }
  }
  S.hit_sum[2 * s] = hx;
  S.hit_sum[2 * s + 1] = hy;
  S.landed[s] = landed;
  for (int j = 0; j < 6; ++j)
    if (c[j]) atomicAdd(&S.counters[j], c[j]);
}

// trace_debug (engine.cpp:605-624): one ray, its trajectory records.
__global__ void trace_debug_kernel(const __grid_constant__ KScene S, const Field64 F, int64_t src,
                                   int ray, double* rec, int64_t cap, int64_t* n_rec) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint64_t sid = S.source_ids ? (uint64_t)S.source_ids[src] : (uint64_t)src;
  const double3 so = make_double3(S.sources[3 * src], S.sources[3 * src + 1], S.sources[3 * src + 2]);
  const double3 p = aperture_point(S, mix_bits(S.key_seed + sid), ray);
  const double3 to = p - so;
  double3 o = so, d = to / norm(to);
  Recorder obs{rec, cap, 0};
  int steps = 0;
  grin64(F, S.h, S.max_steps, o, d, steps, &obs);
  *n_rec = obs.n;
}

// FP64 GriddedField nodes from the density volume (scene.cpp:53-92), the same
// explicitly-rounded arithmetic as K0's float4 build.
__device__ __forceinline__ double n_of64(const float* rho, double k, size_t q) {
  return __dadd_rn(__dmul_rn(k, (double)rho[q]), 1.0);
}

__global__ void build_fp64_kernel(const float* __restrict__ rho, int nx, int ny, int nz, double k,
                                  double3 sp, double* n, double* gx, double* gy, double* gz) {
  const int64_t plane = (int64_t)nx * ny;
  const int64_t count = plane * nz;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int kk = (int)(q / plane);
    const int64_t rem = q % plane;
    const int j = (int)(rem / nx), i = (int)(rem % nx);
    const double nq = n_of64(rho, k, q);
    const int idx[3] = {i, j, kk}, dim[3] = {nx, ny, nz};
    const int64_t stride[3] = {1, nx, plane};
    const double h[3] = {sp.x, sp.y, sp.z};
    double g[3];
    for (int a = 0; a < 3; ++a) {
      if (idx[a] == 0)
        g[a] = (n_of64(rho, k, q + stride[a]) - nq) / h[a];
      else if (idx[a] == dim[a] - 1)
        g[a] = (nq - n_of64(rho, k, q - stride[a])) / h[a];
      else
        g[a] = (n_of64(rho, k, q + stride[a]) - n_of64(rho, k, q - stride[a])) / (2.0 * h[a]);
    }
    n[q] = nq;
    gx[q] = g[0];
    gy[q] = g[1];
    gz[q] = g[2];
  }
}

}  // namespace

cudaError_t launch_trace_rays_fp64(const KScene& s, const Field64& f, int64_t n, const int64_t* src,
                                   const int32_t* ray, double* uv, int32_t* status,
                                   int32_t* steps, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  trace_rays_fp64_kernel<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(s, f, n, src, ray, uv,
                                                                           status, steps);
  return cudaGetLastError();
}

cudaError_t launch_source_stats_fp64(const KScene& s, const Field64& f, cudaStream_t stream) {
  if (s.n_sources <= 0) return cudaSuccess;
  source_stats_fp64_kernel<<<(unsigned)((s.n_sources + 63) / 64), 64, 0, stream>>>(s, f);
  return cudaGetLastError();
}

cudaError_t launch_trace_debug(const KScene& s, const Field64& f, int64_t src, int ray,
                               double* rec, int64_t cap, int64_t* n_rec, cudaStream_t stream) {
  trace_debug_kernel<<<1, 32, 0, stream>>>(s, f, src, ray, rec, cap, n_rec);
  return cudaGetLastError();
}

cudaError_t launch_build_fp64(const float* rho, int nx, int ny, int nz, double k, double3 spacing,
                              double* n, double* gx, double* gy, double* gz, cudaStream_t stream) {
  build_fp64_kernel<<<148 * 8, 256, 0, stream>>>(rho, nx, ny, nz, k, spacing, n, gx, gy, gz);
  return cudaGetLastError();
}

}  // namespace rbk
