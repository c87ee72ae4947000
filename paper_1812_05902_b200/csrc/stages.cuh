// stages.cuh — FP64 stages of the per-ray pipeline shared by K1 (render.cuh,
// compiled with FMA contraction) and the FP64 validation kernels
// (kernels_fp64.cu, compiled with -fmad=false so every operation rounds like
// the reference's x86-64 build).  Included inside namespace rbk::(anonymous).
//   stage 1  ray generation   raygen.cpp:12-88, CounterRng core.hpp:80-107
//   stage 3  optics chain     optics.cpp:15-158
//   stage 4a sensor hit       sensor.cpp:27-34
#pragma once

// ---------------------------------------------------------------- math
__device__ __forceinline__ double3 operator+(double3 a, double3 b) {
  return make_double3(a.x + b.x, a.y + b.y, a.z + b.z);
}
__device__ __forceinline__ double3 operator-(double3 a, double3 b) {
  return make_double3(a.x - b.x, a.y - b.y, a.z - b.z);
}
__device__ __forceinline__ double3 operator*(double3 a, double s) {
  return make_double3(a.x * s, a.y * s, a.z * s);
}
// RB_FAST_DIV (K1, kernels.cu and kernels_nomedium.cu): one reciprocal and three
// multiplies instead of three FP64 divisions (they were 9% of a no-medium
// render); ≤1 ulp per component, ~1e-17 m at the sensor.  The FP64 validation
// build (kernels_fp64.cu) divides the components as the reference does.
__device__ __forceinline__ double3 operator/(double3 a, double s) {
#if RB_FAST_DIV
  const double inv = 1.0 / s;
  return make_double3(a.x * inv, a.y * inv, a.z * inv);
#else
  return make_double3(a.x / s, a.y / s, a.z / s);
#endif
}
__device__ __forceinline__ double3 neg(double3 a) { return make_double3(-a.x, -a.y, -a.z); }
__device__ __forceinline__ double dot(double3 a, double3 b) {
  return a.x * b.x + a.y * b.y + a.z * b.z;
}
__device__ __forceinline__ double norm(double3 v) { return sqrt(dot(v, v)); }
__device__ __forceinline__ double3 normalized(double3 v) { return v / norm(v); }

// SplitMix64 finalizer, core.hpp:81-86.
__device__ __forceinline__ uint64_t mix_bits(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// CounterRng::uniform for draw number n of an element key, core.hpp:97-100.
__device__ __forceinline__ double u01(uint64_t key, uint64_t n) {
  return (double)(mix_bits(key + 0x9e3779b97f4a7c15ULL * n) >> 11) * 0x1p-53;
}

enum { kMissed = 0, kTraced = 1, kLost = 2, kInvalid = 3 };
enum { kBrNone = 0, kBrAperture = 1, kBrMissed = 2, kBrTir = 3 };

// ------------------------------------------------------- stage 1: raygen
// sample_aperture_points (raygen.cpp:27-65) for one ray; ekey is
// mix_bits(mix_bits(seed ^ salt) + source_index), the per-source part of the
// CounterRng key.
__device__ __forceinline__ double3 aperture_point(const KScene& S, uint64_t ekey, int i) {
  double u, v;
  const uint64_t key = mix_bits(ekey + (uint64_t)i);
  if (S.sampling == 0) {
    if (S.rays == 1) {
      u = v = 0.5;
    } else {
      const int cx = i % S.cells, cy = i / S.cells;
      u = ((double)cx + u01(key, 1)) / (double)S.cells;
      v = ((double)cy + u01(key, 2)) / (double)S.cells;
    }
  } else {
    // raygen.cpp:60 under GCC: v takes the first draw, u the second.
    v = u01(key, 1);
    u = u01(key, 2);
  }
  // concentric_disk_map, raygen.cpp:12-25
  const double sx = 2.0 * u - 1.0, sy = 2.0 * v - 1.0;
  double dx = 0.0, dy = 0.0;
  if (!(sx == 0.0 && sy == 0.0)) {
    double r, phi;
    if (fabs(sx) > fabs(sy)) {
      r = sx;
      phi = (M_PI / 4.0) * (sy / sx);
    } else {
      r = sy;
      phi = M_PI / 2.0 - (M_PI / 4.0) * (sx / sy);
    }
    double sn, cs;
#ifdef RB_CORRECTLY_ROUNDED_SINCOS
    cr_sincos(phi, sn, cs);  // FP64 validation build: matches glibc bit for bit
#else
    sincos(phi, &sn, &cs);
#endif
    dx = r * cs;
    dy = r * sn;
  }
  return S.pupil_center + (S.e1 * dx + S.e2 * dy) * S.pupil_radius;
}

// ------------------------------------------------------- stage 3: optics
constexpr double kForwardEps = 1e-12;  // optics.cpp:13

__device__ __forceinline__ double radial_distance(double3 p, double3 axis_point, double3 axis) {
  const double3 rel = p - axis_point;
  return norm(rel - axis * dot(rel, axis));
}

// intersect_plane_cap, optics.cpp:20-30
__device__ __forceinline__ bool plane_cap(double3 o, double3 d, double3 point, double3 axis,
                                          double clear, double3& hp, double3& hn) {
  const double denom = dot(d, axis);
  if (denom == 0.0) return false;
  const double t = dot(point - o, axis) / denom;
  if (t <= kForwardEps) return false;
  const double3 p = o + d * t;
  if (radial_distance(p, point, axis) > clear) return false;
  hp = p;
  hn = denom < 0.0 ? axis : neg(axis);
  return true;
}

// intersect_sphere, optics.cpp:34-57
__device__ bool sphere_hit(double3 o, double3 d, const DSurface& s, double3& hp, double3& hn) {
  if (s.planar) return plane_cap(o, d, s.vertex, s.axis, s.aperture, hp, hn);
  const double3 oc = o - s.center;
  const double b = dot(oc, d);
  const double c = dot(oc, oc) - s.R * s.R;
  const double disc = b * b - c;
  if (disc < 0.0) return false;
  const double sq = sqrt(disc);
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double t = k == 0 ? -b - sq : -b + sq;
    if (t <= kForwardEps) continue;
    const double3 p = o + d * t;
    if (dot(p - s.center, s.vertex - s.center) <= 0.0) continue;
    if (radial_distance(p, s.vertex, s.axis) > s.aperture) continue;
    double3 n = (p - s.center) / s.absR;
    if (dot(d, n) > 0.0) n = neg(n);
    hp = p;
    hn = n;
    return true;
  }
  return false;
}

// refract, optics.cpp:59-65
__device__ __forceinline__ bool refract(double3 dir, double3 n, double ni, double nf, double3& out) {
  const double eta = ni / nf;
  const double cos_i = -dot(dir, n);
  const double k = 1.0 - eta * eta * (1.0 - cos_i * cos_i);
  if (k < 0.0) return false;
  out = normalized(dir * eta + n * (eta * cos_i - sqrt(k)));
  return true;
}

// propagate_chain, optics.cpp:143-158 (first block wins).
__device__ __forceinline__ int optics_chain(const KScene& S, double3& o, double3& d) {
  for (int e = 0; e < S.n_elem; ++e) {
    const DElement& el = S.elem[e];
    if (el.kind == 0) {  // apply_aperture, optics.cpp:108-116: does not advance the ray
      const double denom = dot(d, el.axis);
      if (denom == 0.0) return kBrMissed;
      const double t = dot(el.center - o, el.axis) / denom;
      if (t <= kForwardEps) return kBrMissed;
      const double3 p = o + d * t;
      if (norm(p - el.center) > el.radius) return kBrAperture;
    } else if (el.kind == 2) {  // propagate_thin_lens, optics.cpp:118-132
      double3 hp, hn;
      if (!plane_cap(o, d, el.center, el.axis, el.half_diameter, hp, hn)) return kBrMissed;
      const double dz = dot(d, el.axis);
      if (dz <= 0.0) return kBrMissed;
      const double3 focal_point = el.center + d * (el.focal / dz);
      o = hp;
      d = normalized((focal_point - hp) * (el.focal > 0.0 ? 1.0 : -1.0));
    } else if (el.kind == 1) {  // propagate_through_lens, optics.cpp:85-106
#if RB_COMPACT_OPTICS
      // the two surfaces as one rolled loop: the same operations, half the code
      // (RB_COMPACT_OPTICS: the instruction-cache-bound no-medium kernel)
#pragma unroll 1
      for (int sf = 0; sf < 2; ++sf) {
        const DSurface& srf = sf ? el.back : el.front;
        double3 hp, hn, out_dir;
        if (!sphere_hit(o, d, srf, hp, hn)) return kBrMissed;
        if (!refract(d, hn, srf.n_before, srf.n_after, out_dir)) return kBrTir;
        o = hp;
        d = out_dir;
      }
#else
      double3 hp, hn, in_dir, out_dir;
      if (!sphere_hit(o, d, el.front, hp, hn)) return kBrMissed;
      if (!refract(d, hn, el.front.n_before, el.front.n_after, in_dir)) return kBrTir;
      double3 bp, bn;
      if (!sphere_hit(hp, in_dir, el.back, bp, bn)) return kBrMissed;
      if (!refract(in_dir, bn, el.back.n_before, el.back.n_after, out_dir)) return kBrTir;
      o = bp;
      d = out_dir;
#endif
    } else {  // reflect_on_mirror, optics.cpp:134-141
      double3 hp, hn;
      if (!sphere_hit(o, d, el.front, hp, hn)) return kBrMissed;
      o = hp;
      d = d - hn * (2.0 * dot(d, hn));
    }
  }
  return kBrNone;
}

// ----------------------------------------------- stage 4: sensor + spot
// intersect_sensor, sensor.cpp:27-34 (no frame check: off-frame hits land).
__device__ __forceinline__ bool sensor_hit(const KScene& S, double3 o, double3 d, double& u,
                                           double& v) {
  const double denom = dot(d, S.s_normal);
  if (denom == 0.0) return false;
  const double t = dot(S.s_center - o, S.s_normal) / denom;
  if (t <= 0.0) return false;
  const double3 p = o + d * t;
  u = dot(p - S.s_center, S.s_eu);
  v = dot(p - S.s_center, S.s_ev);
  return true;
}
