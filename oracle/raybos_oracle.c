/*
 * raybos_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU checker for the GPU path.
 *
 * A plain-C, FP64 restatement of the reference hot path
 *   run_trace -> process_source -> {sample_aperture_points, emit_rays,
 *   trace_through_volume, propagate_chain, intersect_sensor} -> make_tile /
 *   accumulate_spot -> composite_tile
 * following the reference's operation order so that, built without FMA
 * contraction against the same libm, it reproduces the reference bit for bit
 * (pinned by tests/test_oracle.py against oracle/_ref and tests/golden/).
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library.  The product (libraybos_gpu.so) never links or calls it.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "raybos_gpu.h"

typedef struct { double x, y, z; } V3;
typedef struct { double x, y; } V2;

/* ---- core.hpp:28-75 --------------------------------------------------- */
static V3 add(V3 a, V3 b) { V3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static V3 sub(V3 a, V3 b) { V3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static V3 mul(V3 a, double s) { V3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static V3 dvd(V3 a, double s) { V3 r = {a.x / s, a.y / s, a.z / s}; return r; }
static V3 neg(V3 a) { V3 r = {-a.x, -a.y, -a.z}; return r; }
static double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static V3 cross(V3 a, V3 b) {
  V3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
  return r;
}
static double norm2(V3 v) { return dot(v, v); }
static double norm(V3 v) { return sqrt(norm2(v)); }
static V3 normalized(V3 v) { return dvd(v, norm(v)); }
static int finite3(V3 v) { return isfinite(v.x) && isfinite(v.y) && isfinite(v.z); }
static V3 cv(rb_vec3 v) { V3 r = {v.x, v.y, v.z}; return r; }

/* plane_basis, core.hpp:62-67 */
static void plane_basis(V3 axis, V3* e1, V3* e2) {
  V3 helper = fabs(axis.x) < 0.9 ? (V3){1.0, 0.0, 0.0} : (V3){0.0, 1.0, 0.0};
  *e1 = normalized(cross(helper, axis));
  *e2 = cross(axis, *e1);
}

typedef struct { V3 lo, hi; } Aabb;
/* Aabb::contains, core.hpp:73-75 */
static int contains(const Aabb* b, V3 p) {
  return p.x >= b->lo.x && p.x <= b->hi.x && p.y >= b->lo.y && p.y <= b->hi.y &&
         p.z >= b->lo.z && p.z <= b->hi.z;
}

/* mix_bits / CounterRng, core.hpp:80-107 */
static uint64_t mix_bits(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
typedef struct { uint64_t key, n; } Rng;
static Rng rng_make(uint64_t seed, uint64_t stream, uint64_t element) {
  Rng r = {mix_bits(mix_bits(mix_bits(seed) + stream) + element), 0};
  return r;
}
static double rng_uniform(Rng* r) {
  uint64_t x = mix_bits(r->key + 0x9e3779b97f4a7c15ULL * ++r->n);
  return ldexp((double)(x >> 11), -53);
}

/* ---- raygen.cpp --------------------------------------------------------- */
/* concentric_disk_map, raygen.cpp:12-25 */
static V2 concentric_disk_map(double u, double v) {
  const double pi = 3.141592653589793238462643383279502884;
  double sx = 2.0 * u - 1.0, sy = 2.0 * v - 1.0, r, phi;
  if (sx == 0.0 && sy == 0.0) return (V2){0.0, 0.0};
  if (fabs(sx) > fabs(sy)) {
    r = sx;
    phi = (pi / 4.0) * (sy / sx);
  } else {
    r = sy;
    phi = pi / 2.0 - (pi / 4.0) * (sx / sy);
  }
  return (V2){r * cos(phi), r * sin(phi)};
}

/* One aperture point of sample_aperture_points, raygen.cpp:27-65. */
static V3 aperture_point(const rb_scene* s, V3 e1, V3 e2, int cells, uint64_t source_index,
                         int i) {
  const uint64_t kApertureSalt = 0xa93c0de5u;
  const int n = s->rays_per_source;
  V2 d;
  if (s->sampling == RB_SAMPLING_STRATIFIED) {
    double u, v;
    if (n == 1) {
      u = v = 0.5;
    } else {
      Rng rng = rng_make(s->seed ^ kApertureSalt, source_index, (uint64_t)i);
      int cx = i % cells, cy = i / cells;
      u = (cx + rng_uniform(&rng)) / cells;
      v = (cy + rng_uniform(&rng)) / cells;
    }
    d = concentric_disk_map(u, v);
  } else {
    /* raygen.cpp:60 evaluates concentric_disk_map(rng.uniform(), rng.uniform());
     * GCC evaluates the arguments right to left, so v takes the first draw. */
    Rng rng = rng_make(s->seed ^ kApertureSalt, source_index, (uint64_t)i);
    double v = rng_uniform(&rng);
    double u = rng_uniform(&rng);
    d = concentric_disk_map(u, v);
  }
  return add(cv(s->pupil_center), mul(add(mul(e1, d.x), mul(e2, d.y)), s->pupil_radius));
}

/* ---- scene.cpp:94-135 GriddedField::bounds / sample ---------------------- */
typedef struct {
  int nx, ny, nz;
  V3 origin, spacing;
  const double *n, *gx, *gy, *gz;
} Field;

static Aabb field_bounds(const Field* f) {
  Aabb b;
  b.lo = f->origin;
  b.hi = add(f->origin, (V3){(f->nx - 1) * f->spacing.x, (f->ny - 1) * f->spacing.y,
                            (f->nz - 1) * f->spacing.z});
  return b;
}

/* Returns 0 for nullopt. */
static int field_sample(const Field* f, V3 p, double* n_out, V3* g_out) {
  Aabb b = field_bounds(f);
  if (!contains(&b, p)) return 0;
  double qx = (p.x - f->origin.x) / f->spacing.x;
  double qy = (p.y - f->origin.y) / f->spacing.y;
  double qz = (p.z - f->origin.z) / f->spacing.z;
  int i = (int)qx, j = (int)qy, k = (int)qz;
  if (i > f->nx - 2) i = f->nx - 2;
  if (j > f->ny - 2) j = f->ny - 2;
  if (k > f->nz - 2) k = f->nz - 2;
  double fx = qx - i, fy = qy - j, fz = qz - k;
  size_t q000 = ((size_t)k * f->ny + j) * f->nx + i;
  size_t q100 = q000 + 1, q010 = q000 + f->nx, q110 = q010 + 1;
  size_t q001 = q000 + (size_t)f->nx * f->ny, q101 = q001 + 1, q011 = q001 + f->nx,
         q111 = q011 + 1;
  double w000 = (1 - fx) * (1 - fy) * (1 - fz);
  double w100 = fx * (1 - fy) * (1 - fz);
  double w010 = (1 - fx) * fy * (1 - fz);
  double w110 = fx * fy * (1 - fz);
  double w001 = (1 - fx) * (1 - fy) * fz;
  double w101 = fx * (1 - fy) * fz;
  double w011 = (1 - fx) * fy * fz;
  double w111 = fx * fy * fz;
#define LERP(g)                                                                         \
  (w000 * g[q000] + w100 * g[q100] + w010 * g[q010] + w110 * g[q110] + w001 * g[q001] + \
   w101 * g[q101] + w011 * g[q011] + w111 * g[q111])
  *n_out = LERP(f->n);
  g_out->x = LERP(f->gx);
  g_out->y = LERP(f->gy);
  g_out->z = LERP(f->gz);
#undef LERP
  return 1;
}

/* ---- grin.cpp ----------------------------------------------------------- */
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* ClampedD, grin.cpp:23-33 */
static V3 clamped_d(const Field* f, const Aabb* box, V3 r) {
  V3 q = {clampd(r.x, box->lo.x, box->hi.x), clampd(r.y, box->lo.y, box->hi.y),
          clampd(r.z, box->lo.z, box->hi.z)};
  double n;
  V3 g;
  if (!field_sample(f, q, &n, &g)) return (V3){0, 0, 0};
  return mul(g, n);
}

/* rk4_step_impl, grin.cpp:35-44 */
static void rk4_step(const Field* f, const Aabb* box, V3 r, V3 t, double h, V3* nr, V3* nt) {
  V3 a = mul(clamped_d(f, box, r), h);
  V3 b = mul(clamped_d(f, box, add(r, mul(add(mul(t, 0.5), mul(a, 0.125)), h))), h);
  V3 c = mul(clamped_d(f, box, add(r, mul(add(t, mul(b, 0.5)), h))), h);
  *nr = add(r, mul(add(t, mul(add(a, mul(b, 2.0)), 1.0 / 6.0)), h));
  *nt = add(t, mul(add(add(a, mul(b, 4.0)), c), 1.0 / 6.0));
}

/* aabb_intersect, grin.cpp:52-72; returns 0 for nullopt */
static int aabb_intersect(V3 origin, V3 dir, const Aabb* box, double* tn, double* tf) {
  double t_near = -INFINITY, t_far = INFINITY;
  const double o[3] = {origin.x, origin.y, origin.z};
  const double d[3] = {dir.x, dir.y, dir.z};
  const double lo[3] = {box->lo.x, box->lo.y, box->lo.z};
  const double hi[3] = {box->hi.x, box->hi.y, box->hi.z};
  for (int axis = 0; axis < 3; ++axis) {
    if (d[axis] == 0.0) {
      if (o[axis] < lo[axis] || o[axis] > hi[axis]) return 0;
      continue;
    }
    double t0 = (lo[axis] - o[axis]) / d[axis];
    double t1 = (hi[axis] - o[axis]) / d[axis];
    if (t0 > t1) {
      double tmp = t0;
      t0 = t1;
      t1 = tmp;
    }
    t_near = t_near < t0 ? t0 : t_near; /* std::max(t_near, t0) */
    t_far = t1 < t_far ? t1 : t_far;    /* std::min(t_far, t1)  */
  }
  if (t_far < t_near || t_far < 0.0) return 0;
  *tn = t_near < 0.0 ? 0.0 : t_near; /* std::max(t_near, 0.0) */
  *tf = t_far;
  return 1;
}

enum { TS_MISSED = 0, TS_TRACED = 1, TS_LOST = 2, TS_INVALID = 3 };

/* trace_through_volume, grin.cpp:74-134.  Updates origin/dir on kTraced. */
static int trace_through_volume(const Field* f, double h, int max_steps, V3* origin, V3* dir,
                                int* steps) {
  Aabb box = field_bounds(f);
  double tn, tf;
  *steps = 0;
  if (!aabb_intersect(*origin, *dir, &box, &tn, &tf)) return TS_MISSED;
  if (!(h > 0.0)) return TS_INVALID;
  const double kEntryNudge = 1e-9;
  V3 r = add(*origin, mul(*dir, tn + kEntryNudge));
  if (!contains(&box, r)) return TS_MISSED;
  double n_e;
  V3 g_e;
  V3 t = mul(*dir, field_sample(f, r, &n_e, &g_e) ? n_e : 1.0);
  for (int step = 0; step < max_steps; ++step) {
    V3 nr, nt;
    rk4_step(f, &box, r, t, h, &nr, &nt);
    if (!finite3(nr) || !finite3(nt)) {
      *steps = step;
      return TS_INVALID;
    }
    if (contains(&box, nr)) {
      r = nr;
      t = nt;
      continue;
    }
    double s = 1.0;
    const double r0[3] = {r.x, r.y, r.z}, r1[3] = {nr.x, nr.y, nr.z};
    const double lo[3] = {box.lo.x, box.lo.y, box.lo.z}, hi[3] = {box.hi.x, box.hi.y, box.hi.z};
    for (int axis = 0; axis < 3; ++axis) {
      double delta = r1[axis] - r0[axis];
      if (r1[axis] < lo[axis]) {
        double c = (lo[axis] - r0[axis]) / delta;
        s = c < s ? c : s;
      }
      if (r1[axis] > hi[axis]) {
        double c = (hi[axis] - r0[axis]) / delta;
        s = c < s ? c : s;
      }
    }
    s = clampd(s, 0.0, 1.0);
    V3 er = add(r, mul(sub(nr, r), s));
    V3 et = add(t, mul(sub(nt, t), s));
    *origin = er;
    *dir = normalized(et);
    *steps = step + 1;
    return TS_TRACED;
  }
  *steps = max_steps;
  return TS_LOST;
}

/* ---- optics.cpp --------------------------------------------------------- */
enum { BR_NONE = 0, BR_APERTURE = 1, BR_MISSED = 2, BR_TIR = 3 };
static const double kForwardEps = 1e-12; /* optics.cpp:13 */

/* radial_distance, optics.cpp:15-18 */
static double radial_distance(V3 p, V3 axis_point, V3 axis) {
  V3 rel = sub(p, axis_point);
  return norm(sub(rel, mul(axis, dot(rel, axis))));
}

typedef struct { V3 point, normal; } Hit;

/* intersect_plane_cap, optics.cpp:20-30 */
static int intersect_plane_cap(V3 o, V3 d, V3 point, V3 axis, double clear, Hit* hit) {
  double denom = dot(d, axis);
  if (denom == 0.0) return 0;
  double t = dot(sub(point, o), axis) / denom;
  if (t <= kForwardEps) return 0;
  V3 p = add(o, mul(d, t));
  if (radial_distance(p, point, axis) > clear) return 0;
  hit->point = p;
  hit->normal = denom < 0.0 ? axis : neg(axis);
  return 1;
}

/* intersect_sphere, optics.cpp:34-57 */
static int intersect_sphere(V3 o, V3 d, const rb_surface* s, Hit* hit) {
  if (!isfinite(s->curvature_radius))
    return intersect_plane_cap(o, d, cv(s->vertex), cv(s->axis), s->aperture_radius, hit);
  V3 center = add(cv(s->vertex), mul(cv(s->axis), s->curvature_radius));
  V3 oc = sub(o, center);
  double b = dot(oc, d);
  double c = norm2(oc) - s->curvature_radius * s->curvature_radius;
  double disc = b * b - c;
  if (disc < 0.0) return 0;
  double sq = sqrt(disc);
  const double ts[2] = {-b - sq, -b + sq};
  for (int k = 0; k < 2; ++k) {
    double t = ts[k];
    if (t <= kForwardEps) continue;
    V3 p = add(o, mul(d, t));
    if (dot(sub(p, center), sub(cv(s->vertex), center)) <= 0.0) continue;
    if (radial_distance(p, cv(s->vertex), cv(s->axis)) > s->aperture_radius) continue;
    V3 normal = dvd(sub(p, center), fabs(s->curvature_radius));
    if (dot(d, normal) > 0.0) normal = neg(normal);
    hit->point = p;
    hit->normal = normal;
    return 1;
  }
  return 0;
}

/* refract, optics.cpp:59-65; returns 0 on TIR */
static int refract(V3 dir, V3 normal, double n_i, double n_f, V3* out) {
  double eta = n_i / n_f;
  double cos_i = -dot(dir, normal);
  double k = 1.0 - eta * eta * (1.0 - cos_i * cos_i);
  if (k < 0.0) return 0;
  *out = normalized(add(mul(dir, eta), mul(normal, eta * cos_i - sqrt(k))));
  return 1;
}

/* propagate_chain, optics.cpp:143-158, with the element functions
 * apply_aperture (108-116), propagate_thin_lens (118-132),
 * propagate_through_lens (85-106), reflect_on_mirror (134-141). */
static int propagate_chain(const rb_scene* s, V3* o, V3* d) {
  for (int e = 0; e < s->n_elements; ++e) {
    const rb_element* el = &s->elements[e];
    if (el->kind == RB_ELEM_APERTURE) {
      V3 c = cv(el->center), nrm = cv(el->axis);
      double denom = dot(*d, nrm);
      if (denom == 0.0) return BR_MISSED;
      double t = dot(sub(c, *o), nrm) / denom;
      if (t <= kForwardEps) return BR_MISSED;
      V3 p = add(*o, mul(*d, t));
      if (norm(sub(p, c)) > el->radius) return BR_APERTURE;
    } else if (el->kind == RB_ELEM_THIN_LENS) {
      Hit hit;
      V3 c = cv(el->center), ax = cv(el->axis);
      if (!intersect_plane_cap(*o, *d, c, ax, 0.5 * el->diameter, &hit)) return BR_MISSED;
      double dz = dot(*d, ax);
      if (dz <= 0.0) return BR_MISSED;
      V3 focal_point = add(c, mul(*d, el->focal_length / dz));
      *o = hit.point;
      *d = normalized(mul(sub(focal_point, hit.point), el->focal_length > 0.0 ? 1.0 : -1.0));
    } else if (el->kind == RB_ELEM_SINGLET) {
      Hit fh, bh;
      V3 in_dir, out_dir;
      if (!intersect_sphere(*o, *d, &el->front, &fh)) return BR_MISSED;
      if (!refract(*d, fh.normal, el->front.n_before, el->front.n_after, &in_dir)) return BR_TIR;
      if (!intersect_sphere(fh.point, in_dir, &el->back, &bh)) return BR_MISSED;
      if (!refract(in_dir, bh.normal, el->back.n_before, el->back.n_after, &out_dir))
        return BR_TIR;
      *o = bh.point;
      *d = out_dir;
    } else { /* mirror */
      Hit hit;
      if (!intersect_sphere(*o, *d, &el->front, &hit)) return BR_MISSED;
      *o = hit.point;
      *d = sub(*d, mul(hit.normal, 2.0 * dot(*d, hit.normal))); /* reflect, optics.cpp:67 */
    }
  }
  return BR_NONE;
}

/* ---- sensor.cpp --------------------------------------------------------- */
/* intersect_sensor, sensor.cpp:27-34 */
static int intersect_sensor(const rb_sensor* s, V3 o, V3 d, V2* uv) {
  V3 n = cv(s->normal), c = cv(s->center);
  double denom = dot(d, n);
  if (denom == 0.0) return 0;
  double t = dot(sub(c, o), n) / denom;
  if (t <= 0.0) return 0;
  V3 p = add(o, mul(d, t));
  uv->x = dot(sub(p, c), cv(s->e_u));
  uv->y = dot(sub(p, c), cv(s->e_v));
  return 1;
}

typedef struct {
  int w, h;
  double* data;   /* FP64 accumulation (deterministic-tiled reference order) */
  uint64_t* fx;   /* fixed-point accumulation (radiance * 2^31), or NULL */
} Img;

/* accumulate_spot, sensor.cpp:57-122.  In fixed-point mode every contribution
 * is rounded to the nearest multiple of 2^-31 and added as an integer. */
static void accumulate_spot(Img* img, const rb_sensor* s, V2 center, double d_tau,
                            double energy) {
  const double sqrt2 = 1.41421356237309504880168872420969808;
  if (energy == 0.0) return;
  const double pitch = s->pitch;
  const int w_px = img->w, h_px = img->h;
  const double sigma = 0.25 * d_tau;
  const double cc = center.x / pitch + 0.5 * w_px;
  const double rc = 0.5 * h_px - center.y / pitch;
  if (sigma < 1e-3 * pitch) {
    int col = (int)floor(cc), row = (int)floor(rc);
    if (col >= 0 && col < w_px && row >= 0 && row < h_px) {
      size_t q = (size_t)row * w_px + col;
      if (img->fx)
        img->fx[q] += (uint64_t)llrint(energy * RB_IMAGE_FIXED_SCALE);
      else
        img->data[q] += energy;
    }
    return;
  }
  const double half_width = s->window_sigmas * sigma / pitch;
  const int c0 = (int)floor(cc - half_width), c1 = (int)floor(cc + half_width);
  const int r0 = (int)floor(rc - half_width), r1 = (int)floor(rc + half_width);
  const double inv_s = 1.0 / (sigma * sqrt2 / pitch);
  double* wu = (double*)malloc(sizeof(double) * (size_t)(c1 - c0 + 1));
  double* wv = (double*)malloc(sizeof(double) * (size_t)(r1 - r0 + 1));
  for (int c = c0; c <= c1; ++c)
    wu[c - c0] = 0.5 * (erf((c + 1 - cc) * inv_s) - erf((c - cc) * inv_s));
  for (int r = r0; r <= r1; ++r)
    wv[r - r0] = 0.5 * (erf((r + 1 - rc) * inv_s) - erf((r - rc) * inv_s));
  const double mass_u = 0.5 * (erf((c1 + 1 - cc) * inv_s) - erf((c0 - cc) * inv_s));
  const double mass_v = 0.5 * (erf((r1 + 1 - rc) * inv_s) - erf((r0 - rc) * inv_s));
  const double scale = energy / (mass_u * mass_v);
  const int cb = c0 > 0 ? c0 : 0, ce = c1 < w_px - 1 ? c1 : w_px - 1;
  const int rb = r0 > 0 ? r0 : 0, re = r1 < h_px - 1 ? r1 : h_px - 1;
  for (int r = rb; r <= re; ++r) {
    const double row_w = wv[r - r0] * scale;
    for (int c = cb; c <= ce; ++c) {
      size_t q = (size_t)r * w_px + c;
      double v = wu[c - c0] * row_w;
      if (img->fx)
        img->fx[q] += (uint64_t)llrint(v * RB_IMAGE_FIXED_SCALE);
      else
        img->data[q] += v;
    }
  }
  free(wu);
  free(wv);
}

/* spot_pixel_window, sensor.cpp:44-55 (for the tile bbox of make_tile) */
static void spot_window(const rb_sensor* s, int w, int h, V2 c, double d_tau, int* c0, int* c1,
                        int* r0, int* r1) {
  const double cc = c.x / s->pitch + 0.5 * w;
  const double rc = 0.5 * h - c.y / s->pitch;
  const double hw = s->window_sigmas * 0.25 * d_tau / s->pitch;
  int a = (int)floor(cc - hw), b = (int)floor(cc + hw), p = (int)floor(rc - hw),
      q = (int)floor(rc + hw);
  *c0 = a > 0 ? a : 0;
  *c1 = b < w - 1 ? b : w - 1;
  *r0 = p > 0 ? p : 0;
  *r1 = q < h - 1 ? q : h - 1;
}

/* ---- engine.cpp:107-140 process_source, per ray ------------------------- */
typedef struct {
  const rb_scene* s;
  const Field* field; /* NULL when no field or with_field == 0 */
  V3 e1, e2;
  int cells;
} Ctx;

static int trace_one(const Ctx* c, uint64_t source_index, V3 source, int i, double radiance,
                     V2* uv, int* steps, V3* exit_o, V3* exit_d) {
  (void)radiance;
  V3 p = aperture_point(c->s, c->e1, c->e2, c->cells, source_index, i);
  V3 to_point = sub(p, source);
  double len = norm(to_point);
  V3 o = source, d = dvd(to_point, len); /* emit_rays, raygen.cpp:74-80 */
  *steps = 0;
  if (c->field) {
    int st = trace_through_volume(c->field, c->s->delta_xi, c->s->max_steps, &o, &d, steps);
    if (st == TS_LOST || st == TS_INVALID) return RB_RAY_LOST;
  }
  if (exit_o) {
    *exit_o = o;
    *exit_d = d;
  }
  int br = propagate_chain(c->s, &o, &d);
  if (br == BR_APERTURE) return RB_RAY_APERTURE;
  if (br == BR_TIR) return RB_RAY_TIR;
  if (br != BR_NONE) return RB_RAY_MISSED;
  if (!intersect_sensor(&c->s->sensor, o, d, uv)) return RB_RAY_SENSOR_MISS;
  return RB_RAY_LANDED;
}

static void set_err(char* err, size_t len, const char* msg) {
  if (err && len) {
    strncpy(err, msg, len - 1);
    err[len - 1] = 0;
  }
}

static int validate_scene(const rb_scene* s, char* err, size_t errlen) {
  if (s->n_sources == 0) return 0;
  /* raygen.cpp:29-31, 69 (raised when the first source is processed) */
  if (s->rays_per_source < 1) {
    set_err(err, errlen, "sample_aperture_points: rays_per_source must be >= 1");
    return RB_E_INVALID;
  }
  if (s->pupil_radius <= 0.0) {
    set_err(err, errlen, "sample_aperture_points: radius must be > 0");
    return RB_E_INVALID;
  }
  if (s->wavelength <= 0.0) {
    set_err(err, errlen, "emit_rays: wavelength must be positive");
    return RB_E_INVALID;
  }
  return 0;
}

static void make_ctx(Ctx* c, const rb_scene* s, const Field* f) {
  c->s = s;
  c->field = f;
  plane_basis(cv(s->pupil_axis), &c->e1, &c->e2);
  c->cells = (int)ceil(sqrt((double)s->rays_per_source));
}

/*
 * oracle_trace: run_trace (engine.cpp:429-507) in deterministic mode.
 *   field arrays may be NULL (no field).  fixed_image (W*H uint64, may be NULL)
 *   selects fixed-point accumulation instead of out->image.  When shard_of is
 *   non-NULL only sources with shard_of[s] == shard_index are traced.
 */
int oracle_trace(const rb_scene* s, const rb_field_desc* fd, const double* fn, const double* fgx,
                 const double* fgy, const double* fgz, int with_field, int accumulate_image,
                 const int32_t* shard_of, int32_t shard_index, uint64_t* fixed_image,
                 rb_trace_out* out, char* err, size_t errlen) {
  int rc = validate_scene(s, err, errlen);
  if (rc) return rc;
  Field field;
  const Field* fp = NULL;
  if (with_field && fd && fn) {
    field.nx = fd->nx;
    field.ny = fd->ny;
    field.nz = fd->nz;
    field.origin = cv(fd->origin);
    field.spacing = cv(fd->spacing);
    field.n = fn;
    field.gx = fgx;
    field.gy = fgy;
    field.gz = fgz;
    fp = &field;
  }
  Ctx c;
  make_ctx(&c, s, fp);
  const int W = s->sensor.width_px, H = s->sensor.height_px;
  const size_t npx = (size_t)W * H;
  Img scratch = {W, H, NULL, NULL};
  if (accumulate_image) {
    if (fixed_image) {
      scratch.fx = fixed_image;
    } else {
      scratch.data = (double*)calloc(npx, sizeof(double));
      memset(out->image, 0, npx * sizeof(double));
    }
  }
  int64_t lost = 0, ap = 0, miss = 0, tir = 0, smiss = 0, landed_total = 0, steps_total = 0;
  const int N = s->rays_per_source;
  const double radiance = 1.0 / (double)N; /* emit_rays normalisation, raygen.cpp:86 */
  for (int64_t d = 0; d < s->n_sources; ++d) {
    if (shard_of && shard_of[d] != shard_index) continue;
    const uint64_t sid = s->source_ids ? (uint64_t)s->source_ids[d] : (uint64_t)d;
    const V3 src = cv(s->sources[d]);
    V2 hit_sum = {0.0, 0.0};
    int64_t landed = 0;
    int bc0 = W, bc1 = -1, br0 = H, br1 = -1;
    for (int i = 0; i < N; ++i) {
      V2 uv;
      int steps;
      int st = trace_one(&c, sid, src, i, radiance, &uv, &steps, NULL, NULL);
      steps_total += steps;
      switch (st) {
        case RB_RAY_LOST: ++lost; continue;
        case RB_RAY_APERTURE: ++ap; continue;
        case RB_RAY_TIR: ++tir; continue;
        case RB_RAY_MISSED: ++miss; continue;
        case RB_RAY_SENSOR_MISS: ++smiss; continue;
        default: break;
      }
      hit_sum.x += uv.x;
      hit_sum.y += uv.y;
      ++landed;
      if (accumulate_image) {
        /* make_tile, engine.cpp:150-179: deposits in ray order into a zeroed
         * scratch, bbox tracked with spot_pixel_window. */
        int a, b, p, q;
        spot_window(&s->sensor, W, H, uv, s->d_tau, &a, &b, &p, &q);
        if (!(b < a || q < p)) {
          bc0 = a < bc0 ? a : bc0;
          bc1 = b > bc1 ? b : bc1;
          br0 = p < br0 ? p : br0;
          br1 = q > br1 ? q : br1;
          accumulate_spot(&scratch, &s->sensor, uv, s->d_tau, radiance);
        }
      }
    }
    if (accumulate_image && scratch.data && bc1 >= bc0 && br1 >= br0) {
      /* composite_tile in source order, engine.cpp:181-187, 484 */
      for (int r = br0; r <= br1; ++r)
        for (int cc = bc0; cc <= bc1; ++cc) {
          size_t q = (size_t)r * W + cc;
          out->image[q] += scratch.data[q];
          scratch.data[q] = 0.0;
        }
    }
    if (out->hit_sum) {
      out->hit_sum[2 * d] = hit_sum.x;
      out->hit_sum[2 * d + 1] = hit_sum.y;
    }
    if (out->landed) out->landed[d] = landed;
    landed_total += landed;
  }
  free(scratch.data);
  int64_t owned = 0;
  for (int64_t d = 0; d < s->n_sources; ++d)
    if (!shard_of || shard_of[d] == shard_index) ++owned;
  out->emitted = owned * N;
  out->landed_total = landed_total;
  out->lost = lost;
  out->blocked_aperture = ap;
  out->blocked_miss = miss;
  out->blocked_tir = tir;
  out->blocked_sensor_miss = smiss;
  out->threads = 1;
  out->config_hash = s->config_hash;
  out->total_steps = steps_total;
  out->wall_seconds = 0.0;
  out->kernel_ms = 0.0;
  return 0;
}

/* Per-ray replay (same contract as rb_trace_rays), plus the ray state after
 * the volume in exit_state[6*q] (origin, dir) when non-NULL. */
int oracle_trace_rays(const rb_scene* s, const rb_field_desc* fd, const double* fn,
                      const double* fgx, const double* fgy, const double* fgz, int with_field,
                      int64_t n, const int64_t* src, const int32_t* ray, double* uv,
                      int32_t* status, int32_t* steps, double* exit_state, char* err,
                      size_t errlen) {
  int rc = validate_scene(s, err, errlen);
  if (rc) return rc;
  Field field;
  const Field* fp = NULL;
  if (with_field && fd && fn) {
    field.nx = fd->nx;
    field.ny = fd->ny;
    field.nz = fd->nz;
    field.origin = cv(fd->origin);
    field.spacing = cv(fd->spacing);
    field.n = fn;
    field.gx = fgx;
    field.gy = fgy;
    field.gz = fgz;
    fp = &field;
  }
  Ctx c;
  make_ctx(&c, s, fp);
  for (int64_t q = 0; q < n; ++q) {
    V2 h = {NAN, NAN};
    int st_steps = 0;
    V3 eo = {NAN, NAN, NAN}, ed = {NAN, NAN, NAN};
    const uint64_t sid = s->source_ids ? (uint64_t)s->source_ids[src[q]] : (uint64_t)src[q];
    int st = trace_one(&c, sid, cv(s->sources[src[q]]), ray[q], 1.0 / s->rays_per_source, &h,
                       &st_steps, &eo, &ed);
    status[q] = st;
    steps[q] = st_steps;
    uv[2 * q] = st == RB_RAY_LANDED ? h.x : NAN;
    uv[2 * q + 1] = st == RB_RAY_LANDED ? h.y : NAN;
    if (exit_state) {
      exit_state[6 * q + 0] = eo.x;
      exit_state[6 * q + 1] = eo.y;
      exit_state[6 * q + 2] = eo.z;
      exit_state[6 * q + 3] = ed.x;
      exit_state[6 * q + 4] = ed.y;
      exit_state[6 * q + 5] = ed.z;
    }
  }
  return 0;
}

/* GriddedField constructor restated (scene.cpp:53-92): n = K*rho + 1 and the
 * central / one-sided node gradients, FP64, x-fastest. */
void oracle_field_from_density(const rb_field_desc* d, const float* rho, double k, double* n,
                               double* gx, double* gy, double* gz) {
  const int nx = d->nx, ny = d->ny, nz = d->nz;
  const size_t count = (size_t)nx * ny * nz;
  for (size_t q = 0; q < count; ++q) n[q] = k * (double)rho[q] + 1.0;
#define IDX(i, j, kk) (((size_t)(kk) * ny + (j)) * nx + (i))
  for (int kk = 0; kk < nz; ++kk)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        size_t q = IDX(i, j, kk);
        if (i == 0)
          gx[q] = (n[IDX(1, j, kk)] - n[IDX(0, j, kk)]) / d->spacing.x;
        else if (i == nx - 1)
          gx[q] = (n[IDX(nx - 1, j, kk)] - n[IDX(nx - 2, j, kk)]) / d->spacing.x;
        else
          gx[q] = (n[IDX(i + 1, j, kk)] - n[IDX(i - 1, j, kk)]) / (2.0 * d->spacing.x);
        if (j == 0)
          gy[q] = (n[IDX(i, 1, kk)] - n[IDX(i, 0, kk)]) / d->spacing.y;
        else if (j == ny - 1)
          gy[q] = (n[IDX(i, ny - 1, kk)] - n[IDX(i, ny - 2, kk)]) / d->spacing.y;
        else
          gy[q] = (n[IDX(i, j + 1, kk)] - n[IDX(i, j - 1, kk)]) / (2.0 * d->spacing.y);
        if (kk == 0)
          gz[q] = (n[IDX(i, j, 1)] - n[IDX(i, j, 0)]) / d->spacing.z;
        else if (kk == nz - 1)
          gz[q] = (n[IDX(i, j, nz - 1)] - n[IDX(i, j, nz - 2)]) / d->spacing.z;
        else
          gz[q] = (n[IDX(i, j, kk + 1)] - n[IDX(i, j, kk - 1)]) / (2.0 * d->spacing.z);
      }
#undef IDX
}
