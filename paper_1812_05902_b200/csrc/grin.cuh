// grin.cuh — stage 2 of K1: ray propagation through the gridded index field.
//
// Restates trace_through_volume (reference proj/src/grin.cpp:74-134) with the
// RK4-Nystrom step of rk4_step_impl (grin.cpp:35-44), ClampedD (grin.cpp:23-33)
// and GriddedField::sample (scene.cpp:99-135), in perturbation form:
//
//   r_i = R0 + T0 * (i h) + dr_i,   t_i = T0 + dt_i
//
// where R0 is the volume entry point and T0 = dir * n(R0).  The RK4 step acts on
// the small (dr, dt) only, in FP32, with dr kept in grid units:
//   a = D(r_i) h,  b = D(r_i + (t_i/2 + a/8) h) h,  c = D(r_i + (t_i + b/2) h) h
//   dr_{i+1} = dr_i + (dt_i + (a + 2b)/6) h,   dt_{i+1} = dt_i + (a + 4b + c)/6
// The unperturbed line R0 + T0 * xi is never accumulated (it is re-evaluated
// from the step index), so FP32 rounding cannot drift the ray; R0, T0 and the
// exit cut-back are FP64 (<= 4e-5 px vs FP64).
// Included by kernels.cu inside namespace rbk::(anonymous), after the FP64
// vector helpers and the status enums.
#pragma once


struct GridView {
  const float4* __restrict__ g;
  unsigned nx, nxny, ix, iy, iz;  // row / plane strides, last cell index per axis
  float mx, my, mz;               // n - 1 per axis: the box in grid coordinates
};

// D = n grad(n) at grid coordinates (qx, qy, qz): trilinear interpolation of
// the float4 nodes (n-1, dn/dx, dn/dy, dn/dz) with the point clamped to the box
// first.  Index clamp: the unsigned conversion saturates negatives to cell 0;
// the fraction is saturated to [0, 1], which together equal clamping q.
__device__ __forceinline__ float3 sample_d(const GridView& G, float qx, float qy, float qz) {
  const unsigned i = min(__float2uint_rz(qx), G.ix);
  const unsigned j = min(__float2uint_rz(qy), G.iy);
  const unsigned k = min(__float2uint_rz(qz), G.iz);
  const float fx = __saturatef(qx - (float)i);
  const float fy = __saturatef(qy - (float)j);
  const float fz = __saturatef(qz - (float)k);
  const float4* p0 = G.g + (k * G.nxny + j * G.nx + i);
  const float4* p1 = p0 + G.nxny;
  const float4 c000 = __ldg(p0), c100 = __ldg(p0 + 1);
  const float4 c010 = __ldg(p0 + G.nx), c110 = __ldg(p0 + G.nx + 1);
  const float4 c001 = __ldg(p1), c101 = __ldg(p1 + 1);
  const float4 c011 = __ldg(p1 + G.nx), c111 = __ldg(p1 + G.nx + 1);
  const float gx = 1.0f - fx, gy = 1.0f - fy, gz = 1.0f - fz;
  const float w00 = gx * gy, w10 = fx * gy, w01 = gx * fy, w11 = fx * fy;
  const float w000 = w00 * gz, w100 = w10 * gz, w010 = w01 * gz, w110 = w11 * gz;
  const float w001 = w00 * fz, w101 = w10 * fz, w011 = w01 * fz, w111 = w11 * fz;
#define RB_LERP(ch)                                                                         \
  (w000 * c000.ch + w100 * c100.ch + w010 * c010.ch + w110 * c110.ch + w001 * c001.ch +    \
   w101 * c101.ch + w011 * c011.ch + w111 * c111.ch)
  const float n = 1.0f + RB_LERP(x);
  return make_float3(RB_LERP(y) * n, RB_LERP(z) * n, RB_LERP(w) * n);
#undef RB_LERP
}

__device__ __forceinline__ float sample_nm1(const GridView& G, float qx, float qy, float qz) {
  const unsigned i = min(__float2uint_rz(qx), G.ix);
  const unsigned j = min(__float2uint_rz(qy), G.iy);
  const unsigned k = min(__float2uint_rz(qz), G.iz);
  const float fx = __saturatef(qx - (float)i);
  const float fy = __saturatef(qy - (float)j);
  const float fz = __saturatef(qz - (float)k);
  const float* p0 = reinterpret_cast<const float*>(G.g + (k * G.nxny + j * G.nx + i));
  const float* p1 = p0 + 4 * G.nxny;
  const float gx = 1.0f - fx, gy = 1.0f - fy, gz = 1.0f - fz;
  return gx * gy * gz * __ldg(p0) + fx * gy * gz * __ldg(p0 + 4) +
         gx * fy * gz * __ldg(p0 + 4 * G.nx) + fx * fy * gz * __ldg(p0 + 4 * G.nx + 4) +
         gx * gy * fz * __ldg(p1) + fx * gy * fz * __ldg(p1 + 4) +
         gx * fy * fz * __ldg(p1 + 4 * G.nx) + fx * fy * fz * __ldg(p1 + 4 * G.nx + 4);
}

__device__ __forceinline__ bool box_contains(const KScene& S, double3 p) {  // Aabb::contains
  return p.x >= S.box_lo.x && p.x <= S.box_hi.x && p.y >= S.box_lo.y && p.y <= S.box_hi.y &&
         p.z >= S.box_lo.z && p.z <= S.box_hi.z;
}

// aabb_intersect, grin.cpp:52-72 (FP64, once per ray).
__device__ __forceinline__ bool aabb_intersect(const KScene& S, double3 o, double3 d, double& tn) {
  double t_near = -INFINITY, t_far = INFINITY;
  const double oo[3] = {o.x, o.y, o.z}, dd[3] = {d.x, d.y, d.z};
  const double lo[3] = {S.box_lo.x, S.box_lo.y, S.box_lo.z};
  const double hi[3] = {S.box_hi.x, S.box_hi.y, S.box_hi.z};
#pragma unroll
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

// Returns kMissed / kTraced / kLost / kInvalid; on kTraced (o, d) is the exit ray.
__device__ __forceinline__ int grin_trace(const KScene& S, double3& o, double3& d, int& steps) {
  steps = 0;
  double tn;
  if (!aabb_intersect(S, o, d, tn)) return kMissed;
  if (!(S.h > 0.0)) return kInvalid;
  const double3 R0 = o + d * (tn + 1e-9);  // kEntryNudge, grin.cpp:85-88
  if (!box_contains(S, R0)) return kMissed;

  GridView G;
  G.g = S.grid;
  G.nx = (unsigned)S.nx;
  G.nxny = (unsigned)S.nx * (unsigned)S.ny;
  G.ix = (unsigned)S.nx - 2;
  G.iy = (unsigned)S.ny - 2;
  G.iz = (unsigned)S.nz - 2;
  G.mx = (float)(S.nx - 1);
  G.my = (float)(S.ny - 1);
  G.mz = (float)(S.nz - 1);

  const float q0x = (float)((R0.x - S.origin.x) / S.spacing.x);
  const float q0y = (float)((R0.y - S.origin.y) / S.spacing.y);
  const float q0z = (float)((R0.z - S.origin.z) / S.spacing.z);
  const double n_e = 1.0 + (double)sample_nm1(G, q0x, q0y, q0z);
  const double3 T0 = d * n_e;  // grin.cpp:91-92
  // Per-axis constants (grid units).  hs = h / spacing.
  const double hsx = S.h / S.spacing.x, hsy = S.h / S.spacing.y, hsz = S.h / S.spacing.z;
  const float ax = (float)(T0.x * hsx), ay = (float)(T0.y * hsy), az = (float)(T0.z * hsz);
  const float hx = (float)hsx, hy = (float)hsy, hz = (float)hsz;        // dt -> dr
  const float kbx = (float)(0.125 * S.h * hsx), kby = (float)(0.125 * S.h * hsy),
              kbz = (float)(0.125 * S.h * hsz);                         // a/8 h
  const float kcx = (float)(0.5 * S.h * hsx), kcy = (float)(0.5 * S.h * hsy),
              kcz = (float)(0.5 * S.h * hsz);                           // b/2 h
  const float krx = (float)(S.h * hsx / 6.0), kry = (float)(S.h * hsy / 6.0),
              krz = (float)(S.h * hsz / 6.0);                           // (a+2b)/6 h
  const float kt = (float)(S.h / 6.0);                                  // (a+4b+c)/6
  const float hhx = 0.5f * hx, hhy = 0.5f * hy, hhz = 0.5f * hz;

  float drx = 0.f, dry = 0.f, drz = 0.f, dtx = 0.f, dty = 0.f, dtz = 0.f;
  float pax = q0x, pay = q0y, paz = q0z;  // unperturbed line at xi = step * h
  const int max_steps = S.max_steps;
  for (int step = 0; step < max_steps; ++step) {
    const float fs = (float)step;
    const float pbx = fmaf(ax, fs + 0.5f, q0x), pby = fmaf(ay, fs + 0.5f, q0y),
                pbz = fmaf(az, fs + 0.5f, q0z);
    const float pcx = fmaf(ax, fs + 1.0f, q0x), pcy = fmaf(ay, fs + 1.0f, q0y),
                pcz = fmaf(az, fs + 1.0f, q0z);
    const float3 Da = sample_d(G, pax + drx, pay + dry, paz + drz);
    const float3 Db = sample_d(G, fmaf(Da.x, kbx, fmaf(dtx, hhx, pbx + drx)),
                               fmaf(Da.y, kby, fmaf(dty, hhy, pby + dry)),
                               fmaf(Da.z, kbz, fmaf(dtz, hhz, pbz + drz)));
    const float bx = fmaf(dtx, hx, drx), by = fmaf(dty, hy, dry), bz = fmaf(dtz, hz, drz);
    const float3 Dc = sample_d(G, fmaf(Db.x, kcx, pcx + bx), fmaf(Db.y, kcy, pcy + by),
                               fmaf(Db.z, kcz, pcz + bz));
    const float ndrx = fmaf(fmaf(Db.x, 2.0f, Da.x), krx, bx);
    const float ndry = fmaf(fmaf(Db.y, 2.0f, Da.y), kry, by);
    const float ndrz = fmaf(fmaf(Db.z, 2.0f, Da.z), krz, bz);
    const float ndtx = fmaf(fmaf(Db.x, 4.0f, Da.x) + Dc.x, kt, dtx);
    const float ndty = fmaf(fmaf(Db.y, 4.0f, Da.y) + Dc.y, kt, dty);
    const float ndtz = fmaf(fmaf(Db.z, 4.0f, Da.z) + Dc.z, kt, dtz);
    const float qx = pcx + ndrx, qy = pcy + ndry, qz = pcz + ndrz;
    // Inside the box (grid coordinates) -> accept (grin.cpp:101-106).  NaN
    // compares false, so a non-finite state always takes the exit path.
    if (qx >= 0.0f && qx <= G.mx && qy >= 0.0f && qy <= G.my && qz >= 0.0f && qz <= G.mz) {
      drx = ndrx;
      dry = ndry;
      drz = ndrz;
      dtx = ndtx;
      dty = ndty;
      dtz = ndtz;
      pax = pcx;
      pay = pcy;
      paz = pcz;
      continue;
    }
    if (!(isfinite(ndrx) && isfinite(ndry) && isfinite(ndrz) && isfinite(ndtx) &&
          isfinite(ndty) && isfinite(ndtz))) {
      steps = step;
      return kInvalid;  // grin.cpp:99
    }
    // Crossed the boundary: cut back to the first face crossing (grin.cpp:110-130),
    // evaluated on the FP64 reconstruction of both states.
    const double xi0 = (double)step * S.h, xi1 = (double)(step + 1) * S.h;
    const double3 r0 = make_double3(R0.x + T0.x * xi0 + (double)drx * S.spacing.x,
                                    R0.y + T0.y * xi0 + (double)dry * S.spacing.y,
                                    R0.z + T0.z * xi0 + (double)drz * S.spacing.z);
    const double3 r1 = make_double3(R0.x + T0.x * xi1 + (double)ndrx * S.spacing.x,
                                    R0.y + T0.y * xi1 + (double)ndry * S.spacing.y,
                                    R0.z + T0.z * xi1 + (double)ndrz * S.spacing.z);
    const double3 t0 = make_double3(T0.x + (double)dtx, T0.y + (double)dty, T0.z + (double)dtz);
    const double3 t1 =
        make_double3(T0.x + (double)ndtx, T0.y + (double)ndty, T0.z + (double)ndtz);
    double s = 1.0;
    const double a0[3] = {r0.x, r0.y, r0.z}, a1[3] = {r1.x, r1.y, r1.z};
    const double lo[3] = {S.box_lo.x, S.box_lo.y, S.box_lo.z};
    const double hi[3] = {S.box_hi.x, S.box_hi.y, S.box_hi.z};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double delta = a1[a] - a0[a];
      if (a1[a] < lo[a]) s = fmin(s, (lo[a] - a0[a]) / delta);
      if (a1[a] > hi[a]) s = fmin(s, (hi[a] - a0[a]) / delta);
    }
    s = fmin(fmax(s, 0.0), 1.0);
    o = r0 + (r1 - r0) * s;
    d = normalized(t0 + (t1 - t0) * s);
    steps = step + 1;
    return kTraced;
  }
  steps = max_steps;
  return kLost;
}

