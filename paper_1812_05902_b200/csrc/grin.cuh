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
// Included by render.cuh inside namespace rbk::(anonymous), after the FP64
// vector helpers and the status enums.
#pragma once

#ifndef RB_UNIFORM_RELOAD
#define RB_UNIFORM_RELOAD 0  // see sample_d_poly
#endif
#ifndef RB_NPLUS1
#define RB_NPLUS1 1  // see cell_coefficients (measured +2.0% tomo, +1.8% bos)
#endif
#ifndef RB_SHALLOW_TREE
#define RB_SHALLOW_TREE 1  // see poly_eval (tomo +1.2%, bos +1.0%, 1024^3 +0.9%)
#endif
#ifndef RB_BFROMQ
#define RB_BFROMQ 1  // see the stage-b point in grin_trace (+0.5% more)
#endif


// Grid geometry, read straight from the kernel parameters (constant bank) so
// it occupies no registers in the RK4 loop.
struct GridView {
  const KScene& S;
  __device__ __forceinline__ explicit GridView(const KScene& s) : S(s) {}
};

// D = n grad(n) at grid coordinates q: the trilinear interpolation of the float4
// nodes (n-1, dn/dx, dn/dy, dn/dz) of GriddedField::sample (scene.cpp:99-135)
// with the point clamped to the box first (ClampedD, grin.cpp:23-33).  Index
// clamp: the unsigned conversion saturates negatives to cell 0; the fraction
// is saturated to [0, 1], which together equal clamping q.
//
// Cached cell in polynomial form.  On a cell change the 8 corners are loaded
// once and turned into the coefficients of
//   v(fx,fy,fz) = a + b fx + c fy + d fz + e fx fy + f fx fz + g fy fz + h fx fy fz
// (the trilinear interpolant of GriddedField::sample, scene.cpp:117-133, in
// another basis); a sample then costs 7 FFMA per channel in Horner form and
// a 3-FADD "still in the cell" test instead of the index/weight computation.
struct CellPoly {
  float ox, oy, oz;  // cached cell origin (grid coordinates); ox = -1e30 = empty
  float4 a, b, c, d, e, f, g, h;
};

__device__ __forceinline__ float4 f4sub(float4 p, float4 q) {
  return make_float4(p.x - q.x, p.y - q.y, p.z - q.z, p.w - q.w);
}

// Corner values -> polynomial coefficients (shared by the in-loop reload and
// the table build so both give the same bits).
__device__ __forceinline__ void cell_coefficients(float4 c000, float4 c100, float4 c010,
                                                  float4 c110, float4 c001, float4 c101,
                                                  float4 c011, float4 c111, float4& a, float4& b,
                                                  float4& c, float4& d, float4& e, float4& f,
                                                  float4& g, float4& h) {
  // RB_NPLUS1: the constant term of the n channel carries the +1, so a sample
  // yields n itself (one FADD less per sample; n is only a factor of D = n grad n,
  // so its FP32 rounding at magnitude 1 is a 6e-8 relative error of D)
  a = RB_NPLUS1 ? make_float4(c000.x + 1.0f, c000.y, c000.z, c000.w) : c000;
  b = f4sub(c100, c000);
  c = f4sub(c010, c000);
  d = f4sub(c001, c000);
  const float4 e0 = f4sub(c110, c010), f0 = f4sub(c101, c001), g0 = f4sub(c011, c001);
  e = f4sub(e0, b);
  f = f4sub(f0, b);
  g = f4sub(g0, c);
  h = f4sub(f4sub(f4sub(c111, c011), e0), f);  // (c111-c011) - (c110-c010) - (c101-c001) + b
}

// kCells: read the cell's coefficients from the precomputed table (one 128 B
// line, computed by build_cells_kernel with exactly these FP32 subtractions, so
// both forms are bit-identical) instead of deriving them from the 8 corners.
template <bool kCells>
__device__ __forceinline__ void poly_load(const GridView& G, CellPoly& P, float qx, float qy,
                                          float qz, float& fx, float& fy, float& fz) {
  const unsigned i = min(__float2uint_rz(qx), G.S.g_ix);
  const unsigned j = min(__float2uint_rz(qy), G.S.g_iy);
  const unsigned k = min(__float2uint_rz(qz), G.S.g_iz);
  const float ox = (float)i, oy = (float)j, oz = (float)k;
  // ClampedD: points outside the box use the face value (fraction saturated)
  fx = __saturatef(qx - ox);
  fy = __saturatef(qy - oy);
  fz = __saturatef(qz - oz);
  if (ox == P.ox && oy == P.oy && oz == P.oz) return;
  P.ox = ox;
  P.oy = oy;
  P.oz = oz;
  if (kCells) {
    RB_CHECK(G.S, k * G.S.c_nxny + j * G.S.c_nx + i < G.S.n_cells, 6);
    const float4* c = G.S.cell_table[k * G.S.c_nxny + j * G.S.c_nx + i].c;
    P.a = __ldg(c);
    P.b = __ldg(c + 1);
    P.c = __ldg(c + 2);
    P.d = __ldg(c + 3);
    P.e = __ldg(c + 4);
    P.f = __ldg(c + 5);
    P.g = __ldg(c + 6);
    P.h = __ldg(c + 7);  // (LDG.256 pairs measured 2% slower)
    return;
  }
  RB_CHECK(G.S, (k + 1) * G.S.g_nxny + (j + 1) * G.S.g_nx + i + 1 <
                   G.S.g_nxny * (unsigned)G.S.nz, 7);
  const float4* p0 = G.S.grid + (k * G.S.g_nxny + j * G.S.g_nx + i);
  const float4* p1 = p0 + G.S.g_nxny;
  const float4 c000 = __ldg(p0), c100 = __ldg(p0 + 1), c010 = __ldg(p0 + G.S.g_nx),
               c110 = __ldg(p0 + G.S.g_nx + 1), c001 = __ldg(p1), c101 = __ldg(p1 + 1),
               c011 = __ldg(p1 + G.S.g_nx), c111 = __ldg(p1 + G.S.g_nx + 1);
  cell_coefficients(c000, c100, c010, c110, c001, c101, c011, c111, P.a, P.b, P.c, P.d, P.e, P.f,
                    P.g, P.h);
}

#ifndef RB_FFMA2
#define RB_FFMA2 1
#endif
// Packed FP32 pairs (sm_100 FFMA2 / FMUL2: two lanes per instruction, each
// rounded exactly like fmaf / a single multiply, so results are bit-identical
// to the scalar form).  A scalar operand packed as {s, s} becomes the
// instruction's broadcast (.F32) operand.
__device__ __forceinline__ unsigned long long f2pk(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 f2up(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(float s, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2pk(s, s)), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long fmul2(float s, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pk(s, s)), "l"(b));
  return d;
}

__device__ __forceinline__ float3 poly_eval(const CellPoly& P, float fx, float fy, float fz) {
#if RB_FFMA2
#if RB_SHALLOW_TREE
  // depth-3 tree, the same 7 FMAs per channel: the four fz terms are
  // independent, then (b+fz f) fx + (a+fz d) and (e+fz h) fx + (c+fz g), then fy:
  //   v = [(a + fz d) + fx (b + fz f)] + fy [(c + fz g) + fx (e + fz h)]
  // (the Horner tree below chains 4 FMAs; a sample's latency is one FMA shorter)
#define RB_HORNER2(lo, hi)                                                                      \
  ffma2(fy,                                                                                     \
        ffma2(fx, ffma2(fz, f2pk(P.h.lo, P.h.hi), f2pk(P.e.lo, P.e.hi)),                        \
              ffma2(fz, f2pk(P.g.lo, P.g.hi), f2pk(P.c.lo, P.c.hi))),                           \
        ffma2(fx, ffma2(fz, f2pk(P.f.lo, P.f.hi), f2pk(P.b.lo, P.b.hi)),                        \
              ffma2(fz, f2pk(P.d.lo, P.d.hi), f2pk(P.a.lo, P.a.hi))))
#else
  // the same Horner tree as below, channels (x, y) and (z, w) in pairs
#define RB_HORNER2(lo, hi)                                                                      \
  ffma2(fx,                                                                                     \
        ffma2(fz, f2pk(P.f.lo, P.f.hi),                                                         \
              ffma2(fy, ffma2(fz, f2pk(P.h.lo, P.h.hi), f2pk(P.e.lo, P.e.hi)),                   \
                    f2pk(P.b.lo, P.b.hi))),                                                     \
        ffma2(fy, ffma2(fz, f2pk(P.g.lo, P.g.hi), f2pk(P.c.lo, P.c.hi)),                        \
              ffma2(fz, f2pk(P.d.lo, P.d.hi), f2pk(P.a.lo, P.a.hi))))
#endif
  const float2 xy = f2up(RB_HORNER2(x, y));
  const unsigned long long zw = RB_HORNER2(z, w);
#undef RB_HORNER2
  const float n = RB_NPLUS1 ? xy.x : 1.0f + xy.x;
  const float2 nzw = f2up(fmul2(n, zw));
  return make_float3(xy.y * n, nzw.x, nzw.y);
#else
#define RB_HORNER(ch)                                                                         \
  fmaf(fx, fmaf(fz, P.f.ch, fmaf(fy, fmaf(fz, P.h.ch, P.e.ch), P.b.ch)),                     \
       fmaf(fy, fmaf(fz, P.g.ch, P.c.ch), fmaf(fz, P.d.ch, P.a.ch)))
  const float n = RB_NPLUS1 ? RB_HORNER(x) : 1.0f + RB_HORNER(x);
  return make_float3(RB_HORNER(y) * n, RB_HORNER(z) * n, RB_HORNER(w) * n);
#undef RB_HORNER
#endif
}

template <bool kCells>
__device__ __forceinline__ float3 sample_d_poly(const GridView& G, CellPoly& P, float qx, float qy,
                                                float qz) {
  float fx = qx - P.ox, fy = qy - P.oy, fz = qz - P.oz;
  // fast path: inside the cached cell.  For IEEE floats "0 <= f <= 1" is
  // "bits(f) <= bits(1.0f)" as unsigned integers (negative values, -0.0 and
  // NaN all compare above), so one VIMNMX3 + one ISETP test all three axes.
  const bool stay = __vimax3_u32(__float_as_uint(fx), __float_as_uint(fy), __float_as_uint(fz)) <=
                    0x3f800000u;
#if RB_UNIFORM_RELOAD
  // Warp-uniform variant: when any active lane leaves its cell all active lanes
  // take the reload path.  Measured equal to the per-lane branch (the 32 rays
  // of a compact pupil patch cross cell faces together), so it is off.
  const bool reload = __any_sync(__activemask(), !stay);
#else
  const bool reload = !stay;
#endif
  if (reload) poly_load<kCells>(G, P, qx, qy, qz, fx, fy, fz);
  return poly_eval(P, fx, fy, fz);
}

#define RB_SAMPLE_D(qx, qy, qz) sample_d_poly<kCells>(G, cache, qx, qy, qz)

__device__ __forceinline__ float sample_nm1(const GridView& G, float qx, float qy, float qz) {
  const unsigned i = min(__float2uint_rz(qx), G.S.g_ix);
  const unsigned j = min(__float2uint_rz(qy), G.S.g_iy);
  const unsigned k = min(__float2uint_rz(qz), G.S.g_iz);
  const float fx = __saturatef(qx - (float)i);
  const float fy = __saturatef(qy - (float)j);
  const float fz = __saturatef(qz - (float)k);
  RB_CHECK(G.S, (k + 1) * G.S.g_nxny + (j + 1) * G.S.g_nx + i + 1 <
                   G.S.g_nxny * (unsigned)G.S.nz, 13);
  const float* p0 = reinterpret_cast<const float*>(G.S.grid + (k * G.S.g_nxny + j * G.S.g_nx + i));
  const float* p1 = p0 + 4 * G.S.g_nxny;
  const float gx = 1.0f - fx, gy = 1.0f - fy, gz = 1.0f - fz;
  return gx * gy * gz * __ldg(p0) + fx * gy * gz * __ldg(p0 + 4) +
         gx * fy * gz * __ldg(p0 + 4 * G.S.g_nx) + fx * fy * gz * __ldg(p0 + 4 * G.S.g_nx + 4) +
         gx * gy * fz * __ldg(p1) + fx * gy * fz * __ldg(p1 + 4) +
         gx * fy * fz * __ldg(p1 + 4 * G.S.g_nx) + fx * fy * fz * __ldg(p1 + 4 * G.S.g_nx + 4);
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
// scratch: 7 doubles of shared memory for this thread; R0 and T0 are parked
// there during the RK4 loop (they are only needed again at the exit).
template <bool kCells>
__device__ __forceinline__ int grin_trace(const KScene& S, double3& o, double3& d,
                                          unsigned* steps_acc,
                                          double* scratch) {
  double tn;
  if (!aabb_intersect(S, o, d, tn)) return kMissed;
  if (!(S.h > 0.0)) return kInvalid;
  const double3 R0 = o + d * (tn + 1e-9);  // kEntryNudge, grin.cpp:85-88
  if (!box_contains(S, R0)) return kMissed;

  const GridView G(S);

  const float q0x = (float)((R0.x - S.origin.x) / S.spacing.x);
  const float q0y = (float)((R0.y - S.origin.y) / S.spacing.y);
  const float q0z = (float)((R0.z - S.origin.z) / S.spacing.z);
  const double n_e = 1.0 + (double)sample_nm1(G, q0x, q0y, q0z);
  const double3 T0 = d * n_e;  // grin.cpp:91-92
  // Per-ray advance of the unperturbed line per step, in grid units; the other
  // RK4 constants are scene-uniform (KScene::hx ... kt).
  const float ax = (float)(T0.x * S.h / S.spacing.x), ay = (float)(T0.y * S.h / S.spacing.y),
              az = (float)(T0.z * S.h / S.spacing.z);
  // park the FP64 entry state; it is read back only at the exit
  scratch[0] = R0.x;
  scratch[1] = R0.y;
  scratch[2] = R0.z;
  scratch[3] = T0.x;
  scratch[4] = T0.y;
  scratch[5] = T0.z;

  float drx = 0.f, dry = 0.f, drz = 0.f, dtx = 0.f, dty = 0.f, dtz = 0.f;
  // stage-a point (grid units) of the current step: the unperturbed line plus
  // dr, i.e. the previous step's accepted end point qx = pcx + ndrx (the same
  // FADD, so carrying it is bit-identical to recomputing pa + dr)
  float qax = q0x + 0.f, qay = q0y + 0.f, qaz = q0z + 0.f;
  CellPoly cache;
  cache.ox = cache.oy = cache.oz = -1e30f;
  const int max_steps = S.max_steps;
#ifndef RB_STEP_UNROLL
#define RB_STEP_UNROLL 1
#endif
  constexpr int kStepUnroll = RB_STEP_UNROLL;
  // The step count goes straight into the caller's (shared-memory) counter
  // after the loop: returned as a value it was spilled, and the compiler sank
  // the spill store into the loop (two local stores per RK4 step).
  int status = kLost;
  int step = 0;
#pragma unroll kStepUnroll
  for (; step < max_steps; ++step) {
    const float fs = (float)step;
#if RB_BFROMQ
    // stage-b base r_i + T0 h/2 taken from the stage-a point (q_a = anchor_i +
    // dr_i) instead of anchor_{i+1/2} + dr_i: one FFMA instead of FFMA + FADD
    // per axis; the anchor of the accepted point (pc below) is still
    // re-evaluated from the step index, so nothing accumulates
    const float pbx = fmaf(ax, 0.5f, qax), pby = fmaf(ay, 0.5f, qay), pbz = fmaf(az, 0.5f, qaz);
    const float pdx = 0.f, pdy = 0.f, pdz = 0.f;
#else
    const float pbx = fmaf(ax, fs + 0.5f, q0x), pby = fmaf(ay, fs + 0.5f, q0y),
                pbz = fmaf(az, fs + 0.5f, q0z);
    const float pdx = drx, pdy = dry, pdz = drz;
#endif
    const float pcx = fmaf(ax, fs + 1.0f, q0x), pcy = fmaf(ay, fs + 1.0f, q0y),
                pcz = fmaf(az, fs + 1.0f, q0z);
    const float3 Da = RB_SAMPLE_D(qax, qay, qaz);
    const float3 Db = RB_SAMPLE_D(fmaf(Da.x, S.kbx, fmaf(dtx, S.hhx, RB_BFROMQ ? pbx : pbx + pdx)),
                               fmaf(Da.y, S.kby, fmaf(dty, S.hhy, RB_BFROMQ ? pby : pby + pdy)),
                               fmaf(Da.z, S.kbz, fmaf(dtz, S.hhz, RB_BFROMQ ? pbz : pbz + pdz)));
    const float bx = fmaf(dtx, S.hx, drx), by = fmaf(dty, S.hy, dry), bz = fmaf(dtz, S.hz, drz);
    const float3 Dc = RB_SAMPLE_D(fmaf(Db.x, S.kcx, pcx + bx), fmaf(Db.y, S.kcy, pcy + by),
                               fmaf(Db.z, S.kcz, pcz + bz));
    const float ndrx = fmaf(fmaf(Db.x, 2.0f, Da.x), S.krx, bx);
    const float ndry = fmaf(fmaf(Db.y, 2.0f, Da.y), S.kry, by);
    const float ndrz = fmaf(fmaf(Db.z, 2.0f, Da.z), S.krz, bz);
    const float ndtx = fmaf(fmaf(Db.x, 4.0f, Da.x) + Dc.x, S.kt, dtx);
    const float ndty = fmaf(fmaf(Db.y, 4.0f, Da.y) + Dc.y, S.kt, dty);
    const float ndtz = fmaf(fmaf(Db.z, 4.0f, Da.z) + Dc.z, S.kt, dtz);
    const float qx = pcx + ndrx, qy = pcy + ndry, qz = pcz + ndrz;
    // Inside the box (grid coordinates) -> accept (grin.cpp:101-106).  NaN
    // compares false, so a non-finite state always takes the exit path.
    // (as in sample_d_poly: 0 <= q <= m is bits(q) <= bits(m) unsigned)
    if (__float_as_uint(qx) <= __float_as_uint(G.S.g_mx) &&
        __float_as_uint(qy) <= __float_as_uint(G.S.g_my) &&
        __float_as_uint(qz) <= __float_as_uint(G.S.g_mz)) {
      drx = ndrx;
      dry = ndry;
      drz = ndrz;
      dtx = ndtx;
      dty = ndty;
      dtz = ndtz;
      qax = qx;
      qay = qy;
      qaz = qz;
      continue;
    }
    if (!(isfinite(ndrx) && isfinite(ndry) && isfinite(ndrz) && isfinite(ndtx) &&
          isfinite(ndty) && isfinite(ndtz))) {
      status = kInvalid;  // grin.cpp:99
      break;
    }
    // Crossed the boundary: cut back to the first face crossing (grin.cpp:110-130),
    // evaluated on the FP64 reconstruction of both states.
    const volatile double* vs = scratch;
    const double3 R0 = make_double3(vs[0], vs[1], vs[2]);
    const double3 T0 = make_double3(vs[3], vs[4], vs[5]);
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
    status = kTraced;
    break;
  }
  // 32-bit on purpose: a 64-bit add of the exit count made the optimiser widen
  // the loop counter itself to 64 bits (and spill its high word every step)
  *steps_acc += (unsigned)(step + (status == kTraced ? 1 : 0));  // kLost: step == max_steps
  return status;
}

