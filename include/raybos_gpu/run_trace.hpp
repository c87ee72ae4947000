// raybos_gpu/run_trace.hpp — header-only C++ drop-in for the reference hot path.
//
//   raybos::TraceOutputs raybos_gpu::run_trace(const raybos::SceneSetup& setup,
//                                              bool with_field, bool accumulate_image,
//                                              const raybos::RunConfig& run);
//
// has exactly the signature and result types of raybos::run_trace
// (reference proj/include/raybos/engine.hpp:73-78) and is compiled against the
// reference's own public headers.  It flattens the SceneSetup into the C-ABI
// structs of raybos_gpu.h, uploads the GriddedField once per field object
// (node_n / node_grad, scene.hpp:88-92), calls rb_trace, and refills
// TraceOutputs / RunReport so RunReport::accounting_ok() holds
// (engine.hpp:34).  Callers above run_trace (render, bos_run — engine.cpp:509-603)
// keep their host code, quantize/PGM/CSV formats unchanged.
//
// Device selection: RAYBOS_GPUS (count, default all visible) and
// RAYBOS_FIRST_GPU (default 0).  RunConfig::threads is ignored; the report's
// `threads` is the number of GPUs used.  Results are deterministic for any
// GPU count (integer image accumulation), so RunConfig::deterministic is
// always honoured.
#pragma once

#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

#include "raybos/engine.hpp"
#include "raybos_gpu.h"

namespace raybos_gpu {

namespace detail {

inline rb_vec3 v3(const raybos::Vec3& v) { return {v.x, v.y, v.z}; }

inline rb_surface surf(const raybos::SphericalSurface& s) {
  return {v3(s.vertex), v3(s.axis), s.curvature_radius, s.aperture_radius, s.n_before, s.n_after};
}

[[noreturn]] inline void raise(int rc, const char* msg) {
  if (rc == RB_E_INVALID) throw std::invalid_argument(msg);
  throw std::runtime_error(std::string("raybos_gpu: ") + msg);
}

// One process-wide context: device streams, the resident grid, buffers.
struct Context {
  rb_ctx* ctx = nullptr;
  // The uploaded grid, tracked by ownership (not by address: a new field can be
  // allocated where a freed one lived).
  std::weak_ptr<const raybos::GriddedField> field;
  bool has_field = false;
  bool external = false;  // grid streamed by load_medium_gvol, no host GriddedField
  std::mutex mu;

  Context() {
    const char* n = std::getenv("RAYBOS_GPUS");
    const char* f = std::getenv("RAYBOS_FIRST_GPU");
    char err[512] = {0};
    const int rc = rb_create(n ? std::atoi(n) : 0, f ? std::atoi(f) : 0, &ctx, err, sizeof(err));
    if (rc) raise(rc, err);
  }
  ~Context() { rb_destroy(ctx); }

  void ensure_field(const std::shared_ptr<const raybos::GriddedField>& sp) {
    if (has_field && !field.expired() && field.lock() == sp) return;
    external = false;
    if (!sp) {
      rb_clear_field(ctx);
      field.reset();
      has_field = false;
      return;
    }
    const raybos::GriddedField* g = sp.get();
    rb_field_desc d{};
    d.nx = g->nx();
    d.ny = g->ny();
    d.nz = g->nz();
    d.origin = v3(g->origin());
    d.spacing = v3(g->spacing());
    const size_t cnt = static_cast<size_t>(d.nx) * d.ny * d.nz;
    std::vector<double> n(cnt), gx(cnt), gy(cnt), gz(cnt);
    size_t q = 0;
    for (int k = 0; k < d.nz; ++k)
      for (int j = 0; j < d.ny; ++j)
        for (int i = 0; i < d.nx; ++i, ++q) {
          n[q] = g->node_n(i, j, k);
          const raybos::Vec3 gr = g->node_grad(i, j, k);
          gx[q] = gr.x;
          gy[q] = gr.y;
          gz[q] = gr.z;
        }
    const int rc = rb_set_field_nodes(ctx, &d, n.data(), gx.data(), gy.data(), gz.data());
    if (rc) raise(rc, rb_last_error(ctx));
    field = sp;
    has_field = true;
  }
};

inline Context& context() {
  static Context c;
  return c;
}

}  // namespace detail

namespace detail {

// SceneSetup -> rb_scene (engine.hpp:40-60); the vectors back the pointers.
struct FlatScene {
  std::vector<rb_vec3> sources;
  std::vector<rb_element> elements;
  rb_scene s{};
};

inline void flatten(const raybos::SceneSetup& setup, FlatScene& f) {
  f.sources.clear();
  for (const raybos::Vec3& v : setup.sources) f.sources.push_back(v3(v));
  f.elements.clear();
  for (const raybos::OpticalElement& e : setup.elements) {
    rb_element r{};
    std::visit(
        [&](const auto& x) {
          using T = std::decay_t<decltype(x)>;
          if constexpr (std::is_same_v<T, raybos::Aperture>) {
            r.kind = RB_ELEM_APERTURE;
            r.center = v3(x.center);
            r.axis = v3(x.normal);
            r.radius = x.radius;
          } else if constexpr (std::is_same_v<T, raybos::LensElement>) {
            r.kind = RB_ELEM_SINGLET;
            r.front = surf(x.front);
            r.back = surf(x.back);
            r.diameter = x.diameter;
          } else if constexpr (std::is_same_v<T, raybos::ThinLensIdeal>) {
            r.kind = RB_ELEM_THIN_LENS;
            r.center = v3(x.center);
            r.axis = v3(x.axis);
            r.focal_length = x.focal_length;
            r.diameter = x.diameter;
          } else {
            r.kind = RB_ELEM_MIRROR;
            r.front = surf(x.surface);
          }
        },
        e);
    f.elements.push_back(r);
  }
  rb_scene& s = f.s;
  s = rb_scene{};
  s.sources = f.sources.data();
  s.n_sources = static_cast<int64_t>(f.sources.size());
  s.pupil_center = v3(setup.pupil.center);
  s.pupil_axis = v3(setup.pupil.axis);
  s.pupil_radius = setup.pupil.radius;
  s.rays_per_source = setup.bundle.rays_per_source;
  s.sampling = setup.bundle.sampling == raybos::ApertureSampling::kStratified
                   ? RB_SAMPLING_STRATIFIED
                   : RB_SAMPLING_UNIFORM;
  s.seed = setup.bundle.seed;
  s.wavelength = setup.wavelength;
  s.delta_xi = setup.step.delta_xi;
  s.max_steps = setup.step.max_steps;
  s.n_elements = static_cast<int32_t>(f.elements.size());
  s.elements = f.elements.data();
  s.sensor.center = v3(setup.sensor.center);
  s.sensor.normal = v3(setup.sensor.normal);
  s.sensor.e_u = v3(setup.sensor.e_u);
  s.sensor.e_v = v3(setup.sensor.e_v);
  s.sensor.width_px = setup.sensor.width_px;
  s.sensor.height_px = setup.sensor.height_px;
  s.sensor.pitch = setup.sensor.pitch;
  s.sensor.window_sigmas = setup.sensor.window_sigmas;
  s.d_tau = setup.d_tau;
  s.config_hash = setup.config_hash;
}

// rb_trace_out -> TraceOutputs / RunReport (engine.hpp:19-36, 67-71).
inline void unflatten(const rb_trace_out& o, const std::vector<double>& hit,
                      const std::vector<int64_t>& landed, raybos::TraceOutputs& out) {
  out.stats.resize(landed.size());
  for (size_t d = 0; d < landed.size(); ++d) {
    out.stats[d].hit_sum = {hit[2 * d], hit[2 * d + 1]};
    out.stats[d].landed = static_cast<long>(landed[d]);
  }
  raybos::RunReport& r = out.report;
  r.emitted = static_cast<long>(o.emitted);
  r.landed = static_cast<long>(o.landed_total);
  r.lost = static_cast<long>(o.lost);
  r.blocked_aperture = static_cast<long>(o.blocked_aperture);
  r.blocked_miss = static_cast<long>(o.blocked_miss);
  r.blocked_tir = static_cast<long>(o.blocked_tir);
  r.blocked_sensor_miss = static_cast<long>(o.blocked_sensor_miss);
  r.wall_seconds = o.wall_seconds;
  r.threads = o.threads;
  r.config_hash = o.config_hash;
}

}  // namespace detail

// The reference's run_trace contract on B200 (engine.hpp:73-78).
inline raybos::TraceOutputs run_trace(const raybos::SceneSetup& setup, bool with_field,
                                      bool accumulate_image, const raybos::RunConfig& run) {
  (void)run;  // threads / deterministic: see header comment
  detail::Context& C = detail::context();
  std::lock_guard<std::mutex> lock(C.mu);
  if (with_field && setup.field) C.ensure_field(setup.field);
  const bool field = with_field && (setup.field || C.external);
  detail::FlatScene f;
  detail::flatten(setup, f);
  raybos::TraceOutputs out;
  std::vector<double> hit(2 * setup.sources.size());
  std::vector<int64_t> landed(setup.sources.size());
  if (accumulate_image) out.image = raybos::ImageBuffer(setup.sensor.width_px, setup.sensor.height_px);
  rb_trace_out o{};
  o.hit_sum = hit.data();
  o.landed = landed.data();
  o.image = accumulate_image ? out.image.data.data() : nullptr;
  const int rc = rb_trace(C.ctx, &f.s, field ? 1 : 0, accumulate_image ? 1 : 0, &o);
  if (rc) detail::raise(rc, rb_last_error(C.ctx));
  detail::unflatten(o, hit, landed, out);
  return out;
}

// The config's GVOL medium streamed straight to the devices (rb_set_field_gvol),
// recentred like build_medium_volume (engine.cpp:27-37), for volumes whose host
// GriddedField would not fit (1024^3: 34 GB).  Build `setup` with
// build_scene_setup from a copy of the config with medium.type = "none"; this
// then fills in what build_scene_setup derives from the volume (step size,
// max_steps and the BOS depth, engine.cpp:237-252), and run_trace(setup, true,
// ...) traces through the streamed grid while setup.field stays empty.
inline void load_medium_gvol(const raybos::ExperimentConfig& cfg, raybos::SceneSetup& setup) {
  if (cfg.medium.type != "gvol") throw std::runtime_error("raybos_gpu: medium is not gvol");
  detail::Context& C = detail::context();
  std::lock_guard<std::mutex> lock(C.mu);
  C.field.reset();
  C.has_field = false;
  C.external = false;
  const double zc = cfg.geometry.z_dot_to_volume;
  rb_field_desc d{};
  const int rc = rb_set_field_gvol(C.ctx, cfg.medium.path.c_str(), &zc, cfg.gladstone_dale, 0, &d);
  if (rc) detail::raise(rc, rb_last_error(C.ctx));
  C.external = true;
  const raybos::Vec3 sp{d.spacing.x, d.spacing.y, d.spacing.z};
  const raybos::Vec3 lo{d.origin.x, d.origin.y, d.origin.z};
  const raybos::Vec3 hi = lo + raybos::Vec3{(d.nx - 1) * sp.x, (d.ny - 1) * sp.y, (d.nz - 1) * sp.z};
  setup.bos_params.depth = (d.nz - 1) * sp.z;
  setup.step.delta_xi =
      cfg.trace.delta_xi > 0.0 ? cfg.trace.delta_xi : 0.5 * std::min({sp.x, sp.y, sp.z});
  if (cfg.trace.max_steps > 0)
    setup.step.max_steps = cfg.trace.max_steps;
  else
    setup.step.max_steps = static_cast<int>(4.0 * raybos::norm(hi - lo) / setup.step.delta_xi) + 64;
}

// bos_run's two traces (engine.cpp:539-540, write_images off) in one fused
// pass: {run_trace(setup, false, false, run), run_trace(setup, true, false, run)},
// bit-identical to the two separate calls.
inline std::pair<raybos::TraceOutputs, raybos::TraceOutputs> run_trace_bos_pair(
    const raybos::SceneSetup& setup, const raybos::RunConfig& run) {
  (void)run;
  if (!setup.field) throw std::runtime_error("bos_run: config must include a density field");
  detail::Context& C = detail::context();
  std::lock_guard<std::mutex> lock(C.mu);
  C.ensure_field(setup.field);
  detail::FlatScene f;
  detail::flatten(setup, f);
  const size_t n = setup.sources.size();
  std::vector<double> h0(2 * n), h1(2 * n);
  std::vector<int64_t> l0(n), l1(n);
  rb_trace_out o0{}, o1{};
  o0.hit_sum = h0.data();
  o0.landed = l0.data();
  o1.hit_sum = h1.data();
  o1.landed = l1.data();
  const int rc = rb_trace_bos_pair(C.ctx, &f.s, &o0, &o1);
  if (rc) detail::raise(rc, rb_last_error(C.ctx));
  std::pair<raybos::TraceOutputs, raybos::TraceOutputs> out;
  detail::unflatten(o0, h0, l0, out.first);
  detail::unflatten(o1, h1, l1, out.second);
  return out;
}

}  // namespace raybos_gpu
