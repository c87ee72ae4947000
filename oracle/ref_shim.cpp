// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  Never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python test-suite and bench.py's cpu_baseline leg
//   * build a reference SceneSetup from a config (parse_config_json +
//     build_scene_setup, engine.cpp:228-427) or from the reference's canonical
//     validation configs (validate.cpp:344-415),
//   * export it as the flat rb_scene of include/raybos_gpu.h, so the GPU path
//     renders exactly the scene the reference renders,
//   * run the reference run_trace (engine.cpp:429-507) and
//   * replay process_source per ray (engine.cpp:107-140) through the public API
//     (sample_aperture_points -> emit_rays -> trace_through_volume ->
//     propagate_chain -> intersect_sensor).
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <type_traits>
#include <variant>
#include <vector>

#include "raybos/engine.hpp"
#include "raybos/raygen.hpp"
#include "raybos/scene.hpp"
#include "raybos/validate.hpp"
#include "raybos_gpu.h"

namespace {

struct Handle {
  raybos::ExperimentConfig cfg;
  raybos::SceneSetup setup;
  std::vector<rb_vec3> sources;
  std::vector<rb_element> elements;
};

void set_err(char* err, size_t len, const std::string& msg) {
  if (err && len) {
    std::strncpy(err, msg.c_str(), len - 1);
    err[len - 1] = '\0';
  }
}

rb_vec3 v3(const raybos::Vec3& v) { return {v.x, v.y, v.z}; }
raybos::Vec3 v3(const rb_vec3& v) { return {v.x, v.y, v.z}; }

rb_surface surf(const raybos::SphericalSurface& s) {
  return {v3(s.vertex), v3(s.axis), s.curvature_radius, s.aperture_radius, s.n_before, s.n_after};
}

raybos::ExperimentConfig small_config() {  // test_engine.cpp:21-31
  raybos::ExperimentConfig cfg = raybos::make_bos_uniform_config();
  cfg.source.count = 12;
  cfg.source.extent = {0.008, 0.008};
  cfg.bundle.rays_per_source = 400;
  cfg.sensor.width = cfg.sensor.height = 96;
  cfg.bos.grid_nx = cfg.bos.grid_ny = 4;
  cfg.bos.grid_extent = {0.006, 0.006};
  cfg.bos.min_dots = 4;
  return cfg;
}

void refresh_flat(Handle& h) {
  h.sources.clear();
  for (const auto& s : h.setup.sources) h.sources.push_back(v3(s));
  h.elements.clear();
  for (const auto& e : h.setup.elements) {
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
          } else if constexpr (std::is_same_v<T, raybos::Mirror>) {
            r.kind = RB_ELEM_MIRROR;
            r.front = surf(x.surface);
          }
        },
        e);
    h.elements.push_back(r);
  }
}

template <typename F>
int guarded(char* err, size_t len, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    set_err(err, len, e.what());
    return RB_E_INVALID;
  } catch (const std::exception& e) {
    set_err(err, len, e.what());
    return RB_E_RUNTIME;
  }
}

}  // namespace

extern "C" {

// Scalar results of build_scene_setup that are not part of rb_scene.
typedef struct refshim_info {
  double lens_plane_z, focal_length, f_number, magnification, gain, ambient_index,
      volume_center_z, d_tau;
  int32_t bit_depth, has_field;
  uint64_t config_hash;
} refshim_info;

int refshim_create_json(const char* json, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto h = std::make_unique<Handle>();
    h->cfg = raybos::parse_config_json(json);
    h->setup = raybos::build_scene_setup(h->cfg);
    refresh_flat(*h);
    *out = h.release();
  });
}

int refshim_create_builtin(const char* name, void** out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    auto h = std::make_unique<Handle>();
    const std::string n(name);
    if (n == "bos_uniform")
      h->cfg = raybos::make_bos_uniform_config();
    else if (n == "bos_blob")
      h->cfg = raybos::make_bos_blob_config();
    else if (n == "null_test")
      h->cfg = raybos::make_null_test_config();
    else if (n == "determinism")
      h->cfg = raybos::make_determinism_config();
    else if (n == "small")
      h->cfg = small_config();
    else
      throw std::runtime_error("refshim: unknown builtin config '" + n + "'");
    h->setup = raybos::build_scene_setup(h->cfg);
    refresh_flat(*h);
    *out = h.release();
  });
}

void refshim_destroy(void* h) { delete static_cast<Handle*>(h); }

void refshim_export_scene(void* hv, rb_scene* s) {
  Handle& h = *static_cast<Handle*>(hv);
  const raybos::SceneSetup& st = h.setup;
  std::memset(s, 0, sizeof(*s));
  s->sources = h.sources.data();
  s->n_sources = static_cast<int64_t>(h.sources.size());
  s->source_ids = nullptr;
  s->pupil_center = v3(st.pupil.center);
  s->pupil_axis = v3(st.pupil.axis);
  s->pupil_radius = st.pupil.radius;
  s->rays_per_source = st.bundle.rays_per_source;
  s->sampling = st.bundle.sampling == raybos::ApertureSampling::kStratified
                    ? RB_SAMPLING_STRATIFIED
                    : RB_SAMPLING_UNIFORM;
  s->seed = st.bundle.seed;
  s->wavelength = st.wavelength;
  s->delta_xi = st.step.delta_xi;
  s->max_steps = st.step.max_steps;
  s->n_elements = static_cast<int32_t>(h.elements.size());
  s->elements = h.elements.data();
  s->sensor.center = v3(st.sensor.center);
  s->sensor.normal = v3(st.sensor.normal);
  s->sensor.e_u = v3(st.sensor.e_u);
  s->sensor.e_v = v3(st.sensor.e_v);
  s->sensor.width_px = st.sensor.width_px;
  s->sensor.height_px = st.sensor.height_px;
  s->sensor.pitch = st.sensor.pitch;
  s->sensor.window_sigmas = st.sensor.window_sigmas;
  s->d_tau = st.d_tau;
  s->config_hash = st.config_hash;
}

void refshim_info_get(void* hv, refshim_info* o) {
  const raybos::SceneSetup& st = static_cast<Handle*>(hv)->setup;
  o->lens_plane_z = st.lens_plane_z;
  o->focal_length = st.focal_length;
  o->f_number = st.f_number;
  o->magnification = st.magnification;
  o->gain = st.sensor.gain;
  o->ambient_index = st.ambient_index;
  o->volume_center_z = st.volume_center_z;
  o->d_tau = st.d_tau;
  o->bit_depth = st.sensor.bit_depth;
  o->has_field = st.field ? 1 : 0;
  o->config_hash = st.config_hash;
}

// Returns 1 and fills desc when the scene has a GriddedField, else 0.
int refshim_field_desc(void* hv, rb_field_desc* d) {
  const auto& f = static_cast<Handle*>(hv)->setup.field;
  if (!f) return 0;
  std::memset(d, 0, sizeof(*d));
  d->nx = f->nx();
  d->ny = f->ny();
  d->nz = f->nz();
  d->origin = v3(f->origin());
  d->spacing = v3(f->spacing());
  return 1;
}

// Copies GriddedField's node values (scene.hpp:88-92), x-fastest.
void refshim_field_nodes(void* hv, double* n, double* gx, double* gy, double* gz) {
  const auto& f = *static_cast<Handle*>(hv)->setup.field;
  size_t q = 0;
  for (int k = 0; k < f.nz(); ++k)
    for (int j = 0; j < f.ny(); ++j)
      for (int i = 0; i < f.nx(); ++i, ++q) {
        n[q] = f.node_n(i, j, k);
        const raybos::Vec3 g = f.node_grad(i, j, k);
        gx[q] = g.x;
        gy[q] = g.y;
        gz[q] = g.z;
      }
}

// Replaces the scene's field by GriddedField(volume, K) built from rho.
int refshim_set_field_density(void* hv, const rb_field_desc* d, const float* rho, double k,
                              char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    raybos::DensityVolume vol;
    vol.nx = d->nx;
    vol.ny = d->ny;
    vol.nz = d->nz;
    vol.spacing = v3(d->spacing);
    vol.origin = v3(d->origin);
    vol.rho.assign(rho, rho + static_cast<size_t>(d->nx) * d->ny * d->nz);
    static_cast<Handle*>(hv)->setup.field = std::make_shared<raybos::GriddedField>(vol, k);
  });
}

void refshim_clear_field(void* hv) { static_cast<Handle*>(hv)->setup.field.reset(); }

void refshim_set_step(void* hv, double delta_xi, int32_t max_steps) {
  auto& st = static_cast<Handle*>(hv)->setup.step;
  st.delta_xi = delta_xi;
  st.max_steps = max_steps;
}

void refshim_set_sources(void* hv, const rb_vec3* src, int64_t n) {
  Handle& h = *static_cast<Handle*>(hv);
  h.setup.sources.clear();
  for (int64_t i = 0; i < n; ++i) h.setup.sources.push_back(v3(src[i]));
  h.setup.dot_positions.clear();
  refresh_flat(h);
}

void refshim_set_bundle(void* hv, int32_t rays, int32_t sampling, uint64_t seed) {
  auto& b = static_cast<Handle*>(hv)->setup.bundle;
  b.rays_per_source = rays;
  b.sampling = sampling == RB_SAMPLING_STRATIFIED ? raybos::ApertureSampling::kStratified
                                                  : raybos::ApertureSampling::kUniformRandom;
  b.seed = seed;
}

// Replaces the whole optics/sensor/pupil part of the setup from a flat scene
// (used to run the reference on synthetic bench scenes).
void refshim_set_flat(void* hv, const rb_scene* s) {
  Handle& h = *static_cast<Handle*>(hv);
  raybos::SceneSetup& st = h.setup;
  st.sources.clear();
  for (int64_t i = 0; i < s->n_sources; ++i) st.sources.push_back(v3(s->sources[i]));
  st.pupil = {v3(s->pupil_center), v3(s->pupil_axis), s->pupil_radius};
  st.bundle.rays_per_source = s->rays_per_source;
  st.bundle.sampling = s->sampling == RB_SAMPLING_STRATIFIED
                           ? raybos::ApertureSampling::kStratified
                           : raybos::ApertureSampling::kUniformRandom;
  st.bundle.seed = s->seed;
  st.wavelength = s->wavelength;
  st.step.delta_xi = s->delta_xi;
  st.step.max_steps = s->max_steps;
  st.elements.clear();
  auto to_surf = [](const rb_surface& r) {
    raybos::SphericalSurface x;
    x.vertex = v3(r.vertex);
    x.axis = v3(r.axis);
    x.curvature_radius = r.curvature_radius;
    x.aperture_radius = r.aperture_radius;
    x.n_before = r.n_before;
    x.n_after = r.n_after;
    return x;
  };
  for (int32_t e = 0; e < s->n_elements; ++e) {
    const rb_element& r = s->elements[e];
    if (r.kind == RB_ELEM_APERTURE) {
      st.elements.push_back(raybos::Aperture{v3(r.center), v3(r.axis), r.radius});
    } else if (r.kind == RB_ELEM_THIN_LENS) {
      st.elements.push_back(
          raybos::ThinLensIdeal{v3(r.center), v3(r.axis), r.focal_length, r.diameter});
    } else if (r.kind == RB_ELEM_SINGLET) {
      raybos::LensElement l;
      l.front = to_surf(r.front);
      l.back = to_surf(r.back);
      l.diameter = r.diameter;
      st.elements.push_back(l);
    } else {
      st.elements.push_back(raybos::Mirror{to_surf(r.front)});
    }
  }
  st.sensor.center = v3(s->sensor.center);
  st.sensor.normal = v3(s->sensor.normal);
  st.sensor.e_u = v3(s->sensor.e_u);
  st.sensor.e_v = v3(s->sensor.e_v);
  st.sensor.width_px = s->sensor.width_px;
  st.sensor.height_px = s->sensor.height_px;
  st.sensor.pitch = s->sensor.pitch;
  st.sensor.window_sigmas = s->sensor.window_sigmas;
  st.d_tau = s->d_tau;
  st.config_hash = s->config_hash;
  refresh_flat(h);
}

// The reference run_trace.  out->image must hold W*H doubles when
// accumulate_image is set.
int refshim_run_trace(void* hv, int with_field, int accumulate_image, int threads,
                      int deterministic, rb_trace_out* out, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const Handle& h = *static_cast<Handle*>(hv);
    raybos::RunConfig run;
    run.threads = threads;
    run.deterministic = deterministic != 0;
    const raybos::TraceOutputs t =
        raybos::run_trace(h.setup, with_field != 0, accumulate_image != 0, run);
    for (size_t d = 0; d < t.stats.size(); ++d) {
      if (out->hit_sum) {
        out->hit_sum[2 * d] = t.stats[d].hit_sum.x;
        out->hit_sum[2 * d + 1] = t.stats[d].hit_sum.y;
      }
      if (out->landed) out->landed[d] = t.stats[d].landed;
    }
    if (accumulate_image && out->image)
      std::memcpy(out->image, t.image.data.data(), t.image.data.size() * sizeof(double));
    out->emitted = t.report.emitted;
    out->landed_total = t.report.landed;
    out->lost = t.report.lost;
    out->blocked_aperture = t.report.blocked_aperture;
    out->blocked_miss = t.report.blocked_miss;
    out->blocked_tir = t.report.blocked_tir;
    out->blocked_sensor_miss = t.report.blocked_sensor_miss;
    out->wall_seconds = t.report.wall_seconds;
    out->threads = t.report.threads;
    out->config_hash = t.report.config_hash;
    out->total_steps = -1;
    out->kernel_ms = 0.0;
  });
}

// Per-ray replay of process_source (engine.cpp:107-140) with the public API.
// exit_state (optional, 6 doubles per ray): origin and dir of the ray after
// the volume (or the emitted ray when it missed / with_field == 0).
int refshim_trace_rays(void* hv, int with_field, int64_t n, const int64_t* src,
                       const int32_t* ray, double* uv, int32_t* status, int32_t* steps,
                       double* exit_state, char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const raybos::SceneSetup& st = static_cast<Handle*>(hv)->setup;
    int64_t cached = -1;
    std::vector<raybos::Ray> rays;
    for (int64_t q = 0; q < n; ++q) {
      if (src[q] != cached) {
        const auto pts = raybos::sample_aperture_points(st.pupil, st.bundle,
                                                        static_cast<std::uint64_t>(src[q]));
        rays = raybos::emit_rays(st.sources[src[q]], pts, st.wavelength);
        cached = src[q];
      }
      raybos::Ray r = rays[ray[q]];
      uv[2 * q] = uv[2 * q + 1] = std::nan("");
      steps[q] = 0;
      if (with_field && st.field) {
        const raybos::TraceResult tr = raybos::trace_through_volume(r, *st.field, st.step);
        steps[q] = tr.steps;
        if (!tr.ok()) {
          status[q] = RB_RAY_LOST;
          continue;
        }
        r = tr.ray;
      }
      if (exit_state) {
        exit_state[6 * q + 0] = r.origin.x;
        exit_state[6 * q + 1] = r.origin.y;
        exit_state[6 * q + 2] = r.origin.z;
        exit_state[6 * q + 3] = r.dir.x;
        exit_state[6 * q + 4] = r.dir.y;
        exit_state[6 * q + 5] = r.dir.z;
      }
      const raybos::OpticsResult o = raybos::propagate_chain(r, st.elements);
      if (!o.ok()) {
        switch (o.reason) {
          case raybos::BlockReason::kApertureStop: status[q] = RB_RAY_APERTURE; break;
          case raybos::BlockReason::kTotalInternalReflection: status[q] = RB_RAY_TIR; break;
          default: status[q] = RB_RAY_MISSED; break;
        }
        continue;
      }
      const auto hit = raybos::intersect_sensor(o.ray, st.sensor);
      if (!hit) {
        status[q] = RB_RAY_SENSOR_MISS;
        continue;
      }
      status[q] = RB_RAY_LANDED;
      uv[2 * q] = hit->x;
      uv[2 * q + 1] = hit->y;
    }
  });
}

// trace_debug's records (engine.cpp:605-624) for (dot, ray) via the public
// API: sample_aperture_points -> emit_rays -> trace_through_volume with a
// StepObserver.  Writes up to cap records of 7 doubles; returns the count.
int64_t refshim_trace_debug(void* hv, int64_t dot, int32_t ray, double* rec, int64_t cap) {
  const raybos::SceneSetup& st = static_cast<Handle*>(hv)->setup;
  const auto pts = raybos::sample_aperture_points(st.pupil, st.bundle, static_cast<std::uint64_t>(dot));
  const auto rays = raybos::emit_rays(st.sources[dot], pts, st.wavelength);
  int64_t n = 0;
  raybos::StepObserver obs = [&](double xi, const raybos::RayState& s) {
    if (n < cap) {
      double* q = rec + 7 * n;
      q[0] = xi;
      q[1] = s.r.x;
      q[2] = s.r.y;
      q[3] = s.r.z;
      q[4] = s.t.x;
      q[5] = s.t.y;
      q[6] = s.t.z;
    }
    ++n;
  };
  raybos::trace_through_volume(rays[ray], *st.field, st.step, &obs);
  return n;
}

// quantize (sensor.cpp:124-135), for PGM byte-compatibility checks.
int refshim_quantize(const double* img, int64_t n, int bit_depth, double gain, uint16_t* out,
                     char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    raybos::ImageBuffer b;
    b.width = static_cast<int>(n);
    b.height = 1;
    b.data.assign(img, img + n);
    const auto q = raybos::quantize(b, bit_depth, gain);
    std::memcpy(out, q.data(), q.size() * sizeof(uint16_t));
  });
}

// bos post-processing on the per-dot stats of two traces (bos.cpp:97-112 +
// 114-201 + 203-244), so BOS metrics can be compared end to end.
int refshim_bos_metrics(void* hv, const double* ref_hit, const int64_t* ref_landed,
                        const double* grad_hit, const int64_t* grad_landed, double* metrics6,
                        char* err, size_t errlen) {
  return guarded(err, errlen, [&] {
    const Handle& h = *static_cast<Handle*>(hv);
    const raybos::SceneSetup& st = h.setup;
    const size_t nd = st.dot_positions.size();
    std::vector<raybos::DotHitStats> a(nd), b(nd);
    for (size_t d = 0; d < nd; ++d) {
      a[d].hit_sum = {ref_hit[2 * d], ref_hit[2 * d + 1]};
      a[d].landed = ref_landed[d];
      b[d].hit_sum = {grad_hit[2 * d], grad_hit[2 * d + 1]};
      b[d].landed = grad_landed[d];
    }
    const double shrink = 1.0 - st.volume_center_z / st.pupil.center.z;
    std::vector<raybos::Vec2> attach(nd);
    for (size_t d = 0; d < nd; ++d) attach[d] = st.dot_positions[d] * shrink;
    const auto scattered = raybos::measure_dot_displacements(attach, a, b);
    raybos::DisplacementField measured = raybos::grid_displacements(scattered, st.grid);
    const raybos::GriddedField& field = *st.field;
    raybos::GradientSlice slice;
    slice.nx = field.nx();
    slice.ny = field.ny();
    slice.x0 = field.origin().x;
    slice.y0 = field.origin().y;
    slice.dx = field.spacing().x;
    slice.dy = field.spacing().y;
    slice.grad.resize(static_cast<size_t>(slice.nx) * slice.ny);
    for (int j = 0; j < slice.ny; ++j)
      for (int i = 0; i < slice.nx; ++i) {
        raybos::Vec2 g{};
        for (int k = 0; k < field.nz(); ++k) {
          const raybos::Vec3 gn = field.node_grad(i, j, k);
          g += raybos::Vec2{gn.x, gn.y};
        }
        slice.grad[slice.index(i, j)] = g / (field.nz() * h.cfg.gladstone_dale);
      }
    raybos::DisplacementField theory =
        raybos::theoretical_displacement(slice, st.bos_params, st.grid);
    const double s = h.cfg.bos.units == "px" ? 1.0 / st.sensor.pitch : 1.0;
    for (auto& d : measured.delta) d = d * s;
    for (auto& d : theory.delta) d = d * s;
    const raybos::FieldMetrics m = raybos::compare_fields(theory, measured);
    metrics6[0] = m.rms_error;
    metrics6[1] = m.peak_abs_error;
    metrics6[2] = m.pearson_correlation;
    metrics6[3] = m.peak_a;
    metrics6[4] = m.peak_b;
    metrics6[5] = m.nodes;
  });
}

}  // extern "C"
