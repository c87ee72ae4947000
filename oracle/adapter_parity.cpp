// adapter_parity.cpp — TEST INFRASTRUCTURE ONLY (built into oracle/_ref/ by
// oracle/Makefile against the reference's own headers and library).
//
// Drives the C++ drop-in raybos_gpu::run_trace (include/raybos_gpu/run_trace.hpp)
// exactly where the reference calls raybos::run_trace: on SceneSetups built by
// the reference's build_scene_setup for its canonical configs
// (validate.cpp:344-415), and through the bos_run post-processing chain
// (engine.cpp:532-603: measure_dot_displacements -> grid_displacements ->
// theoretical_displacement -> compare_fields).  Prints one JSON line per
// check; exit status 0 iff every check is within the north-star tolerances.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "raybos/bos.hpp"
#include "raybos/engine.hpp"
#include "raybos/scene.hpp"
#include "raybos/sensor.hpp"
#include "raybos/validate.hpp"
#include "raybos_gpu/run_trace.hpp"

using namespace raybos;

namespace {

int failures = 0;

void check(const std::string& what, bool ok, const std::string& detail) {
  std::printf("{\"check\": \"%s\", \"ok\": %s, %s}\n", what.c_str(), ok ? "true" : "false",
              detail.c_str());
  std::fflush(stdout);
  failures += ok ? 0 : 1;
}

std::string num(const char* k, double v) {
  char b[128];
  std::snprintf(b, sizeof(b), "\"%s\": %.6g", k, v);
  return b;
}

void compare_traces(const std::string& name, const SceneSetup& setup, bool with_field,
                    const SceneSetup* gpu_setup = nullptr) {
  RunConfig run;
  run.threads = 0;
  const TraceOutputs ref = raybos::run_trace(setup, with_field, true, run);
  const TraceOutputs gpu = raybos_gpu::run_trace(gpu_setup ? *gpu_setup : setup, with_field, true, run);
  const RunReport& a = ref.report;
  const RunReport& b = gpu.report;
  const bool counters = a.emitted == b.emitted && a.landed == b.landed && a.lost == b.lost &&
                        a.blocked_aperture == b.blocked_aperture &&
                        a.blocked_miss == b.blocked_miss && a.blocked_tir == b.blocked_tir &&
                        a.blocked_sensor_miss == b.blocked_sensor_miss;
  double max_px = 0.0;
  bool landed_eq = ref.stats.size() == gpu.stats.size();
  for (size_t d = 0; landed_eq && d < ref.stats.size(); ++d) {
    landed_eq = ref.stats[d].landed == gpu.stats[d].landed;
    if (ref.stats[d].landed == 0) continue;
    const Vec2 ma = ref.stats[d].hit_sum / static_cast<double>(ref.stats[d].landed);
    const Vec2 mb = gpu.stats[d].hit_sum / static_cast<double>(gpu.stats[d].landed);
    max_px = std::max(max_px, norm(ma - mb) / setup.sensor.pitch);
  }
  double num2 = 0.0, den2 = 0.0;
  for (size_t q = 0; q < ref.image.data.size(); ++q) {
    const double d = gpu.image.data[q] - ref.image.data[q];
    num2 += d * d;
    den2 += ref.image.data[q] * ref.image.data[q];
  }
  const double rel = den2 > 0 ? std::sqrt(num2 / den2) : std::sqrt(num2);
  // PGM bytes (render, engine.cpp:513-528): quantize both images with the gain
  const auto qa = quantize(ref.image, setup.sensor.bit_depth, setup.sensor.gain);
  const auto qb = quantize(gpu.image, setup.sensor.bit_depth, setup.sensor.gain);
  long diff = 0, maxd = 0;
  for (size_t q = 0; q < qa.size(); ++q) {
    const long d = std::labs(static_cast<long>(qa[q]) - static_cast<long>(qb[q]));
    diff += d != 0;
    maxd = std::max(maxd, d);
  }
  // north-star gates: counts exact, per-dot means within 1e-3 px, image within 1e-4
  // relative L2 (the quantized PGM difference is reported, not gated)
  const bool ok = counters && landed_eq && max_px < 1e-3 && rel < 1e-4 && b.accounting_ok();
  check(name + (with_field ? "/field" : "/nofield"), ok,
        num("emitted", a.emitted) + ", " + num("counters_equal", counters) + ", " +
            num("landed_equal", landed_eq) + ", " + num("max_mean_hit_px", max_px) + ", " +
            num("image_rel_l2", rel) + ", " + num("pgm_pixels_differing", diff) + ", " +
            num("pgm_max_count_diff", maxd) + ", " + num("gpu_threads", b.threads));
}

// bos_run's metric chain (engine.cpp:542-597) on reference vs drop-in stats.
void compare_bos(const std::string& name, const ExperimentConfig& cfg) {
  const SceneSetup setup = build_scene_setup(cfg);
  RunConfig run;
  FieldMetrics m[2];
  for (int impl = 0; impl < 2; ++impl) {
    // impl 1: the fused drop-in (one pass, both legs)
    std::pair<TraceOutputs, TraceOutputs> legs;
    if (impl)
      legs = raybos_gpu::run_trace_bos_pair(setup, run);
    else
      legs = {raybos::run_trace(setup, false, false, run), raybos::run_trace(setup, true, false, run)};
    const TraceOutputs& r0 = legs.first;
    const TraceOutputs& r1 = legs.second;
    const double shrink = 1.0 - setup.volume_center_z / setup.pupil.center.z;
    std::vector<Vec2> attach(setup.dot_positions.size());
    for (size_t d = 0; d < attach.size(); ++d) attach[d] = setup.dot_positions[d] * shrink;
    const auto sc = measure_dot_displacements(attach, r0.stats, r1.stats);
    DisplacementField meas = grid_displacements(sc, setup.grid);
    const GriddedField& f = *setup.field;
    GradientSlice slice;
    slice.nx = f.nx();
    slice.ny = f.ny();
    slice.x0 = f.origin().x;
    slice.y0 = f.origin().y;
    slice.dx = f.spacing().x;
    slice.dy = f.spacing().y;
    slice.grad.resize(static_cast<size_t>(slice.nx) * slice.ny);
    for (int j = 0; j < slice.ny; ++j)
      for (int i = 0; i < slice.nx; ++i) {
        Vec2 g{};
        for (int k = 0; k < f.nz(); ++k) {
          const Vec3 gn = f.node_grad(i, j, k);
          g += Vec2{gn.x, gn.y};
        }
        slice.grad[slice.index(i, j)] = g / (f.nz() * cfg.gladstone_dale);
      }
    DisplacementField th = theoretical_displacement(slice, setup.bos_params, setup.grid);
    for (auto& d : meas.delta) d = d * (1.0 / setup.sensor.pitch);
    for (auto& d : th.delta) d = d * (1.0 / setup.sensor.pitch);
    m[impl] = compare_fields(th, meas);
  }
  auto rel = [](double x, double y) { return std::abs(x - y) / std::max(std::abs(y), 1e-30); };
  // measured-vs-theory metrics, per the reference's own bos-* criteria; the drop-in
  // must reproduce them (same node mask, values to 1e-3 relative)
  const bool ok = m[0].nodes == m[1].nodes && rel(m[1].rms_error, m[0].rms_error) < 1e-3 &&
                  rel(m[1].peak_abs_error, m[0].peak_abs_error) < 1e-3 &&
                  rel(m[1].pearson_correlation, m[0].pearson_correlation) < 1e-3 &&
                  rel(m[1].peak_b, m[0].peak_b) < 1e-3;
  check(name + "/bos_metrics", ok,
        num("nodes_ref", m[0].nodes) + ", " + num("nodes_gpu", m[1].nodes) + ", " +
            num("rms_ref_px", m[0].rms_error) + ", " + num("rms_gpu_px", m[1].rms_error) + ", " +
            num("pearson_ref", m[0].pearson_correlation) + ", " +
            num("pearson_gpu", m[1].pearson_correlation) + ", " +
            num("peak_measured_ref_px", m[0].peak_b) + ", " +
            num("peak_measured_gpu_px", m[1].peak_b));
}

}  // namespace

int main() {
  struct Named {
    const char* name;
    ExperimentConfig cfg;
  };
  ExperimentConfig small = make_bos_uniform_config();  // test_engine.cpp:21-31
  small.source.count = 12;
  small.source.extent = {0.008, 0.008};
  small.bundle.rays_per_source = 400;
  small.sensor.width = small.sensor.height = 96;
  small.bos.grid_nx = small.bos.grid_ny = 4;
  small.bos.grid_extent = {0.006, 0.006};
  const std::vector<Named> configs = {
      {"small", small},
      {"null_test", make_null_test_config()},
      {"determinism", make_determinism_config()},
      {"bos_uniform", make_bos_uniform_config()},
      {"bos_blob", make_bos_blob_config()},
  };
  for (const Named& c : configs) {
    const SceneSetup setup = build_scene_setup(c.cfg);
    compare_traces(c.name, setup, true);
    if (std::string(c.name) == "small" || std::string(c.name) == "determinism")
      compare_traces(c.name, setup, false);
  }
  {  // GVOL medium: the reference loads it into a host GriddedField; the drop-in
     // streams the file to the GPU (load_medium_gvol) and never builds one
    DensityVolume vol;
    vol.nx = 40;
    vol.ny = 36;
    vol.nz = 24;
    vol.spacing = {4e-4, 4.5e-4, 5e-4};
    vol.origin = {0.003, -0.002, 0.1};  // recentred by build_medium_volume
    vol.rho.resize(static_cast<size_t>(vol.nx) * vol.ny * vol.nz);
    for (int k = 0; k < vol.nz; ++k)
      for (int j = 0; j < vol.ny; ++j)
        for (int i = 0; i < vol.nx; ++i) {
          const double x = (i - 17.0) / 7.0, y = (j - 19.0) / 6.0, z = (k - 11.0) / 5.0;
          vol.rho[vol.index(i, j, k)] = static_cast<float>(1.2 + 3.0 * std::exp(-(x * x + y * y + z * z)));
        }
    const std::string path = "/tmp/raybos_adapter_parity.gvol";
    save_density_volume(vol, path);
    ExperimentConfig cfg = make_bos_blob_config();
    cfg.medium.type = "gvol";
    cfg.medium.path = path;
    const SceneSetup ref_setup = build_scene_setup(cfg);
    ExperimentConfig none = cfg;
    none.medium.type = "none";
    SceneSetup gpu_setup = build_scene_setup(none);
    raybos_gpu::load_medium_gvol(cfg, gpu_setup);
    const bool same = gpu_setup.step.delta_xi == ref_setup.step.delta_xi &&
                      gpu_setup.step.max_steps == ref_setup.step.max_steps &&
                      gpu_setup.bos_params.depth == ref_setup.bos_params.depth && !gpu_setup.field;
    check("gvol_stream/setup", same,
          num("delta_xi", gpu_setup.step.delta_xi) + ", " + num("max_steps", gpu_setup.step.max_steps));
    compare_traces("gvol_stream", ref_setup, true, &gpu_setup);
    std::remove(path.c_str());
  }
  compare_bos("bos_uniform", make_bos_uniform_config());
  compare_bos("bos_blob", make_bos_blob_config());
  std::printf("{\"failures\": %d}\n", failures);
  return failures == 0 ? 0 : 1;
}
