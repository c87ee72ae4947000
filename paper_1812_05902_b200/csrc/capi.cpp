// capi.cpp — host side of the C-ABI (include/raybos_gpu.h).
//
// The B200 replacement for run_trace's driver (reference
// proj/src/engine.cpp:429-507): instead of a std::thread pool over contiguous
// source ranges with private tiles composited in source order, the sources are
// ordered along a Z-order curve (so concurrently resident CTAs trace
// neighbouring cones through the same part of the grid), dealt to GPUs in
// interleaved tiles, rendered by one persistent K1 launch per GPU into a 64-bit
// fixed-point image, and the partial images are summed by one NCCL reduce.
// Integer accumulation makes the result independent of the split.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <numeric>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/raybos_gpu.h"
#include "kernels.h"

namespace {

constexpr int kShardTile = 32;  // consecutive (Z-ordered) sources per shard tile

// NVTX range for the duration of a scope (header-only NVTX 3: free unless a
// tool such as Nsight Systems attaches), so the host phases of a call — shard
// plan, launches, the exchange, the readback, field builds — line up with the
// kernels on a timeline.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Device allocation owned by one Device (move-only; freed on destruction, on
// the device it was allocated on), so early error returns cannot leak it.
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  int dev = -1;
  Buf() = default;
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : p(o.p), cap(o.cap), dev(o.dev) {
    o.p = nullptr;
    o.cap = 0;
  }
  Buf& operator=(Buf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      cap = o.cap;
      dev = o.dev;
      o.p = nullptr;
      o.cap = 0;
    }
    return *this;
  }
  ~Buf() { release(); }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    release();
    const size_t want = std::max<size_t>(bytes, 256);
    cudaGetDevice(&dev);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    else p = nullptr;
    return e;
  }
  void release() {
    if (p) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (dev >= 0 && dev != cur) cudaSetDevice(dev);
      cudaFree(p);
      if (dev >= 0 && dev != cur && cur >= 0) cudaSetDevice(cur);
    }
    p = nullptr;
    cap = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Pinned host staging (move-only, freed on destruction).
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  HostBuf(HostBuf&& o) noexcept : p(o.p), cap(o.cap) {
    o.p = nullptr;
    o.cap = 0;
  }
  ~HostBuf() { release(); }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    release();
    const size_t want = std::max<size_t>(bytes, 4096);
    cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocPortable);
    if (e == cudaSuccess) cap = want;
    else p = nullptr;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
  template <typename T>
  T* as(size_t off = 0) const {
    return reinterpret_cast<T*>(static_cast<char*>(p) + off);
  }
};

// Everything a render returns besides the image lives in one device block,
// so a call zeroes it with one memset and reads it back with one D2H copy
// into pinned memory: [counters u64 x8 | counters0 u64 x8 | queue, err_flag |
// check_fail x2 | hit_sum 2n f64 | landed n i64 | hit_sum0 2n | landed0 n]
// (the *0 entries only in bos pair mode; check_fail only written by the
// checked build).
struct StatsLayout {
  size_t n;
  static constexpr size_t kCounters = 0, kCounters0 = 64, kQueue = 128, kCheck = 136,
                          kHeader = 144;
  size_t hit() const { return kHeader; }
  size_t landed() const { return kHeader + 16 * n; }
  size_t hit0() const { return kHeader + 24 * n; }
  size_t landed0() const { return kHeader + 40 * n; }
  size_t bytes(bool pair) const { return kHeader + (pair ? 48 : 24) * n; }
};

struct Device {
  int ordinal = 0;
  int sms = 148;
  int blocks_per_sm[2][3] = {{1, 1, 1}, {1, 1, 1}};  // render kernel, [pair][field mode]
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_join = nullptr;  // orders our stream after the legacy default stream
  float4* grid = nullptr;
  size_t grid_bytes = 0;
  rbk::CellCoef* cells = nullptr;  // per-cell coefficient table (optional, 8x the grid)
  size_t cells_bytes = 0;
  Buf sources, ids, order, image, hit, landed, counters, queue, err, dimage, rays_src, rays_idx,
      rays_uv, rays_status, rays_steps;
  Buf f64[4];  // FP64 node copy (n, gx, gy, gz) for the validation build
  Buf qimage, dbg, dbg_n;
  Buf hit_part, landed_part, hit_part0, landed_part0;  // split-emitter partials
  // rb_trace's cached shard plan on this device (ShardPlan): sources, RNG
  // stream ids and this device's work order, uploaded once per scene
  Buf plan_sources, plan_ids, plan_order;
  bool plan_on_device = false;
  Buf stats;       // StatsLayout block of launch_on / collect_on
  HostBuf hstats;  // its pinned host copy
};

// rb_trace / rb_trace_bos_pair's shard plan, cached across calls on the same
// emitters (bos_run's two traces, a bench's repeated images, an application
// rendering frame after frame): the Z-order sort of the sources (10 ms for 1e5
// sources), the per-device work lists and the device copies of the sources are
// reused when the sources, stream ids and pupil axis are bit-identical to the
// previous call's (checked with memcmp on every call, so the cache can never
// serve a stale plan).
struct ShardPlan {
  bool valid = false;
  std::vector<rb_vec3> sources;
  std::vector<int64_t> ids;
  bool has_ids = false;
  rb_vec3 axis{};
  std::vector<std::vector<int32_t>> work;  // per device of this process
  bool box_valid = false;
  double3 box_lo{}, box_hi{};
  double f_in = 0.0;  // fraction of sources inside the field box (emitter_split)
};

// NCCL, dlopen'ed on first multi-GPU use (libnccl.so.2 — the copy torch has
// already loaded, or the system one; RAYBOS_NCCL_LIB overrides the path, which
// the tests use to substitute a host-staged stand-in on a one-GPU box).
struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclReduce) reduce = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclCommCount) count = nullptr;
  decltype(&ncclGetVersion) version = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* path = std::getenv("RAYBOS_NCCL_LIB");
    if (!path || !*path) path = "libnccl.so.2";
    h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("cannot load ") + path + ": " + dlerror();
      return false;
    }
#define RB_SYM(field, name) field = reinterpret_cast<decltype(field)>(dlsym(h, name))
    RB_SYM(get_unique_id, "ncclGetUniqueId");
    RB_SYM(init_all, "ncclCommInitAll");
    RB_SYM(init_rank, "ncclCommInitRank");
    RB_SYM(reduce, "ncclReduce");
    RB_SYM(all_reduce, "ncclAllReduce");
    RB_SYM(group_start, "ncclGroupStart");
    RB_SYM(group_end, "ncclGroupEnd");
    RB_SYM(destroy, "ncclCommDestroy");
    RB_SYM(count, "ncclCommCount");
    RB_SYM(version, "ncclGetVersion");
#undef RB_SYM
    if (!get_unique_id || !init_all || !init_rank || !reduce || !all_reduce || !group_start ||
        !group_end || !destroy || !count || !version) {
      err = std::string(path) + " lacks required NCCL symbols";
      dlclose(h);
      h = nullptr;
      return false;
    }
    return true;
  }
};

}  // namespace

struct rb_ctx {
  std::vector<Device> devs;
  std::mutex err_mu;  // fail() may run on several device threads at once
  std::string last_error;
  bool has_field = false;
  bool has_field64 = false;  // FP64 node copy present (grids <= RB_FP64_MAX_NODES)
  rb_field_desc field{};
  double3 box_lo{}, box_hi{};
  NcclApi nccl;
  // Multi-GPU.  In-process: one communicator per device (ncclCommInitAll).
  // Rank mode (one process per GPU, rb_create_rank): one device, one
  // communicator, and this process renders shard `rank` of `world`.  Either
  // way every device of every process takes part in every collective.
  std::vector<ncclComm_t> comms;
  int rank = 0, world = 1;
  bool rank_mode = false;  // rb_create_rank made a communicator (also for a one-rank job)
  ShardPlan plan;
};

namespace {

int fail(rb_ctx* ctx, int code, const std::string& msg, char* err = nullptr, size_t len = 0) {
  if (ctx) {
    std::lock_guard<std::mutex> lk(ctx->err_mu);
    ctx->last_error = msg;
  }
  if (err && len) {
    std::strncpy(err, msg.c_str(), len - 1);
    err[len - 1] = '\0';
  }
  return code;
}

#define RB_CUDA(ctx, call)                                                                   \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(ctx, RB_E_CUDA, std::string(#call ": ") + cudaGetErrorString(e_));        \
  } while (0)

double3 d3(const rb_vec3& v) { return make_double3(v.x, v.y, v.z); }

// plane_basis (core.hpp:62-67), evaluated on the host exactly as the reference does.
void plane_basis(const rb_vec3& a, double3& e1, double3& e2) {
  const double3 helper = std::abs(a.x) < 0.9 ? make_double3(1, 0, 0) : make_double3(0, 1, 0);
  const double3 c = make_double3(helper.y * a.z - helper.z * a.y, helper.z * a.x - helper.x * a.z,
                                 helper.x * a.y - helper.y * a.x);
  const double n = std::sqrt(c.x * c.x + c.y * c.y + c.z * c.z);
  e1 = make_double3(c.x / n, c.y / n, c.z / n);
  e2 = make_double3(a.y * e1.z - a.z * e1.y, a.z * e1.x - a.x * e1.z, a.x * e1.y - a.y * e1.x);
}

uint64_t mix_bits(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

rbk::DSurface dsurf(const rb_surface& s) {
  rbk::DSurface d{};
  d.vertex = d3(s.vertex);
  d.axis = d3(s.axis);
  d.R = s.curvature_radius;
  d.planar = std::isfinite(s.curvature_radius) ? 0 : 1;
  // curvature_center(), optics.hpp:35
  d.center = d.planar ? d.vertex
                      : make_double3(s.vertex.x + s.axis.x * s.curvature_radius,
                                     s.vertex.y + s.axis.y * s.curvature_radius,
                                     s.vertex.z + s.axis.z * s.curvature_radius);
  d.absR = std::abs(s.curvature_radius);
  d.aperture = s.aperture_radius;
  d.n_before = s.n_before;
  d.n_after = s.n_after;
  return d;
}

// Reference validation order for the errors run_trace can raise
// (raygen.cpp:29-31, raygen.cpp:69), plus the limits of this implementation.
int validate_scene(rb_ctx* ctx, const rb_scene* s) {
  if (!s) return fail(ctx, RB_E_INVALID, "rb_trace: scene is NULL");
  if (s->n_sources < 0) return fail(ctx, RB_E_INVALID, "rb_trace: negative source count");
  if (s->n_sources > 0x7fffffffLL) return fail(ctx, RB_E_INVALID, "rb_trace: too many sources");
  if (s->sensor.width_px < 1 || s->sensor.height_px < 1)
    return fail(ctx, RB_E_INVALID, "SensorModel: resolution must be positive");
  if (s->n_sources == 0) return RB_OK;
  if (s->rays_per_source < 1)
    return fail(ctx, RB_E_INVALID, "sample_aperture_points: rays_per_source must be >= 1");
  if (s->pupil_radius <= 0.0)
    return fail(ctx, RB_E_INVALID, "sample_aperture_points: radius must be > 0");
  if (s->wavelength <= 0.0)
    return fail(ctx, RB_E_INVALID, "emit_rays: wavelength must be positive");
  if (s->n_elements < 0 || s->n_elements > rbk::kMaxElements)
    return fail(ctx, RB_E_INVALID, "rb_trace: at most 8 optical elements are supported");
  if (s->n_elements > 0 && !s->elements)
    return fail(ctx, RB_E_INVALID, "rb_trace: elements is NULL");
  if (!s->sources) return fail(ctx, RB_E_INVALID, "rb_trace: sources is NULL");
  return RB_OK;
}

// Rows per band of the warp patches (kernels.h): a CTA iteration's 8 patches
// then cover a (256 / rows) x rows block of the pupil lattice.  Without a medium 4
// (8x4 patches, the spot rows of a warp coincide); with one 8 (4x8 patches, a
// 32x8 block per iteration instead of 64x4: 1024^3 +0.9%, tomo / bos +-0.1%;
// 16: tomo -0.5%; scripts/gpu_ab_r02p.sh).  RAYBOS_BAND_ROWS = 4, 8 or 16 overrides.
int band_rows(const rb_ctx* ctx, int with_field) {
  if (!(with_field && ctx->has_field)) return 4;
  int bh = 8;
  if (const char* e = std::getenv("RAYBOS_BAND_ROWS")) bh = std::atoi(e);
  return bh == 4 || bh == 16 ? bh : 8;
}

rbk::KScene make_kscene(const rb_ctx* ctx, const rb_scene* s, int with_field, int accumulate) {
  rbk::KScene k{};
  k.n_sources = s->n_sources;
  k.pupil_center = d3(s->pupil_center);
  plane_basis(s->pupil_axis, k.e1, k.e2);
  k.pupil_radius = s->pupil_radius;
  // emit_rays normalises unit weights by their sum, which is exactly N.
  k.radiance = 1.0 / static_cast<double>(s->rays_per_source);
  k.key_seed = mix_bits(s->seed ^ 0xa93c0de5ULL);
  k.rays = s->rays_per_source;
  k.cells = static_cast<int32_t>(std::ceil(std::sqrt(static_cast<double>(s->rays_per_source))));
  k.sampling = s->sampling == RB_SAMPLING_STRATIFIED ? 0 : 1;
  {
    const int rows = (s->rays_per_source + k.cells - 1) / k.cells;
    const int bh = band_rows(ctx, with_field);
    k.band_h = bh;
    k.band_sh = bh == 16 ? 4 : (bh == 8 ? 3 : 2);
    k.band_rays = bh * k.cells;
    k.band_full = rows / bh;
    k.band_tail = rows - k.band_full * bh;
    k.patch_count = static_cast<int32_t>((static_cast<int64_t>(rows) * k.cells + 31) / 32);
    const int warps = rbk::kBlock / 32;
    // Without a medium the unit's first patch iteration is its pilot, so a
    // coprime stride deals that iteration's 8 patches across the whole pupil
    // (the tile then covers defocused spots); with a medium the pilot is a
    // separate straight trace spread over the unit, and stride 1 keeps a CTA's
    // 8 warps on neighbouring patches — one narrow cone of cells in L1
    // (bos +0.9%, 1024^3 +1.9%, tomo +0.4%).
    int st = std::max(1, k.patch_count / warps);
    while (std::gcd(st, k.patch_count) != 1) ++st;
    k.patch_stride = st % std::max(1, k.patch_count) == 0 ? 1 : st;
  }
  k.with_field = (with_field && ctx->has_field) ? 1 : 0;
  if (k.with_field) k.patch_stride = 1;  // see the patch order above
  if (k.with_field) {
    k.nx = ctx->field.nx;
    k.ny = ctx->field.ny;
    k.nz = ctx->field.nz;
    k.origin = d3(ctx->field.origin);
    k.spacing = d3(ctx->field.spacing);
    k.box_lo = ctx->box_lo;
    k.box_hi = ctx->box_hi;
    k.h = s->delta_xi;
    k.max_steps = s->max_steps;
    k.g_nx = static_cast<unsigned>(k.nx);
    k.g_nxny = static_cast<unsigned>(k.nx) * static_cast<unsigned>(k.ny);
    k.g_ix = static_cast<unsigned>(k.nx - 2);
    k.g_iy = static_cast<unsigned>(k.ny - 2);
    k.g_iz = static_cast<unsigned>(k.nz - 2);
    k.g_mx = static_cast<float>(k.nx - 1);
    k.g_my = static_cast<float>(k.ny - 1);
    k.g_mz = static_cast<float>(k.nz - 1);
    k.c_nx = static_cast<unsigned>(k.nx - 1);
    k.c_nxny = static_cast<unsigned>(k.nx - 1) * static_cast<unsigned>(k.ny - 1);
    k.n_cells = k.c_nxny * static_cast<unsigned>(k.nz - 1);
    const double h = s->delta_xi;
    const double hs[3] = {h / k.spacing.x, h / k.spacing.y, h / k.spacing.z};
    float* dst[6][3] = {{&k.hx, &k.hy, &k.hz},    {&k.hhx, &k.hhy, &k.hhz},
                        {&k.kbx, &k.kby, &k.kbz}, {&k.kcx, &k.kcy, &k.kcz},
                        {&k.krx, &k.kry, &k.krz}, {nullptr, nullptr, nullptr}};
    const double mul[5] = {1.0, 0.5, 0.125 * h, 0.5 * h, h / 6.0};
    for (int r = 0; r < 5; ++r)
      for (int a = 0; a < 3; ++a) *dst[r][a] = static_cast<float>(mul[r] * hs[a]);
    k.kt = static_cast<float>(h / 6.0);
  }
  k.n_elem = s->n_elements;
  for (int e = 0; e < s->n_elements; ++e) {
    const rb_element& x = s->elements[e];
    rbk::DElement& d = k.elem[e];
    d.kind = x.kind;
    d.center = d3(x.center);
    d.axis = d3(x.axis);
    d.radius = x.radius;
    d.focal = x.focal_length;
    d.half_diameter = 0.5 * x.diameter;  // propagate_thin_lens clear radius, optics.cpp:119
    d.front = dsurf(x.front);
    d.back = dsurf(x.back);
  }
  const rb_sensor& se = s->sensor;
  k.s_center = d3(se.center);
  k.s_normal = d3(se.normal);
  k.s_eu = d3(se.e_u);
  k.s_ev = d3(se.e_v);
  k.W = se.width_px;
  k.H = se.height_px;
  k.pitch = se.pitch;
  k.sigma = 0.25 * s->d_tau;                                   // sensor.cpp:65
  k.half_width = se.window_sigmas * k.sigma / se.pitch;        // sensor.cpp:79
  k.inv_s = 1.0 / (k.sigma * 1.41421356237309504880 / se.pitch);  // sensor.cpp:86
  k.inv_s_f = static_cast<float>(k.inv_s);
  k.degenerate = k.sigma < 1e-3 * se.pitch ? 1 : 0;              // sensor.cpp:71
  k.hit_limit = std::ldexp(1.0, 22) / std::max(1, s->rays_per_source);  // render.cuh add_hit
  k.accumulate = accumulate ? 1 : 0;
  return k;
}

uint32_t spread16(uint32_t x) {
  x &= 0xffff;
  x = (x | (x << 8)) & 0x00ff00ff;
  x = (x | (x << 4)) & 0x0f0f0f0f;
  x = (x | (x << 2)) & 0x33333333;
  x = (x | (x << 1)) & 0x55555555;
  return x;
}

// Z-order of the sources' positions projected on the pupil plane, then dealt
// to shards in tiles of kShardTile.  Returns the Z-ordered source list.
std::vector<int32_t> zorder(const rb_scene* s) {
  const int64_t n = s->n_sources;
  std::vector<int32_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  if (n < 2) return idx;
  double3 e1, e2;
  plane_basis(s->pupil_axis, e1, e2);
  std::vector<double> a(n), b(n);
  double amin = 1e300, amax = -1e300, bmin = 1e300, bmax = -1e300;
  for (int64_t i = 0; i < n; ++i) {
    const rb_vec3& p = s->sources[i];
    a[i] = p.x * e1.x + p.y * e1.y + p.z * e1.z;
    b[i] = p.x * e2.x + p.y * e2.y + p.z * e2.z;
    amin = std::min(amin, a[i]);
    amax = std::max(amax, a[i]);
    bmin = std::min(bmin, b[i]);
    bmax = std::max(bmax, b[i]);
  }
  const double sa = amax > amin ? 65535.0 / (amax - amin) : 0.0;
  const double sb = bmax > bmin ? 65535.0 / (bmax - bmin) : 0.0;
  std::vector<uint32_t> key(n);
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t ia = static_cast<uint32_t>((a[i] - amin) * sa);
    const uint32_t ib = static_cast<uint32_t>((b[i] - bmin) * sb);
    key[i] = spread16(ia) | (spread16(ib) << 1);
  }
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t x, int32_t y) { return key[x] < key[y]; });
  return idx;
}

std::vector<int32_t> shard_list(const std::vector<int32_t>& z, int64_t index, int64_t count) {
  std::vector<int32_t> out;
  out.reserve(z.size() / std::max<int64_t>(count, 1) + kShardTile);
  for (size_t p = 0; p < z.size(); ++p)
    if ((static_cast<int64_t>(p) / kShardTile) % count == index) out.push_back(z[p]);
  return out;
}

struct PartialOut {
  std::vector<double> hit, hit0;
  std::vector<long long> landed, landed0;
  unsigned long long counters[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long counters0[6] = {0, 0, 0, 0, 0, 0};
  float ms = 0.f;
  int err_flag = 0;
  int launches = 0;  // kernels launch_on launched
  int k1 = 0;        // rb_trace_out::k1_kernel of this launch
  bool pair = false;
  unsigned check_fail[2] = {0, 0};  // checked build: violations, last site code
};

// CTAs per emitter (KScene::split).  Splitting an emitter's rays over several
// CTAs keeps fewer distinct cones in flight, so the cells they read stay in
// L2; each chunk costs one pilot, one tile flush and a barrier wait for its
// slowest warp.  The chunk is sized to about 1.25e6 RK4 steps, estimating the
// steps per ray as the box depth along the pupil axis over h, halved for
// emitters inside the box.  Measured optimum with the band-order patches
// (scripts/gpu_ab_r02m.sh / r02n.sh): tomo 1 (+1.7% over 8), bos 4 (+1.7% over
// 20), 1024^3 20-40 (one or two patch iterations per chunk; 5: -0.8%).  (With
// the earlier coprime patch stride the optimum was 8 / 24 / 48: each chunk
// then spanned the whole cone.)  Independently, a work list
// shorter than the resident CTAs is split until every CTA gets two units (3
// emitters x 4e6 rays: 1.29 s -> 17 ms), never below one patch iteration per
// unit.  RAYBOS_SPLIT overrides.
// Fraction of the sources inside the field's box.
double inside_fraction(const rb_ctx* ctx, const rb_scene* s) {
  int64_t inside = 0;
  for (int64_t q = 0; q < s->n_sources; ++q) {
    const rb_vec3 p = s->sources[q];
    inside += (p.x >= ctx->box_lo.x && p.x <= ctx->box_hi.x && p.y >= ctx->box_lo.y &&
               p.y <= ctx->box_hi.y && p.z >= ctx->box_lo.z && p.z <= ctx->box_hi.z);
  }
  return s->n_sources ? static_cast<double>(inside) / s->n_sources : 0.0;
}

int emitter_split(const rb_ctx* ctx, const rb_scene* s, const rbk::KScene& k, size_t n_work,
                  int resident_ctas, double f_in) {
  const int iters = std::max(1, (k.patch_count + rbk::kBlock / 32 - 1) / (rbk::kBlock / 32));
  const int cap = std::min(iters, 4096);
  if (const char* e = std::getenv("RAYBOS_SPLIT")) return std::max(1, std::min(cap, std::atoi(e)));
  double split = 1.0;
  if (k.with_field && k.h > 0.0) {
    const double ext[3] = {ctx->box_hi.x - ctx->box_lo.x, ctx->box_hi.y - ctx->box_lo.y,
                           ctx->box_hi.z - ctx->box_lo.z};
    const double ax[3] = {s->pupil_axis.x, s->pupil_axis.y, s->pupil_axis.z};
    const double an = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
    double depth = 0.0;
    for (int a = 0; a < 3; ++a) depth += std::fabs(ext[a] * ax[a]) / (an > 0.0 ? an : 1.0);
    // emitters inside the box (Tomo particles) trace half the depth on average
    const double steps = std::min<double>(depth / k.h * (1.0 - 0.5 * f_in), s->max_steps);
    split = std::min(128.0, std::round(static_cast<double>(s->rays_per_source) * steps / 1.25e6));
  }
  if (n_work > 0 && n_work < static_cast<size_t>(resident_ctas))
    split = std::max(split, std::ceil(2.0 * resident_ctas / static_cast<double>(n_work)));
  // K1 gives each chunk ceil(iters / split) patch iterations; trim the split to
  // the chunks that then have work (bos: 25 -> 20, five empty units per emitter)
  const int sp = static_cast<int>(std::max(1.0, std::min(static_cast<double>(cap), split)));
  const int per = (iters + sp - 1) / sp;
  return (iters + per - 1) / per;
}

// One device renders the given work list into dev.image (already zeroed or
// caller-owned when image_override != nullptr).
// Caller-provided device buffers (rb_trace_shard's image, rb_image_from_fixed's
// input) are typically written on the caller's stream, usually the device's
// legacy default stream (torch's default).  Our stream is non-blocking, so make
// it wait for everything already queued there before touching them.
cudaError_t join_default_stream(Device& dev) {
  cudaError_t e = cudaEventRecord(dev.ev_join, 0);
  if (e != cudaSuccess) return e;
  return cudaStreamWaitEvent(dev.stream, dev.ev_join, 0);
}

// Runs fn(dev) for every device of the context, each on its own host thread
// when there are several (field builds of a 1024^3 grid take ~1 s per device,
// so N devices build in parallel rather than in N seconds).
template <typename F>
int for_each_device(rb_ctx* ctx, F&& fn) {
  const size_t nd = ctx->devs.size();
  if (nd == 1) return fn(ctx->devs[0]);
  std::vector<int> rcs(nd, RB_OK);
  std::vector<std::thread> pool;
  for (size_t i = 0; i < nd; ++i) pool.emplace_back([&, i] { rcs[i] = fn(ctx->devs[i]); });
  for (auto& t : pool) t.join();
  for (int rc : rcs)
    if (rc) return rc;
  return RB_OK;
}

// Phase 1 of a render on one device: uploads, zeroing, K1 (+ the split-stats
// kernel), all queued on the device's stream.  image_target: a caller-owned
// device image to accumulate into instead of the device's own (zeroed) one.
// zero_stats: also zero the per-source stats, so entries this device does not
// own are 0 rather than stale (rank mode sums them across processes).
// use_plan: the work list is ctx->plan's for this device, and the sources /
// ids / order live in the device's plan buffers (uploaded on first use).
int launch_on(rb_ctx* ctx, Device& dev, const rb_scene* s, const rbk::KScene& base,
              const std::vector<int32_t>& work, unsigned long long* image_target, bool zero_stats,
              bool use_plan, double f_in, PartialOut& po) {
  NvtxRange nvtx_("raybos launch");
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  const int64_t n = s->n_sources;
  const size_t npx = static_cast<size_t>(s->sensor.width_px) * s->sensor.height_px;
  cudaStream_t st = dev.stream;
  rbk::KScene k = base;
  po.pair = k.pair != 0;
  if (image_target) RB_CUDA(ctx, join_default_stream(dev));
  Buf& bsrc = use_plan ? dev.plan_sources : dev.sources;
  Buf& bids = use_plan ? dev.plan_ids : dev.ids;
  Buf& bord = use_plan ? dev.plan_order : dev.order;
  const bool upload = !use_plan || !dev.plan_on_device;
  if (upload) {
    RB_CUDA(ctx, bsrc.ensure(sizeof(double) * 3 * n));
    RB_CUDA(ctx, cudaMemcpyAsync(bsrc.p, s->sources, sizeof(double) * 3 * n,
                                 cudaMemcpyHostToDevice, st));
    if (s->source_ids) {
      RB_CUDA(ctx, bids.ensure(sizeof(int64_t) * n));
      RB_CUDA(ctx, cudaMemcpyAsync(bids.p, s->source_ids, sizeof(int64_t) * n,
                                   cudaMemcpyHostToDevice, st));
    }
    RB_CUDA(ctx, bord.ensure(sizeof(int32_t) * std::max<size_t>(work.size(), 1)));
    if (!work.empty())
      RB_CUDA(ctx, cudaMemcpyAsync(bord.p, work.data(), sizeof(int32_t) * work.size(),
                                   cudaMemcpyHostToDevice, st));
    if (use_plan) dev.plan_on_device = true;
  }
  k.sources = bsrc.as<double>();
  k.source_ids = s->source_ids ? bids.as<int64_t>() : nullptr;
  k.order = bord.as<int32_t>();
  k.n_work = static_cast<int32_t>(work.size());
  const StatsLayout L{static_cast<size_t>(n)};
  RB_CUDA(ctx, dev.stats.ensure(L.bytes(true)));
  // zero_stats: the per-source entries too, so entries this device does not own
  // are 0 (rank mode sums them across processes); else the header only
  RB_CUDA(ctx, cudaMemsetAsync(dev.stats.p, 0, zero_stats ? L.bytes(k.pair) : L.kHeader, st));
  char* sb = dev.stats.as<char>();
  k.hit_sum = reinterpret_cast<double*>(sb + L.hit());
  k.landed = reinterpret_cast<long long*>(sb + L.landed());
  k.counters = reinterpret_cast<unsigned long long*>(sb + L.kCounters);
  if (k.pair) {
    k.hit_sum0 = reinterpret_cast<double*>(sb + L.hit0());
    k.landed0 = reinterpret_cast<long long*>(sb + L.landed0());
    k.counters0 = reinterpret_cast<unsigned long long*>(sb + L.kCounters0);
  }
  k.queue = reinterpret_cast<int*>(sb + L.kQueue);
  k.err_flag = k.queue + 1;
  k.check_fail = reinterpret_cast<unsigned*>(sb + L.kCheck);
  k.grid = dev.grid;
  k.cell_table = dev.cells;
  if (k.accumulate) {
    if (image_target) {
      k.image = image_target;
    } else {
      RB_CUDA(ctx, dev.image.ensure(sizeof(unsigned long long) * npx));
      RB_CUDA(ctx, cudaMemsetAsync(dev.image.p, 0, sizeof(unsigned long long) * npx, st));
      k.image = dev.image.as<unsigned long long>();
    }
  }
  if (k.with_field && !dev.grid) return fail(ctx, RB_E_RUNTIME, "rb_trace: field not uploaded");
  k.split = emitter_split(ctx, s, k, work.size(),
                          dev.sms * dev.blocks_per_sm[k.pair ? 1 : 0][rbk::field_mode(k)], f_in);
  if (const char* e = std::getenv("RAYBOS_K1"); e && e[0] == 'w' && k.with_field && !k.pair) {
    // render_warps (warp-level work items, no CTA barrier): the
    // split becomes items per emitter, kWarps per render_emitters chunk
    k.warp_mode = 1;
    const int warps = rbk::kBlock / 32;
    const int want = std::max(1, std::min(k.patch_count, k.split * warps));
    const int per = (k.patch_count + want - 1) / want;
    k.split = (k.patch_count + per - 1) / per;
  }
  po.k1 = k.warp_mode ? 2 : 1;
  if (k.split > 1) {
    const size_t units = work.size() * static_cast<size_t>(k.split);
    RB_CUDA(ctx, dev.hit_part.ensure(sizeof(long long) * 2 * units));
    RB_CUDA(ctx, dev.landed_part.ensure(sizeof(long long) * units));
    k.hit_part = dev.hit_part.as<long long>();
    k.landed_part = dev.landed_part.as<long long>();
    if (k.pair) {
      RB_CUDA(ctx, dev.hit_part0.ensure(sizeof(long long) * 2 * units));
      RB_CUDA(ctx, dev.landed_part0.ensure(sizeof(long long) * units));
      k.hit_part0 = dev.hit_part0.as<long long>();
      k.landed_part0 = dev.landed_part0.as<long long>();
    }
  }
  const int64_t units = static_cast<int64_t>(work.size()) * k.split;
  const int grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(dev.sms * dev.blocks_per_sm[k.pair ? 1 : 0][rbk::field_mode(k)],
                           std::max<int64_t>(1, units))));
  RB_CUDA(ctx, cudaEventRecord(dev.ev0, st));
  po.launches = 0;
  if (!work.empty()) {
    RB_CUDA(ctx, rbk::launch_render(k, grid, st));
    RB_CUDA(ctx, rbk::launch_emitter_stats(k, st));
    po.launches = 1 + (k.split > 1 && k.n_work > 0 ? 1 : 0);
  }
  RB_CUDA(ctx, cudaEventRecord(dev.ev1, st));
  return RB_OK;
}

// Phase 3: per-source stats, counters and the error flag to the host, then
// wait for the device's stream (which also covers any collective queued on it).
int collect_on(rb_ctx* ctx, Device& dev, const rb_scene* s, PartialOut& po) {
  NvtxRange nvtx_("raybos readback");
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  const int64_t n = s->n_sources;
  const StatsLayout L{static_cast<size_t>(n)};
  const size_t bytes = L.bytes(po.pair);
  RB_CUDA(ctx, dev.hstats.ensure(bytes));
  RB_CUDA(ctx, cudaMemcpyAsync(dev.hstats.p, dev.stats.p, bytes, cudaMemcpyDeviceToHost,
                               dev.stream));
  RB_CUDA(ctx, cudaStreamSynchronize(dev.stream));
  const HostBuf& h = dev.hstats;
  po.hit.assign(h.as<double>(L.hit()), h.as<double>(L.hit()) + 2 * n);
  po.landed.assign(h.as<long long>(L.landed()), h.as<long long>(L.landed()) + n);
  std::memcpy(po.counters, h.as<unsigned long long>(L.kCounters), sizeof(po.counters));
  if (po.pair) {
    po.hit0.assign(h.as<double>(L.hit0()), h.as<double>(L.hit0()) + 2 * n);
    po.landed0.assign(h.as<long long>(L.landed0()), h.as<long long>(L.landed0()) + n);
    std::memcpy(po.counters0, h.as<unsigned long long>(L.kCounters0), sizeof(po.counters0));
  }
  po.err_flag = *h.as<int>(L.kQueue + sizeof(int));
  po.check_fail[0] = *h.as<unsigned>(L.kCheck);
  po.check_fail[1] = *h.as<unsigned>(L.kCheck + sizeof(unsigned));
  RB_CUDA(ctx, cudaEventElapsedTime(&po.ms, dev.ev0, dev.ev1));
  return RB_OK;
}

// One device renders the given work list (rb_trace_shard): phase 1 + phase 3.
int render_on(rb_ctx* ctx, Device& dev, const rb_scene* s, const rbk::KScene& base,
              const std::vector<int32_t>& work, unsigned long long* image_target,
              PartialOut& po) {
  const double f_in = base.with_field ? inside_fraction(ctx, s) : 0.0;
  if (int rc = launch_on(ctx, dev, s, base, work, image_target, false, false, f_in, po)) return rc;
  return collect_on(ctx, dev, s, po);
}

// The kernel's error flag (KScene::err_flag) as the reference's exception text.
int flag_error(rb_ctx* ctx, int flag, const rb_scene* s) {
  if (flag & 1) return fail(ctx, RB_E_INVALID, "emit_rays: source coincides with aperture point");
  if (flag & 2) {
    char lim[64];
    std::snprintf(lim, sizeof lim, "%.6g", std::ldexp(1.0, 22) / std::max(1, s->rays_per_source));
    return fail(ctx, RB_E_RUNTIME,
                std::string("rb_trace: a sensor-plane hit (|u| or |v| > ") + lim +
                    " m) exceeds the fixed-point range of DotHitStats::hit_sum");
  }
  return RB_OK;
}

// The checked build's verdict (RB_CHECKED kernels; always 0 otherwise).
int check_error(rb_ctx* ctx, const unsigned* cf) {
  if (!cf[0]) return RB_OK;
  return fail(ctx, RB_E_RUNTIME,
              "checked build: " + std::to_string(cf[0]) +
                  " out-of-range index(es) in K1, last at site " + std::to_string(cf[1]) +
                  " (render.cuh / grin.cuh RB_CHECK)");
}

// Phase 2, the one exchange step, queued on every device's stream after its
// render.  In-process (one communicator per device): a grouped ncclReduce of
// the fixed-point images onto device 0; the stats are merged on the host
// (every source has exactly one owner).  Rank mode (one process per GPU): the
// same image reduce onto rank 0, plus ncclAllReduce of the per-source stats,
// the counters and the error flag, so every rank returns the whole call's
// statistics.  Stats entries have one non-zero contributor and the image is
// an integer, so every sum is exact: bit-identical for any device count.
int exchange(rb_ctx* ctx, const rb_scene* s, bool image, bool pair) {
  NvtxRange nvtx_("raybos exchange (NCCL)");
  NcclApi& api = ctx->nccl;
  const size_t n = static_cast<size_t>(s->n_sources);
  const size_t npx = static_cast<size_t>(s->sensor.width_px) * s->sensor.height_px;
  const bool dist = ctx->rank_mode;
  if (!image && !dist) return RB_OK;
  if (api.group_start() != ncclSuccess) return fail(ctx, RB_E_CUDA, "ncclGroupStart failed");
  ncclResult_t r = ncclSuccess;
  const StatsLayout L{n};
  for (size_t d = 0; d < ctx->devs.size() && r == ncclSuccess; ++d) {
    Device& dv = ctx->devs[d];
    cudaSetDevice(dv.ordinal);
    ncclComm_t c = ctx->comms[d];
    cudaStream_t st = dv.stream;
    char* sb = dv.stats.as<char>();
    if (image) r = api.reduce(dv.image.p, dv.image.p, npx, ncclUint64, ncclSum, 0, c, st);
    if (dist && r == ncclSuccess) {
      ncclResult_t q[8] = {
          api.all_reduce(sb + L.hit(), sb + L.hit(), 2 * n, ncclFloat64, ncclSum, c, st),
          api.all_reduce(sb + L.landed(), sb + L.landed(), n, ncclInt64, ncclSum, c, st),
          api.all_reduce(sb + L.kCounters, sb + L.kCounters, 8, ncclUint64, ncclSum, c, st),
          api.all_reduce(sb + L.kQueue + sizeof(int), sb + L.kQueue + sizeof(int), 1, ncclInt32,
                         ncclMax, c, st),
          ncclSuccess, ncclSuccess, ncclSuccess, ncclSuccess};
      if (pair) {
        q[4] = api.all_reduce(sb + L.hit0(), sb + L.hit0(), 2 * n, ncclFloat64, ncclSum, c, st);
        q[5] = api.all_reduce(sb + L.landed0(), sb + L.landed0(), n, ncclInt64, ncclSum, c, st);
        q[6] = api.all_reduce(sb + L.kCounters0, sb + L.kCounters0, 8, ncclUint64, ncclSum, c,
                              st);
      }
      for (ncclResult_t x : q)
        if (x != ncclSuccess) r = x;
    }
  }
  const ncclResult_t e = api.group_end();
  if (r != ncclSuccess || e != ncclSuccess)
    return fail(ctx, RB_E_CUDA,
                "NCCL collective failed (NCCL error " + std::to_string(r != ncclSuccess ? r : e) +
                    ")");
  return RB_OK;
}

// The cached shard plan for this scene (ShardPlan), rebuilt when the sources,
// stream ids or pupil axis differ from the previous call's: device d of rank r
// takes shard r * nd + d of world * nd, from the same Z-order plan as
// rb_plan_shards.
const ShardPlan& shard_plan(rb_ctx* ctx, const rb_scene* s) {
  NvtxRange nvtx_("raybos shard plan");
  ShardPlan& p = ctx->plan;
  const size_t n = static_cast<size_t>(s->n_sources);
  const bool same =
      p.valid && p.sources.size() == n &&
      std::memcmp(p.sources.data(), s->sources, n * sizeof(rb_vec3)) == 0 &&
      p.has_ids == (s->source_ids != nullptr) &&
      (!s->source_ids || std::memcmp(p.ids.data(), s->source_ids, n * sizeof(int64_t)) == 0) &&
      std::memcmp(&p.axis, &s->pupil_axis, sizeof(rb_vec3)) == 0;
  if (!same) {
    p.sources.assign(s->sources, s->sources + n);
    p.has_ids = s->source_ids != nullptr;
    if (p.has_ids) p.ids.assign(s->source_ids, s->source_ids + n);
    else p.ids.clear();
    p.axis = s->pupil_axis;
    const int nd = static_cast<int>(ctx->devs.size());
    const int64_t total = static_cast<int64_t>(nd) * ctx->world;
    const std::vector<int32_t> z = zorder(s);
    p.work.assign(nd, {});
    for (int d = 0; d < nd; ++d)
      p.work[d] = shard_list(z, static_cast<int64_t>(ctx->rank) * nd + d, total);
    p.box_valid = false;
    p.valid = true;
    for (Device& dev : ctx->devs) dev.plan_on_device = false;
  }
  if (ctx->has_field &&
      (!p.box_valid || std::memcmp(&p.box_lo, &ctx->box_lo, sizeof(double3)) != 0 ||
       std::memcmp(&p.box_hi, &ctx->box_hi, sizeof(double3)) != 0)) {
    p.f_in = inside_fraction(ctx, s);
    p.box_lo = ctx->box_lo;
    p.box_hi = ctx->box_hi;
    p.box_valid = true;
  }
  return p;
}

// Renders this process's shards and combines them (exchange).  Every device
// takes part even when its shard is empty, so the collectives always see every
// rank.  tail: optional work queued on device 0 of rank 0 after the exchange and
// before the stats readback (rb_trace's image copies), so one stream sync covers
// both.
int run_shards(rb_ctx* ctx, const rb_scene* s, const rbk::KScene& base,
               std::vector<std::vector<int32_t>>& work, std::vector<PartialOut>& parts,
               const std::function<int(Device&)>& tail = nullptr) {
  const int nd = static_cast<int>(ctx->devs.size());
  const ShardPlan& plan = shard_plan(ctx, s);
  work = plan.work;
  parts.assign(nd, PartialOut{});
  const bool dist = ctx->rank_mode;
  const double f_in = base.with_field ? plan.f_in : 0.0;
  if (int rc = for_each_device(ctx, [&](Device& dev) -> int {
        const size_t i = static_cast<size_t>(&dev - ctx->devs.data());
        return launch_on(ctx, dev, s, base, work[i], nullptr, dist, true, f_in, parts[i]);
      }))
    return rc;
  if (static_cast<int64_t>(nd) * ctx->world > 1 || ctx->rank_mode)
    if (int rc = exchange(ctx, s, base.accumulate != 0, base.pair != 0)) return rc;
  if (tail && ctx->rank == 0)
    if (int rc = tail(ctx->devs[0])) return rc;
  if (int rc = for_each_device(ctx, [&](Device& dev) -> int {
        const size_t i = static_cast<size_t>(&dev - ctx->devs.data());
        return collect_on(ctx, dev, s, parts[i]);
      }))
    return rc;
  for (const PartialOut& po : parts) {
    if (int rc = check_error(ctx, po.check_fail)) return rc;
    if (po.err_flag) return flag_error(ctx, po.err_flag, s);
  }
  return RB_OK;
}

// Per-source DotHitStats and counters of one leg out of run_shards' parts.
void merge_stats(const rb_ctx* ctx, const rb_scene* s,
                 const std::vector<std::vector<int32_t>>& work,
                 const std::vector<PartialOut>& parts, bool leg0, double* hit_sum, int64_t* landed,
                 unsigned long long c[6], int64_t& landed_total) {
  landed_total = 0;
  for (int j = 0; j < 6; ++j) c[j] = 0;
  auto take = [&](const PartialOut& po, int32_t src) {
    const std::vector<double>& h = leg0 ? po.hit0 : po.hit;
    const std::vector<long long>& l = leg0 ? po.landed0 : po.landed;
    if (hit_sum) {
      hit_sum[2 * src] = h[2 * src];
      hit_sum[2 * src + 1] = h[2 * src + 1];
    }
    if (landed) landed[src] = l[src];
    landed_total += l[src];
  };
  if (ctx->rank_mode) {  // all-reduced: device 0 holds every source and the totals
    const PartialOut& po = parts[0];
    for (int32_t src = 0; src < static_cast<int32_t>(s->n_sources); ++src) take(po, src);
    for (int j = 0; j < 6; ++j) c[j] = leg0 ? po.counters0[j] : po.counters[j];
    return;
  }
  for (size_t d = 0; d < parts.size(); ++d) {
    for (int j = 0; j < 6; ++j) c[j] += leg0 ? parts[d].counters0[j] : parts[d].counters[j];
    for (int32_t src : work[d]) take(parts[d], src);
  }
}

void fill_report(rb_trace_out* out, const rb_scene* s, int64_t owned_sources,
                 const unsigned long long* c, int64_t landed_total) {
  out->emitted = owned_sources * static_cast<int64_t>(s->rays_per_source);
  out->landed_total = landed_total;
  out->lost = static_cast<int64_t>(c[0]);
  out->blocked_aperture = static_cast<int64_t>(c[1]);
  out->blocked_miss = static_cast<int64_t>(c[2]);
  out->blocked_tir = static_cast<int64_t>(c[3]);
  out->blocked_sensor_miss = static_cast<int64_t>(c[4]);
  out->total_steps = static_cast<int64_t>(c[5]);
  out->config_hash = s->config_hash;
}

void free_field(Device& dev) {
  cudaSetDevice(dev.ordinal);
  if (dev.grid) cudaFree(dev.grid);
  if (dev.cells) cudaFree(dev.cells);
  dev.grid = nullptr;
  dev.grid_bytes = 0;
  dev.cells = nullptr;
  dev.cells_bytes = 0;
}

int upload_grid(rb_ctx* ctx, Device& dev, size_t count) {
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  free_field(dev);
  RB_CUDA(ctx, cudaMalloc(&dev.grid, count * sizeof(float4)));
  dev.grid_bytes = count * sizeof(float4);
  return RB_OK;
}

// Per-cell coefficient table (kernels.h CellCoef): a reload in the RK4 loop
// then reads one 128 B line instead of 8 corners + 28 FADDs.  It is 8x the node
// grid, so it is built when it fits in the free memory minus a reserve of
// max(4 GiB, 10% of the device) (1024^3: 137 GB of 183 GB); RAYBOS_CELL_TABLE=0
// turns it off.  Results are bit-identical either way.
int build_cell_table(rb_ctx* ctx, Device& dev, const rb_field_desc* desc) {
  const char* env = std::getenv("RAYBOS_CELL_TABLE");
  if (env && env[0] == '0') return RB_OK;
  const size_t cells = static_cast<size_t>(desc->nx - 1) * (desc->ny - 1) * (desc->nz - 1);
  const size_t bytes = cells * sizeof(rbk::CellCoef);
  size_t free_b = 0, total_b = 0;
  RB_CUDA(ctx, cudaMemGetInfo(&free_b, &total_b));
  const size_t reserve = std::max<size_t>(size_t(4) << 30, total_b / 10);
  if (bytes + reserve > free_b) return RB_OK;
  if (cudaMalloc(&dev.cells, bytes) != cudaSuccess) {
    cudaGetLastError();
    dev.cells = nullptr;
    return RB_OK;
  }
  dev.cells_bytes = bytes;
  RB_CUDA(ctx, rbk::launch_build_cells(dev.grid, desc->nx, desc->ny, desc->nz, dev.cells,
                                       dev.stream));
  return RB_OK;
}

// Keeps the field hot in L2 with an access-policy window on the render stream
// when it fits the persisting carve-out.  A window over a field larger than
// that (the bench scenes' cell tables, 1-137 GB) gave no speedup (the emitter
// split already keeps the cones' cells at 97% L2 hits) and its persisting
// lines pushed the render kernel's spill lines out to DRAM (2.5 GB of
// write-backs per 1e8 Tomo rays, 23 MB without it), so it is left off there.
// RAYBOS_L2_WINDOW=0 / 1 forces it off / on.
void set_l2_window(Device& dev) {
  cudaSetDevice(dev.ordinal);
  int max_persist = 0, max_window = 0;
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev.ordinal);
  cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev.ordinal);
  void* base = dev.cells ? static_cast<void*>(dev.cells) : static_cast<void*>(dev.grid);
  const size_t bytes = dev.cells ? dev.cells_bytes : dev.grid_bytes;
  const char* e = std::getenv("RAYBOS_L2_WINDOW");
  const bool on = e ? e[0] != '0' : bytes <= static_cast<size_t>(std::max(max_persist, 0));
  cudaStreamAttrValue attr{};
  if (on && max_persist > 0 && max_window > 0 && base) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(max_persist));
    const size_t win = std::min<size_t>(bytes, static_cast<size_t>(max_window));
    attr.accessPolicyWindow.base_ptr = base;
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio =
        std::min(1.0f, static_cast<float>(max_persist) / static_cast<float>(win));
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  }
  cudaStreamSetAttribute(dev.stream, cudaStreamAttributeAccessPolicyWindow, &attr);  // or clear it
  cudaGetLastError();  // the window is a hint; never fail on it
}

int check_field_desc(rb_ctx* ctx, const rb_field_desc* d) {
  if (!d) return fail(ctx, RB_E_INVALID, "rb_set_field: desc is NULL");
  if (d->nx < 2 || d->ny < 2 || d->nz < 2)
    return fail(ctx, RB_E_INVALID, "DensityVolume: dims must be >= 2 in each axis");
  if (d->spacing.x <= 0.0 || d->spacing.y <= 0.0 || d->spacing.z <= 0.0)
    return fail(ctx, RB_E_INVALID, "DensityVolume: spacing must be positive");
  const double cnt = static_cast<double>(d->nx) * d->ny * d->nz;
  if (cnt >= 4294967296.0)
    return fail(ctx, RB_E_INVALID, "rb_set_field: grids are limited to 2^32 nodes");
  return RB_OK;
}

// A failed field load leaves no field behind (and no device memory held).
int drop_field(rb_ctx* ctx, int rc) {
  for (Device& dev : ctx->devs) {
    free_field(dev);
    for (Buf& b : dev.f64) b.release();
  }
  ctx->has_field = ctx->has_field64 = false;
  return rc;
}

void set_box(rb_ctx* ctx, const rb_field_desc* d) {
  ctx->field = *d;
  // GriddedField::bounds, scene.cpp:94-97
  ctx->box_lo = d3(d->origin);
  ctx->box_hi = make_double3(d->origin.x + (d->nx - 1) * d->spacing.x,
                             d->origin.y + (d->ny - 1) * d->spacing.y,
                             d->origin.z + (d->nz - 1) * d->spacing.z);
  ctx->has_field = true;
  ctx->has_field64 = static_cast<long long>(d->nx) * d->ny * d->nz <= RB_FP64_MAX_NODES;
}

}  // namespace

extern "C" {

int rb_abi_version(void) { return RB_ABI_VERSION; }

const char* rb_last_error(const rb_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

int rb_device_count(const rb_ctx* ctx) { return ctx ? static_cast<int>(ctx->devs.size()) : 0; }

}  // extern "C"

namespace {

void destroy_device(Device& d) {
  free_field(d);
  for (Buf& b : d.f64) b.release();
  for (Buf* b : {&d.qimage, &d.dbg, &d.dbg_n, &d.hit_part,
                 &d.landed_part, &d.hit_part0, &d.landed_part0, &d.sources, &d.ids, &d.order,
                 &d.image, &d.hit, &d.landed, &d.counters, &d.queue, &d.err, &d.dimage,
                 &d.rays_src, &d.rays_idx, &d.rays_uv, &d.rays_status, &d.rays_steps,
                 &d.plan_sources, &d.plan_ids, &d.plan_order, &d.stats})
    b->release();
  d.hstats.release();
  if (d.ev0) cudaEventDestroy(d.ev0);
  if (d.ev1) cudaEventDestroy(d.ev1);
  if (d.ev_join) cudaEventDestroy(d.ev_join);
  if (d.stream) cudaStreamDestroy(d.stream);
  d.ev0 = d.ev1 = d.ev_join = nullptr;
  d.stream = nullptr;
}

void destroy_ctx(rb_ctx* ctx) {
  for (ncclComm_t c : ctx->comms)
    if (c && ctx->nccl.destroy) ctx->nccl.destroy(c);
  ctx->comms.clear();
  for (Device& d : ctx->devs) destroy_device(d);
  delete ctx;
}

// A context over the given device ordinals (streams, events, occupancy).
int make_ctx(const int* ordinals, int n, rb_ctx** out, char* err, size_t errlen) {
  if (!out) return fail(nullptr, RB_E_INVALID, "rb_create: out is NULL", err, errlen);
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(nullptr, RB_E_NODEVICE,
                std::string("rb_create: no CUDA device (") + cudaGetErrorString(e) +
                    "); this library has no CPU fallback",
                err, errlen);
  if (n < 1) return fail(nullptr, RB_E_INVALID, "rb_create: no devices requested", err, errlen);
  for (int i = 0; i < n; ++i)
    if (ordinals[i] < 0 || ordinals[i] >= count)
      return fail(nullptr, RB_E_INVALID, "rb_create: device ordinal out of range", err, errlen);
  auto* ctx = new rb_ctx();
  for (int i = 0; i < n; ++i) {
    Device dev;
    dev.ordinal = ordinals[i];
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, dev.ordinal);
    if (prop.major != 10) {
      destroy_ctx(ctx);
      return fail(nullptr, RB_E_NODEVICE,
                  std::string("rb_create: device ") + prop.name +
                      " is not sm_100 (Blackwell B200); this build targets sm_100a only",
                  err, errlen);
    }
    cudaSetDevice(dev.ordinal);
    dev.sms = prop.multiProcessorCount;
    ctx->devs.push_back(std::move(dev));
    Device& d = ctx->devs.back();
    if (cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&d.ev0) != cudaSuccess || cudaEventCreate(&d.ev1) != cudaSuccess ||
        cudaEventCreateWithFlags(&d.ev_join, cudaEventDisableTiming) != cudaSuccess) {
      destroy_ctx(ctx);
      return fail(nullptr, RB_E_CUDA, "rb_create: stream/event creation failed", err, errlen);
    }
    rbk::render_occupancy(d.blocks_per_sm);
    for (auto& row : d.blocks_per_sm)
      for (int& b : row) b = std::max(b, 1);
  }
  *out = ctx;
  return RB_OK;
}

}  // namespace

extern "C" {

int rb_create_devices(const int* devices, int n_devices, rb_ctx** out, char* err, size_t errlen) {
  if (!devices) return fail(nullptr, RB_E_INVALID, "rb_create: devices is NULL", err, errlen);
  if (int rc = make_ctx(devices, n_devices, out, err, errlen)) return rc;
  rb_ctx* ctx = *out;
  if (n_devices > 1) {  // one communicator per device, all in this process
    std::string msg;
    if (!ctx->nccl.load(msg)) {
      *out = nullptr;
      destroy_ctx(ctx);
      return fail(nullptr, RB_E_CUDA, msg, err, errlen);
    }
    ctx->comms.assign(n_devices, nullptr);
    const ncclResult_t r = ctx->nccl.init_all(ctx->comms.data(), n_devices, devices);
    if (r != ncclSuccess) {
      ctx->comms.clear();
      *out = nullptr;
      destroy_ctx(ctx);
      return fail(nullptr, RB_E_CUDA,
                  "rb_create: ncclCommInitAll failed (NCCL error " + std::to_string(r) + ")", err,
                  errlen);
    }
  }
  return RB_OK;
}

int rb_create(int n_devices, int first_device, rb_ctx** out, char* err, size_t errlen) {
  if (!out) return fail(nullptr, RB_E_INVALID, "rb_create: out is NULL", err, errlen);
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(nullptr, RB_E_NODEVICE,
                std::string("rb_create: no CUDA device (") + cudaGetErrorString(e) +
                    "); this library has no CPU fallback",
                err, errlen);
  if (first_device < 0 || first_device >= count)
    return fail(nullptr, RB_E_INVALID, "rb_create: first_device out of range", err, errlen);
  const int n = n_devices <= 0 ? count - first_device : n_devices;
  if (first_device + n > count)
    return fail(nullptr, RB_E_INVALID, "rb_create: not enough devices", err, errlen);
  std::vector<int> list(n);
  for (int i = 0; i < n; ++i) list[i] = first_device + i;
  return rb_create_devices(list.data(), n, out, err, errlen);
}

int rb_nccl_unique_id(void* id, size_t len, char* err, size_t errlen) {
  if (!id || len < sizeof(ncclUniqueId))
    return fail(nullptr, RB_E_INVALID, "rb_nccl_unique_id: buffer smaller than ncclUniqueId", err,
                errlen);
  NcclApi api;
  std::string msg;
  if (!api.load(msg)) return fail(nullptr, RB_E_CUDA, msg, err, errlen);
  ncclUniqueId u;
  const ncclResult_t r = api.get_unique_id(&u);
  if (r != ncclSuccess)
    return fail(nullptr, RB_E_CUDA, "ncclGetUniqueId failed (NCCL error " + std::to_string(r) + ")",
                err, errlen);
  std::memcpy(id, &u, sizeof(u));
  return RB_OK;  // the handle stays open: the communicator will use the same library
}

int rb_create_rank(int device, int rank, int world, const void* id, size_t len, rb_ctx** out,
                   char* err, size_t errlen) {
  if (world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, RB_E_INVALID, "rb_create_rank: bad rank/world", err, errlen);
  if (world > 1 && (!id || len < sizeof(ncclUniqueId)))
    return fail(nullptr, RB_E_INVALID, "rb_create_rank: missing ncclUniqueId", err, errlen);
  if (id && len < sizeof(ncclUniqueId))
    return fail(nullptr, RB_E_INVALID, "rb_create_rank: ncclUniqueId too short", err, errlen);
  if (int rc = make_ctx(&device, 1, out, err, errlen)) return rc;
  rb_ctx* ctx = *out;
  ctx->rank = rank;
  ctx->world = world;
  // A communicator whenever an id is given, also for a one-rank job: the rank-mode
  // exchange then runs against the real NCCL on a single GPU (nothing waits on
  // another rank), which is how the collective calls are exercised on this pool.
  if (world > 1 || id) {
    std::string msg;
    if (!ctx->nccl.load(msg)) {
      *out = nullptr;
      destroy_ctx(ctx);
      return fail(nullptr, RB_E_CUDA, msg, err, errlen);
    }
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ctx->comms.assign(1, nullptr);
    cudaSetDevice(device);
    const ncclResult_t r = ctx->nccl.init_rank(&ctx->comms[0], world, u, rank);
    if (r == ncclSuccess) ctx->rank_mode = true;
    if (r != ncclSuccess) {
      ctx->comms.clear();
      *out = nullptr;
      destroy_ctx(ctx);
      return fail(nullptr, RB_E_CUDA,
                  "rb_create_rank: ncclCommInitRank failed (NCCL error " + std::to_string(r) + ")",
                  err, errlen);
    }
  }
  return RB_OK;
}

int rb_comm_info(const rb_ctx* ctx, int* rank, int* world, int* comm_ranks, int* nccl_version) {
  if (!ctx) return RB_E_INVALID;
  if (rank) *rank = ctx->rank;
  if (world) *world = ctx->world;
  int nr = 1, ver = 0;
  if (!ctx->comms.empty() && ctx->nccl.count) {
    ctx->nccl.count(ctx->comms[0], &nr);
    ctx->nccl.version(&ver);
  }
  if (comm_ranks) *comm_ranks = nr;
  if (nccl_version) *nccl_version = ver;
  return RB_OK;
}

void rb_destroy(rb_ctx* ctx) {
  if (ctx) destroy_ctx(ctx);
}

int rb_plan_reset(rb_ctx* ctx) {
  if (!ctx) return RB_E_INVALID;
  ctx->plan.valid = false;
  for (Device& d : ctx->devs) d.plan_on_device = false;
  return RB_OK;
}

void* rb_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void rb_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int rb_set_field_nodes(rb_ctx* ctx, const rb_field_desc* desc, const double* n, const double* gx,
                       const double* gy, const double* gz) {
  NvtxRange nvtx_("raybos set_field_nodes");
  if (!ctx) return RB_E_INVALID;
  if (int rc = check_field_desc(ctx, desc)) return rc;
  if (!n || !gx || !gy || !gz) return fail(ctx, RB_E_INVALID, "rb_set_field_nodes: NULL array");
  ctx->has_field = ctx->has_field64 = false;
  const size_t count = static_cast<size_t>(desc->nx) * desc->ny * desc->nz;
  const size_t chunk = std::min<size_t>(count, size_t(1) << 24);
  const int rc = for_each_device(ctx, [&](Device& dev) -> int {
    if (int rc = upload_grid(ctx, dev, count)) return rc;
    Buf stage;
    RB_CUDA(ctx, stage.ensure(4 * chunk * sizeof(double)));
    double* st = stage.as<double>();
    for (size_t off = 0; off < count; off += chunk) {
      const size_t m = std::min(chunk, count - off);
      const double* src[4] = {n + off, gx + off, gy + off, gz + off};
      for (int a = 0; a < 4; ++a)
        RB_CUDA(ctx, cudaMemcpyAsync(st + a * chunk, src[a], m * sizeof(double),
                                     cudaMemcpyHostToDevice, dev.stream));
      RB_CUDA(ctx, rbk::launch_pack_nodes(st, st + chunk, st + 2 * chunk, st + 3 * chunk,
                                          dev.grid + off, static_cast<int64_t>(m), dev.stream));
    }
    if (int rc = build_cell_table(ctx, dev, desc)) return rc;
    for (Buf& b : dev.f64) b.release();
    if (static_cast<long long>(count) <= RB_FP64_MAX_NODES) {
      const double* src[4] = {n, gx, gy, gz};
      for (int a = 0; a < 4; ++a) {
        RB_CUDA(ctx, dev.f64[a].ensure(count * sizeof(double)));
        RB_CUDA(ctx, cudaMemcpyAsync(dev.f64[a].p, src[a], count * sizeof(double),
                                     cudaMemcpyHostToDevice, dev.stream));
      }
    }
    RB_CUDA(ctx, cudaStreamSynchronize(dev.stream));
    set_l2_window(dev);
    return RB_OK;
  });
  if (rc) return drop_field(ctx, rc);
  set_box(ctx, desc);
  return RB_OK;
}

// GriddedField ctor (scene.cpp:53-92) on device from a device-resident density
// volume: the float4 grid, the cell table and (small grids) the FP64 nodes.
int build_from_device_rho(rb_ctx* ctx, Device& dev, const rb_field_desc* desc, Buf& drho,
                          double k) {
  const size_t count = static_cast<size_t>(desc->nx) * desc->ny * desc->nz;
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  RB_CUDA(ctx, rbk::launch_build_from_density(drho.as<float>(), desc->nx, desc->ny, desc->nz, k,
                                              d3(desc->spacing), dev.grid, 0, desc->nz,
                                              dev.stream));
  if (int rc = build_cell_table(ctx, dev, desc)) return rc;
  for (Buf& b : dev.f64) b.release();
  if (static_cast<long long>(count) <= RB_FP64_MAX_NODES) {
    for (Buf& b : dev.f64) RB_CUDA(ctx, b.ensure(count * sizeof(double)));
    RB_CUDA(ctx, rbk::launch_build_fp64(drho.as<float>(), desc->nx, desc->ny, desc->nz, k,
                                        d3(desc->spacing), dev.f64[0].as<double>(),
                                        dev.f64[1].as<double>(), dev.f64[2].as<double>(),
                                        dev.f64[3].as<double>(), dev.stream));
  }
  RB_CUDA(ctx, cudaStreamSynchronize(dev.stream));
  drho.release();
  set_l2_window(dev);
  return RB_OK;
}

bool valid_density(const float* rho, size_t n) {  // DensityVolume::validate, scene.cpp:30-33
  for (size_t q = 0; q < n; ++q)
    if (!std::isfinite(rho[q]) || rho[q] < 0.0f) return false;
  return true;
}

int rb_set_field_density(rb_ctx* ctx, const rb_field_desc* desc, const float* rho,
                         double gladstone_dale_k) {
  NvtxRange nvtx_("raybos set_field_density");
  if (!ctx) return RB_E_INVALID;
  if (int rc = check_field_desc(ctx, desc)) return rc;
  if (!rho) return fail(ctx, RB_E_INVALID, "rb_set_field_density: rho is NULL");
  if (gladstone_dale_k <= 0.0)
    return fail(ctx, RB_E_INVALID, "gladstone_dale: K must be positive");  // scene.cpp:18
  const size_t count = static_cast<size_t>(desc->nx) * desc->ny * desc->nz;
  if (!valid_density(rho, count))
    return fail(ctx, RB_E_INVALID, "DensityVolume: densities must be finite and >= 0");
  ctx->has_field = ctx->has_field64 = false;
  const int rc = for_each_device(ctx, [&](Device& dev) -> int {
    if (int rc = upload_grid(ctx, dev, count)) return rc;
    Buf drho;
    RB_CUDA(ctx, drho.ensure(count * sizeof(float)));
    RB_CUDA(ctx, cudaMemcpyAsync(drho.p, rho, count * sizeof(float), cudaMemcpyHostToDevice,
                                 dev.stream));
    return build_from_device_rho(ctx, dev, desc, drho, gladstone_dale_k);
  });
  if (rc) return drop_field(ctx, rc);
  set_box(ctx, desc);
  return RB_OK;
}

// load_density_volume (scene.cpp:212-240) streamed: the file is read in z-slabs
// into two pinned buffers, each copied to every device while the next is read,
// so host memory stays at two slabs whatever the volume size; the GriddedField
// ctor then runs on device.  Errors and their order follow the reference
// (open, header, dims/spacing, truncation, then DensityVolume::validate).
int rb_set_field_gvol(rb_ctx* ctx, const char* path, const double* z_center,
                      double gladstone_dale_k, int64_t slab_bytes, rb_field_desc* desc_out) {
  NvtxRange nvtx_("raybos set_field_gvol");
  if (!ctx) return RB_E_INVALID;
  if (!path) return fail(ctx, RB_E_INVALID, "rb_set_field_gvol: path is NULL");
  const std::string p(path);
  if (gladstone_dale_k <= 0.0)
    return fail(ctx, RB_E_INVALID, "gladstone_dale: K must be positive");
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(path, "rb"), &std::fclose);
  if (!f) return fail(ctx, RB_E_INVALID, "load_density_volume: cannot open " + p);
  std::string header;
  int ch;
  while ((ch = std::fgetc(f.get())) != EOF && ch != '\n') header.push_back(static_cast<char>(ch));
  if (header.empty() && ch == EOF)
    return fail(ctx, RB_E_INVALID, "load_density_volume: missing header in " + p);
  std::istringstream hs(header);
  std::string magic;
  rb_field_desc d{};
  hs >> magic >> d.nx >> d.ny >> d.nz >> d.spacing.x >> d.spacing.y >> d.spacing.z >> d.origin.x >>
      d.origin.y >> d.origin.z;
  if (!hs || magic != "GVOL1")
    return fail(ctx, RB_E_INVALID, "load_density_volume: malformed GVOL header in " + p);
  if (d.nx < 2 || d.ny < 2 || d.nz < 2 || d.spacing.x <= 0 || d.spacing.y <= 0 || d.spacing.z <= 0)
    return fail(ctx, RB_E_INVALID, "load_density_volume: invalid dims/spacing in " + p);
  if (z_center) {  // build_medium_volume (engine.cpp:33-37): recentre on (0, 0, z_center)
    // Aabb center of DensityVolume::bounds (scene.hpp:34-36, core.hpp:77), same op order
    const double hi[3] = {d.origin.x + (d.nx - 1) * d.spacing.x, d.origin.y + (d.ny - 1) * d.spacing.y,
                          d.origin.z + (d.nz - 1) * d.spacing.z};
    const double c[3] = {(d.origin.x + hi[0]) * 0.5, (d.origin.y + hi[1]) * 0.5,
                         (d.origin.z + hi[2]) * 0.5};
    d.origin.x += 0.0 - c[0];
    d.origin.y += 0.0 - c[1];
    d.origin.z += *z_center - c[2];
  }
  if (int rc = check_field_desc(ctx, &d)) return rc;
  ctx->has_field = ctx->has_field64 = false;  // the old grid goes now
  const size_t plane = static_cast<size_t>(d.nx) * d.ny;
  const size_t count = plane * d.nz;
  const size_t want = slab_bytes > 0 ? static_cast<size_t>(slab_bytes) : (size_t(64) << 20);
  const size_t planes = std::max<size_t>(1, std::min<size_t>(d.nz, want / (plane * 4)));
  std::vector<Buf> drho(ctx->devs.size());
  // every early return below releases drho (RAII) and the half-built grids
  struct DropOnError {
    rb_ctx* ctx;
    bool armed = true;
    ~DropOnError() {
      if (armed) drop_field(ctx, 0);
    }
  } drop_guard{ctx};
  for (size_t i = 0; i < ctx->devs.size(); ++i) {
    if (int rc = upload_grid(ctx, ctx->devs[i], count)) return rc;
    RB_CUDA(ctx, cudaSetDevice(ctx->devs[i].ordinal));
    RB_CUDA(ctx, drho[i].ensure(count * sizeof(float)));
  }
  float* pinned[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> done[2];
  struct Cleanup {
    float** p;
    std::vector<cudaEvent_t>* e;
    ~Cleanup() {
      for (int b = 0; b < 2; ++b) {
        for (cudaEvent_t x : e[b]) {
          cudaEventSynchronize(x);
          cudaEventDestroy(x);
        }
        if (p[b]) cudaFreeHost(p[b]);
      }
    }
  } cleanup{pinned, done};
  for (int b = 0; b < 2; ++b) {
    RB_CUDA(ctx, cudaHostAlloc(reinterpret_cast<void**>(&pinned[b]), planes * plane * sizeof(float),
                               cudaHostAllocPortable));
    for (Device& dev : ctx->devs) {
      RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
      cudaEvent_t e;
      RB_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      done[b].push_back(e);
    }
  }
  bool valid = true;
  bool used[2] = {false, false};
  int b = 0;
  for (size_t z0 = 0; z0 < static_cast<size_t>(d.nz); z0 += planes, b ^= 1) {
    const size_t nz = std::min(planes, static_cast<size_t>(d.nz) - z0);
    const size_t n = nz * plane;
    if (used[b])  // the copies out of this buffer must be done before refilling it
      for (cudaEvent_t e : done[b]) RB_CUDA(ctx, cudaEventSynchronize(e));
    if (std::fread(pinned[b], sizeof(float), n, f.get()) != n)
      return fail(ctx, RB_E_INVALID, "load_density_volume: truncated data in " + p);
    // GVOL data are little-endian float32, the host's own layout (x86-64 / aarch64)
    valid = valid && valid_density(pinned[b], n);
    for (size_t i = 0; i < ctx->devs.size(); ++i) {
      Device& dev = ctx->devs[i];
      RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
      RB_CUDA(ctx, cudaMemcpyAsync(drho[i].as<float>() + z0 * plane, pinned[b], n * sizeof(float),
                                   cudaMemcpyHostToDevice, dev.stream));
      RB_CUDA(ctx, cudaEventRecord(done[b][i], dev.stream));
    }
    used[b] = true;
  }
  if (!valid) return fail(ctx, RB_E_INVALID, "DensityVolume: densities must be finite and >= 0");
  if (int rc = for_each_device(ctx, [&](Device& dev) -> int {
        const size_t i = static_cast<size_t>(&dev - ctx->devs.data());
        return build_from_device_rho(ctx, dev, &d, drho[i], gladstone_dale_k);
      }))
    return rc;
  drop_guard.armed = false;
  set_box(ctx, &d);
  if (desc_out) *desc_out = d;
  return RB_OK;
}

int rb_clear_field(rb_ctx* ctx) {
  if (!ctx) return RB_E_INVALID;
  for (Device& dev : ctx->devs) {
    free_field(dev);
    set_l2_window(dev);  // no field: clears the stream's access-policy window
    for (Buf& b : dev.f64) b.release();
  }
  ctx->has_field = false;
  ctx->has_field64 = false;
  return RB_OK;
}

int64_t rb_field_bytes(const rb_ctx* ctx) {
  return (ctx && !ctx->devs.empty())
             ? static_cast<int64_t>(ctx->devs[0].grid_bytes + ctx->devs[0].cells_bytes)
             : 0;
}

int rb_trace(rb_ctx* ctx, const rb_scene* s, int with_field, int accumulate_image,
             rb_trace_out* out) {
  NvtxRange nvtx_("raybos rb_trace");
  if (!ctx || !out) return RB_E_INVALID;
  const auto t0 = std::chrono::steady_clock::now();
  if (int rc = validate_scene(ctx, s)) return rc;
  if (accumulate_image && out->quantized) {  // quantize's own checks, sensor.cpp:126-129
    const int b = out->bit_depth;
    if (b != 8 && b != 10 && b != 12 && b != 16)
      return fail(ctx, RB_E_INVALID, "quantize: bit depth must be one of 8, 10, 12, 16");
    if (!(out->gain > 0.0)) return fail(ctx, RB_E_INVALID, "quantize: gain must be positive");
  }
  const int W = s->sensor.width_px, H = s->sensor.height_px;
  const size_t npx = static_cast<size_t>(W) * H;
  const int total = static_cast<int>(ctx->devs.size()) * ctx->world;
  const bool root = ctx->rank == 0;  // the image lands on rank 0, device 0
  out->kernel_ms = 0.0;
  out->kernel_launches = 0;
  out->k1_kernel = 0;
  if (s->n_sources == 0) {  // engine.cpp:436: one "thread", blank image, no stats
    if (accumulate_image && root) {
      if (out->image) std::memset(out->image, 0, npx * sizeof(double));
      if (out->quantized) std::memset(out->quantized, 0, npx * sizeof(uint16_t));
      if (out->image_fixed) {
        RB_CUDA(ctx, cudaSetDevice(ctx->devs[0].ordinal));
        RB_CUDA(ctx, cudaMemset(out->image_fixed, 0, npx * sizeof(uint64_t)));
      }
    }
    const unsigned long long zero[6] = {0, 0, 0, 0, 0, 0};
    fill_report(out, s, 0, zero, 0);
    out->threads = 1;
    out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return RB_OK;
  }
  const rbk::KScene base = make_kscene(ctx, s, with_field, accumulate_image);
  std::vector<std::vector<int32_t>> work;
  std::vector<PartialOut> parts;
  int tail_launches = 0;
  // the image tail on device 0, queued before the stats readback's stream sync
  auto tail = [&](Device& d0) -> int {
    if (!(accumulate_image && (out->image || out->quantized || out->image_fixed))) return RB_OK;
    RB_CUDA(ctx, cudaSetDevice(d0.ordinal));
    if (out->image_fixed)  // device-resident result: the reduced fixed-point image
      RB_CUDA(ctx, cudaMemcpyAsync(out->image_fixed, d0.image.p, npx * sizeof(uint64_t),
                                   cudaMemcpyDeviceToDevice, d0.stream));
    if (out->image || out->quantized) {
      RB_CUDA(ctx, d0.dimage.ensure(npx * sizeof(double)));
      RB_CUDA(ctx, rbk::launch_image_finalize(d0.image.as<unsigned long long>(),
                                              d0.dimage.as<double>(), static_cast<int64_t>(npx),
                                              d0.stream));
      ++tail_launches;
      if (out->image)
        RB_CUDA(ctx, cudaMemcpyAsync(out->image, d0.dimage.p, npx * sizeof(double),
                                     cudaMemcpyDeviceToHost, d0.stream));
      if (out->quantized) {  // render's quantize on device (sensor.cpp:124-135)
        RB_CUDA(ctx, d0.qimage.ensure(npx * sizeof(uint16_t)));
        RB_CUDA(ctx, rbk::launch_quantize(d0.dimage.as<double>(), static_cast<int64_t>(npx),
                                          out->gain, out->bit_depth, d0.qimage.as<uint16_t>(),
                                          d0.stream));
        ++tail_launches;
        RB_CUDA(ctx, cudaMemcpyAsync(out->quantized, d0.qimage.p, npx * sizeof(uint16_t),
                                     cudaMemcpyDeviceToHost, d0.stream));
      }
    }
    return RB_OK;
  };
  if (int rc = run_shards(ctx, s, base, work, parts, tail)) return rc;
  unsigned long long c[6];
  int64_t landed_total = 0;
  merge_stats(ctx, s, work, parts, false, out->hit_sum, out->landed, c, landed_total);
  float ms = 0.f;
  int launches = tail_launches;
  int k1 = 0;
  for (const PartialOut& po : parts) {
    ms = std::max(ms, po.ms);
    launches += po.launches;
    k1 = std::max(k1, po.k1);
  }
  fill_report(out, s, s->n_sources, c, landed_total);
  out->threads = total;
  out->k1_kernel = k1;
  out->kernel_ms = ms;
  out->kernel_launches = launches;
  out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return RB_OK;
}

int rb_trace_shard(rb_ctx* ctx, const rb_scene* s, int with_field, int accumulate_image,
                   int64_t shard_index, int64_t shard_count, uint64_t* image_fixed,
                   rb_trace_out* out) {
  if (!ctx || !out) return RB_E_INVALID;
  const auto t0 = std::chrono::steady_clock::now();
  if (shard_count < 1 || shard_index < 0 || shard_index >= shard_count)
    return fail(ctx, RB_E_INVALID, "rb_trace_shard: bad shard index/count");
  if (int rc = validate_scene(ctx, s)) return rc;
  const unsigned long long zero[6] = {0, 0, 0, 0, 0, 0};
  out->threads = 1;
  out->k1_kernel = 0;
  if (s->n_sources == 0) {
    fill_report(out, s, 0, zero, 0);
    return RB_OK;
  }
  if (accumulate_image && !image_fixed)
    return fail(ctx, RB_E_INVALID, "rb_trace_shard: image_fixed (device) required");
  const rbk::KScene base = make_kscene(ctx, s, with_field, accumulate_image);
  const std::vector<int32_t> work = shard_list(zorder(s), shard_index, shard_count);
  PartialOut po;
  if (int rc = render_on(ctx, ctx->devs[0], s, base, work, reinterpret_cast<unsigned long long*>(image_fixed), po))
    return rc;
  if (int rc = check_error(ctx, po.check_fail)) return rc;
  if (po.err_flag) return flag_error(ctx, po.err_flag, s);
  int64_t landed_total = 0;
  for (int32_t src : work) {
    if (out->hit_sum) {
      out->hit_sum[2 * src] = po.hit[2 * src];
      out->hit_sum[2 * src + 1] = po.hit[2 * src + 1];
    }
    if (out->landed) out->landed[src] = po.landed[src];
    landed_total += po.landed[src];
  }
  fill_report(out, s, static_cast<int64_t>(work.size()), po.counters, landed_total);
  out->kernel_ms = po.ms;
  out->kernel_launches = po.launches;
  out->k1_kernel = po.k1;
  out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return RB_OK;
}

int rb_plan_shards(const rb_scene* s, int64_t shard_count, int32_t* shard_of_source) {
  if (!s || !shard_of_source || shard_count < 1 || s->n_sources < 0) return RB_E_INVALID;
  if (s->n_sources > 0 && !s->sources) return RB_E_INVALID;
  const std::vector<int32_t> z = zorder(s);
  for (size_t p = 0; p < z.size(); ++p)
    shard_of_source[z[p]] = static_cast<int32_t>((static_cast<int64_t>(p) / kShardTile) % shard_count);
  return RB_OK;
}

int rb_image_from_fixed(rb_ctx* ctx, const uint64_t* image_fixed_device, int64_t n_pixels,
                        double* image_host) {
  if (!ctx || !image_fixed_device || !image_host || n_pixels < 0) return RB_E_INVALID;
  Device& d0 = ctx->devs[0];
  RB_CUDA(ctx, cudaSetDevice(d0.ordinal));
  RB_CUDA(ctx, d0.dimage.ensure(static_cast<size_t>(n_pixels) * sizeof(double)));
  RB_CUDA(ctx, join_default_stream(d0));
  RB_CUDA(ctx, rbk::launch_image_finalize(reinterpret_cast<const unsigned long long*>(image_fixed_device),
                                          d0.dimage.as<double>(), n_pixels, d0.stream));
  RB_CUDA(ctx, cudaMemcpyAsync(image_host, d0.dimage.p, static_cast<size_t>(n_pixels) * sizeof(double),
                               cudaMemcpyDeviceToHost, d0.stream));
  RB_CUDA(ctx, cudaStreamSynchronize(d0.stream));
  return RB_OK;
}

int rb_trace_rays(rb_ctx* ctx, const rb_scene* s, int with_field, int64_t n_rays,
                  const int64_t* source_index, const int32_t* ray_index, double* uv,
                  int32_t* status, int32_t* steps) {
  if (!ctx) return RB_E_INVALID;
  if (int rc = validate_scene(ctx, s)) return rc;
  if (n_rays <= 0) return RB_OK;
  for (int64_t q = 0; q < n_rays; ++q)
    if (source_index[q] < 0 || source_index[q] >= s->n_sources || ray_index[q] < 0 ||
        ray_index[q] >= s->rays_per_source)
      return fail(ctx, RB_E_INVALID, "rb_trace_rays: (source, ray) index out of range");
  Device& dev = ctx->devs[0];
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  rbk::KScene k = make_kscene(ctx, s, with_field, 0);
  const int64_t n = s->n_sources;
  cudaStream_t st = dev.stream;
  RB_CUDA(ctx, dev.sources.ensure(sizeof(double) * 3 * n));
  RB_CUDA(ctx, cudaMemcpyAsync(dev.sources.p, s->sources, sizeof(double) * 3 * n,
                               cudaMemcpyHostToDevice, st));
  k.sources = dev.sources.as<double>();
  if (s->source_ids) {
    RB_CUDA(ctx, dev.ids.ensure(sizeof(int64_t) * n));
    RB_CUDA(ctx, cudaMemcpyAsync(dev.ids.p, s->source_ids, sizeof(int64_t) * n,
                                 cudaMemcpyHostToDevice, st));
    k.source_ids = dev.ids.as<int64_t>();
  }
  k.grid = dev.grid;
  k.cell_table = dev.cells;
  RB_CUDA(ctx, dev.queue.ensure(sizeof(int) * 4));
  RB_CUDA(ctx, cudaMemsetAsync(dev.queue.p, 0, sizeof(int) * 4, st));
  k.err_flag = dev.queue.as<int>() + 1;
  k.check_fail = reinterpret_cast<unsigned*>(dev.queue.as<int>() + 2);
  RB_CUDA(ctx, dev.rays_src.ensure(sizeof(int64_t) * n_rays));
  RB_CUDA(ctx, dev.rays_idx.ensure(sizeof(int32_t) * n_rays));
  RB_CUDA(ctx, dev.rays_uv.ensure(sizeof(double) * 2 * n_rays));
  RB_CUDA(ctx, dev.rays_status.ensure(sizeof(int32_t) * n_rays));
  RB_CUDA(ctx, dev.rays_steps.ensure(sizeof(int32_t) * n_rays));
  RB_CUDA(ctx, cudaMemcpyAsync(dev.rays_src.p, source_index, sizeof(int64_t) * n_rays,
                               cudaMemcpyHostToDevice, st));
  RB_CUDA(ctx, cudaMemcpyAsync(dev.rays_idx.p, ray_index, sizeof(int32_t) * n_rays,
                               cudaMemcpyHostToDevice, st));
  RB_CUDA(ctx, rbk::launch_trace_rays(k, n_rays, dev.rays_src.as<int64_t>(),
                                      dev.rays_idx.as<int32_t>(), dev.rays_uv.as<double>(),
                                      dev.rays_status.as<int32_t>(), dev.rays_steps.as<int32_t>(),
                                      st));
  RB_CUDA(ctx, cudaMemcpyAsync(uv, dev.rays_uv.p, sizeof(double) * 2 * n_rays,
                               cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(status, dev.rays_status.p, sizeof(int32_t) * n_rays,
                               cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(steps, dev.rays_steps.p, sizeof(int32_t) * n_rays,
                               cudaMemcpyDeviceToHost, st));
  int flag = 0;
  unsigned cf[2] = {0, 0};
  RB_CUDA(ctx, cudaMemcpyAsync(&flag, k.err_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(cf, k.check_fail, sizeof(cf), cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaStreamSynchronize(st));
  if (int rc = check_error(ctx, cf)) return rc;
  if (flag) return flag_error(ctx, flag, s);
  return RB_OK;
}

}  // extern "C"


// ---- FP64 validation build ------------------------------------------------
namespace {

int upload_scene_arrays(rb_ctx* ctx, Device& dev, const rb_scene* s, rbk::KScene& k) {
  const int64_t n = s->n_sources;
  RB_CUDA(ctx, dev.sources.ensure(sizeof(double) * 3 * std::max<int64_t>(n, 1)));
  if (n)
    RB_CUDA(ctx, cudaMemcpyAsync(dev.sources.p, s->sources, sizeof(double) * 3 * n,
                                 cudaMemcpyHostToDevice, dev.stream));
  k.sources = dev.sources.as<double>();
  k.source_ids = nullptr;
  if (s->source_ids && n) {
    RB_CUDA(ctx, dev.ids.ensure(sizeof(int64_t) * n));
    RB_CUDA(ctx, cudaMemcpyAsync(dev.ids.p, s->source_ids, sizeof(int64_t) * n,
                                 cudaMemcpyHostToDevice, dev.stream));
    k.source_ids = dev.ids.as<int64_t>();
  }
  RB_CUDA(ctx, dev.queue.ensure(sizeof(int) * 2));
  RB_CUDA(ctx, cudaMemsetAsync(dev.queue.p, 0, sizeof(int) * 2, dev.stream));
  k.err_flag = dev.queue.as<int>() + 1;
  return RB_OK;
}

int field64(rb_ctx* ctx, const Device& dev, int with_field, rbk::Field64& f) {
  f = rbk::Field64{};
  if (!(with_field && ctx->has_field)) return RB_OK;
  if (!ctx->has_field64 || !dev.f64[0].p)
    return fail(ctx, RB_E_INVALID, "rb_*_fp64: the FP64 validation build needs a grid of at most "
                                   "2^26 nodes");
  f.n = dev.f64[0].as<double>();
  f.gx = dev.f64[1].as<double>();
  f.gy = dev.f64[2].as<double>();
  f.gz = dev.f64[3].as<double>();
  f.nx = ctx->field.nx;
  f.ny = ctx->field.ny;
  f.nz = ctx->field.nz;
  f.origin = d3(ctx->field.origin);
  f.spacing = d3(ctx->field.spacing);
  f.lo = ctx->box_lo;
  f.hi = ctx->box_hi;
  return RB_OK;
}

}  // namespace

extern "C" int rb_trace_rays_fp64(rb_ctx* ctx, const rb_scene* s, int with_field, int64_t n_rays,
                                  const int64_t* source_index, const int32_t* ray_index,
                                  double* uv, int32_t* status, int32_t* steps) {
  if (!ctx) return RB_E_INVALID;
  if (int rc = validate_scene(ctx, s)) return rc;
  if (n_rays <= 0) return RB_OK;
  for (int64_t q = 0; q < n_rays; ++q)
    if (source_index[q] < 0 || source_index[q] >= s->n_sources || ray_index[q] < 0 ||
        ray_index[q] >= s->rays_per_source)
      return fail(ctx, RB_E_INVALID, "rb_trace_rays_fp64: (source, ray) index out of range");
  Device& dev = ctx->devs[0];
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  rbk::KScene k = make_kscene(ctx, s, with_field, 0);
  rbk::Field64 f;
  if (int rc = field64(ctx, dev, with_field, f)) return rc;
  if (int rc = upload_scene_arrays(ctx, dev, s, k)) return rc;
  cudaStream_t st = dev.stream;
  RB_CUDA(ctx, dev.rays_src.ensure(sizeof(int64_t) * n_rays));
  RB_CUDA(ctx, dev.rays_idx.ensure(sizeof(int32_t) * n_rays));
  RB_CUDA(ctx, dev.rays_uv.ensure(sizeof(double) * 2 * n_rays));
  RB_CUDA(ctx, dev.rays_status.ensure(sizeof(int32_t) * n_rays));
  RB_CUDA(ctx, dev.rays_steps.ensure(sizeof(int32_t) * n_rays));
  RB_CUDA(ctx, cudaMemcpyAsync(dev.rays_src.p, source_index, sizeof(int64_t) * n_rays,
                               cudaMemcpyHostToDevice, st));
  RB_CUDA(ctx, cudaMemcpyAsync(dev.rays_idx.p, ray_index, sizeof(int32_t) * n_rays,
                               cudaMemcpyHostToDevice, st));
  RB_CUDA(ctx, rbk::launch_trace_rays_fp64(k, f, n_rays, dev.rays_src.as<int64_t>(),
                                           dev.rays_idx.as<int32_t>(), dev.rays_uv.as<double>(),
                                           dev.rays_status.as<int32_t>(),
                                           dev.rays_steps.as<int32_t>(), st));
  RB_CUDA(ctx, cudaMemcpyAsync(uv, dev.rays_uv.p, sizeof(double) * 2 * n_rays,
                               cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(status, dev.rays_status.p, sizeof(int32_t) * n_rays,
                               cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(steps, dev.rays_steps.p, sizeof(int32_t) * n_rays,
                               cudaMemcpyDeviceToHost, st));
  int flag = 0;
  RB_CUDA(ctx, cudaMemcpyAsync(&flag, k.err_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaStreamSynchronize(st));
  if (flag) return flag_error(ctx, flag, s);
  return RB_OK;
}

extern "C" int rb_trace_stats_fp64(rb_ctx* ctx, const rb_scene* s, int with_field,
                                   rb_trace_out* out) {
  if (!ctx || !out) return RB_E_INVALID;
  const auto t0 = std::chrono::steady_clock::now();
  if (int rc = validate_scene(ctx, s)) return rc;
  const unsigned long long zero[6] = {0, 0, 0, 0, 0, 0};
  out->threads = 1;
  out->k1_kernel = 0;
  out->kernel_ms = 0.0;
  if (s->n_sources == 0) {
    fill_report(out, s, 0, zero, 0);
    return RB_OK;
  }
  Device& dev = ctx->devs[0];
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  rbk::KScene k = make_kscene(ctx, s, with_field, 0);
  rbk::Field64 f;
  if (int rc = field64(ctx, dev, with_field, f)) return rc;
  if (int rc = upload_scene_arrays(ctx, dev, s, k)) return rc;
  const int64_t n = s->n_sources;
  cudaStream_t st = dev.stream;
  RB_CUDA(ctx, dev.hit.ensure(sizeof(double) * 2 * n));
  RB_CUDA(ctx, dev.landed.ensure(sizeof(long long) * n));
  RB_CUDA(ctx, dev.counters.ensure(sizeof(unsigned long long) * 8));
  RB_CUDA(ctx, cudaMemsetAsync(dev.counters.p, 0, sizeof(unsigned long long) * 8, st));
  k.hit_sum = dev.hit.as<double>();
  k.landed = dev.landed.as<long long>();
  k.counters = dev.counters.as<unsigned long long>();
  RB_CUDA(ctx, rbk::launch_source_stats_fp64(k, f, st));
  std::vector<double> hit(2 * n);
  std::vector<long long> landed(n);
  unsigned long long c[6];
  int flag = 0;
  RB_CUDA(ctx, cudaMemcpyAsync(hit.data(), dev.hit.p, sizeof(double) * 2 * n,
                               cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(landed.data(), dev.landed.p, sizeof(long long) * n,
                               cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(c, dev.counters.p, sizeof(c), cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaMemcpyAsync(&flag, k.err_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  RB_CUDA(ctx, cudaStreamSynchronize(st));
  if (flag) return fail(ctx, RB_E_INVALID, "emit_rays: source coincides with aperture point");
  int64_t landed_total = 0;
  for (int64_t q = 0; q < n; ++q) {
    if (out->hit_sum) {
      out->hit_sum[2 * q] = hit[2 * q];
      out->hit_sum[2 * q + 1] = hit[2 * q + 1];
    }
    if (out->landed) out->landed[q] = landed[q];
    landed_total += landed[q];
  }
  fill_report(out, s, n, c, landed_total);
  out->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return RB_OK;
}

extern "C" int rb_trace_debug(rb_ctx* ctx, const rb_scene* s, int64_t source_index,
                              int32_t ray_index, double* records, int64_t max_records,
                              int64_t* n_records) {
  if (!ctx || !n_records) return RB_E_INVALID;
  if (int rc = validate_scene(ctx, s)) return rc;
  // the reference's own checks, engine.cpp:607-612
  if (!ctx->has_field) return fail(ctx, RB_E_RUNTIME, "trace_debug: config has no density field");
  if (source_index < 0 || source_index >= s->n_sources)
    return fail(ctx, RB_E_RUNTIME, "trace_debug: dot index out of range");
  if (ray_index < 0 || ray_index >= s->rays_per_source)
    return fail(ctx, RB_E_RUNTIME, "trace_debug: ray index out of range");
  if (max_records < 0 || (max_records > 0 && !records)) return RB_E_INVALID;
  Device& dev = ctx->devs[0];
  RB_CUDA(ctx, cudaSetDevice(dev.ordinal));
  rbk::KScene k = make_kscene(ctx, s, 1, 0);
  rbk::Field64 f;
  if (int rc = field64(ctx, dev, 1, f)) return rc;
  if (int rc = upload_scene_arrays(ctx, dev, s, k)) return rc;
  RB_CUDA(ctx, dev.dbg.ensure(sizeof(double) * 7 * std::max<int64_t>(max_records, 1)));
  RB_CUDA(ctx, dev.dbg_n.ensure(sizeof(int64_t)));
  RB_CUDA(ctx, rbk::launch_trace_debug(k, f, source_index, ray_index, dev.dbg.as<double>(),
                                       max_records, dev.dbg_n.as<int64_t>(), dev.stream));
  int64_t n = 0;
  RB_CUDA(ctx, cudaMemcpyAsync(&n, dev.dbg_n.p, sizeof(int64_t), cudaMemcpyDeviceToHost, dev.stream));
  RB_CUDA(ctx, cudaStreamSynchronize(dev.stream));
  const int64_t w = std::min(n, max_records);
  if (w > 0)
    RB_CUDA(ctx, cudaMemcpy(records, dev.dbg.p, sizeof(double) * 7 * w, cudaMemcpyDeviceToHost));
  *n_records = n;
  return RB_OK;
}

extern "C" int rb_trace_bos_pair(rb_ctx* ctx, const rb_scene* s, rb_trace_out* out_ref,
                                 rb_trace_out* out_grad) {
  NvtxRange nvtx_("raybos rb_trace_bos_pair");
  if (!ctx || !out_ref || !out_grad) return RB_E_INVALID;
  const auto t0 = std::chrono::steady_clock::now();
  if (int rc = validate_scene(ctx, s)) return rc;
  if (!ctx->has_field) return fail(ctx, RB_E_RUNTIME, "bos_run: config must include a density field");
  const unsigned long long zero[6] = {0, 0, 0, 0, 0, 0};
  if (s->n_sources == 0) {
    fill_report(out_ref, s, 0, zero, 0);
    fill_report(out_grad, s, 0, zero, 0);
    out_ref->threads = out_grad->threads = 1;
    return RB_OK;
  }
  // With the cell table the field kernel runs at 3 CTAs/SM and the fused pair
  // kernel (which must also hold the reference leg) at 2: two passes are then
  // faster (bos 1e7 rays: 40.3 ms vs 43.7 ms fused; the no-field pass is <1%).
  // On the node grid both run at 2 CTAs/SM and fusing saves the second raygen.
  std::vector<std::vector<int32_t>> work;
  std::vector<PartialOut> parts, ref;
  unsigned long long c[6], c0[6];
  int64_t lt = 0, lt0 = 0;
  if (ctx->devs[0].cells) {
    std::vector<std::vector<int32_t>> work0;
    if (int rc = run_shards(ctx, s, make_kscene(ctx, s, 0, 0), work0, ref)) return rc;
    if (int rc = run_shards(ctx, s, make_kscene(ctx, s, 1, 0), work, parts)) return rc;
    merge_stats(ctx, s, work0, ref, false, out_ref->hit_sum, out_ref->landed, c0, lt0);
    merge_stats(ctx, s, work, parts, false, out_grad->hit_sum, out_grad->landed, c, lt);
  } else {
    rbk::KScene base = make_kscene(ctx, s, 1, 0);
    base.pair = 1;
    if (int rc = run_shards(ctx, s, base, work, parts)) return rc;
    merge_stats(ctx, s, work, parts, true, out_ref->hit_sum, out_ref->landed, c0, lt0);
    merge_stats(ctx, s, work, parts, false, out_grad->hit_sum, out_grad->landed, c, lt);
  }
  float ms = 0.f;
  int launches = 0;
  for (size_t d = 0; d < parts.size(); ++d) {
    ms = std::max(ms, parts[d].ms + (ref.empty() ? 0.f : ref[d].ms));
    launches += parts[d].launches + (ref.empty() ? 0 : ref[d].launches);
  }
  c0[5] = 0;  // no RK4 steps on the reference leg
  fill_report(out_grad, s, s->n_sources, c, lt);
  fill_report(out_ref, s, s->n_sources, c0, lt0);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  out_ref->threads = out_grad->threads = static_cast<int>(ctx->devs.size()) * ctx->world;
  out_ref->kernel_ms = out_grad->kernel_ms = ms;
  out_ref->kernel_launches = out_grad->kernel_launches = launches;
  out_ref->k1_kernel = out_grad->k1_kernel = 1;
  out_ref->wall_seconds = out_grad->wall_seconds = wall;
  return RB_OK;
}
