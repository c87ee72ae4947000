/*
 * raybos_gpu.h — C-ABI of the B200-native per-ray rendering pipeline.
 *
 * This is the drop-in boundary for the reference's hot path
 *
 *     TraceOutputs raybos::run_trace(const SceneSetup& setup, bool with_field,
 *                                    bool accumulate_image, const RunConfig& run);
 *     (reference: proj/include/raybos/engine.hpp:73-78, proj/src/engine.cpp:429-507)
 *
 * The reference has no plugin registry; run_trace is the seam.  Everything it
 * reads from SceneSetup (engine.hpp:40-60) is flattened into the POD structs
 * below (plain pointers and sizes, no C++ or torch types), and everything it
 * returns in TraceOutputs (engine.hpp:67-71: per-source DotHitStats, RunReport,
 * ImageBuffer) is written into caller-owned buffers of rb_trace_out.
 *
 * Conventions
 *  - All entry points return 0 on success and a non-zero RB_E_* code on failure;
 *    the message is copied into the context (rb_last_error) and, when given, into
 *    err/errlen.  Nothing throws across the ABI.  The messages for invalid scenes
 *    are the reference's own exception texts (raygen.cpp:29-31, raygen.cpp:69).
 *  - Caller owns every host buffer; the context owns device memory.  The density
 *    grid persists in the context across rb_trace calls (bos_run traces the same
 *    scene twice, engine.cpp:539-540).
 *  - An rb_ctx is not thread-safe: one caller at a time (the reference's
 *    run_trace is a synchronous call too).
 *  - There is no CPU fallback: rb_create fails when no sm_100 device is present.
 */
#ifndef RAYBOS_GPU_H_
#define RAYBOS_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RB_ABI_VERSION 2

/* ---- status codes ------------------------------------------------------- */
#define RB_OK 0
#define RB_E_INVALID 1   /* std::invalid_argument in the reference            */
#define RB_E_RUNTIME 2   /* std::runtime_error in the reference               */
#define RB_E_CUDA 3      /* CUDA / NCCL failure                                */
#define RB_E_NODEVICE 4  /* no usable sm_100 device                            */

/* ---- per-ray outcome codes (rb_trace_rays) ------------------------------ */
/* Mirrors the counter mapping of process_source, engine.cpp:112-137.        */
#define RB_RAY_LANDED 0
#define RB_RAY_LOST 1           /* TraceStatus kLost or kInvalid (grin.hpp:49-54) */
#define RB_RAY_APERTURE 2       /* BlockReason kApertureStop                    */
#define RB_RAY_MISSED 3         /* BlockReason kMissedElement                   */
#define RB_RAY_TIR 4            /* BlockReason kTotalInternalReflection         */
#define RB_RAY_SENSOR_MISS 5    /* intersect_sensor returned nullopt            */

/* ---- scene ------------------------------------------------------------- */
typedef struct rb_vec3 {
  double x, y, z;
} rb_vec3;

/* raybos::OpticalElement alternatives (optics.hpp:100). */
#define RB_ELEM_APERTURE 0   /* raybos::Aperture        optics.hpp:80-84  */
#define RB_ELEM_SINGLET 1    /* raybos::LensElement     optics.hpp:45-52  */
#define RB_ELEM_THIN_LENS 2  /* raybos::ThinLensIdeal   optics.hpp:88-93  */
#define RB_ELEM_MIRROR 3     /* raybos::Mirror          optics.hpp:84-86  */

/* raybos::SphericalSurface (optics.hpp:26-36).  curvature_radius = +inf
 * (or any non-finite value) marks a plane. */
typedef struct rb_surface {
  rb_vec3 vertex;
  rb_vec3 axis;
  double curvature_radius;
  double aperture_radius;
  double n_before;
  double n_after;
} rb_surface;

typedef struct rb_element {
  int32_t kind; /* RB_ELEM_* */
  int32_t reserved;
  /* aperture: center, axis = normal, radius.
   * thin lens: center, axis, focal_length, diameter. */
  rb_vec3 center;
  rb_vec3 axis;
  double radius;
  double focal_length;
  double diameter;
  /* singlet: front, back.  mirror: front. */
  rb_surface front;
  rb_surface back;
} rb_element;

/* raybos::SensorModel (sensor.hpp:19-32); bit_depth and gain are not read by
 * run_trace (they are used by quantize on the host). */
typedef struct rb_sensor {
  rb_vec3 center;
  rb_vec3 normal;
  rb_vec3 e_u;
  rb_vec3 e_v;
  int32_t width_px;
  int32_t height_px;
  double pitch;
  double window_sigmas;
} rb_sensor;

#define RB_SAMPLING_STRATIFIED 0 /* ApertureSampling::kStratified   */
#define RB_SAMPLING_UNIFORM 1    /* ApertureSampling::kUniformRandom */

/* The parts of raybos::SceneSetup (engine.hpp:40-60) run_trace reads. */
typedef struct rb_scene {
  const rb_vec3* sources; /* SceneSetup::sources                               */
  int64_t n_sources;
  /* Optional RNG stream id per source; NULL means "index in sources", which is
   * what run_trace uses (engine.cpp:459).  Lets a caller trace a subset of a
   * scene, or the gain-calibration dot (stream 0xca1, engine.cpp:25,405),
   * with the reference's ray set. */
  const int64_t* source_ids;
  rb_vec3 pupil_center; /* SceneSetup::pupil (raygen.hpp:32-36)             */
  rb_vec3 pupil_axis;
  double pupil_radius;
  int32_t rays_per_source; /* SceneSetup::bundle (raygen.hpp:24-28)          */
  int32_t sampling;
  uint64_t seed;
  double wavelength;
  double delta_xi; /* SceneSetup::step (grin.hpp:23-26)                       */
  int32_t max_steps;
  int32_t n_elements;
  const rb_element* elements; /* SceneSetup::elements, in order              */
  rb_sensor sensor;
  double d_tau;
  uint64_t config_hash; /* copied into the report                             */
} rb_scene;

/* Geometry of the density grid (GriddedField, scene.hpp:68-105): node
 * (i,j,k) sits at origin + (i*dx, j*dy, k*dz), x-fastest storage. */
typedef struct rb_field_desc {
  int32_t nx, ny, nz;
  int32_t reserved;
  rb_vec3 origin;
  rb_vec3 spacing;
} rb_field_desc;

/* Everything TraceOutputs + RunReport carry (engine.hpp:19-36, 67-71). */
typedef struct rb_trace_out {
  /* caller-owned, may be NULL */
  double* hit_sum; /* [2*n_sources]  DotHitStats::hit_sum (u, v) in metres   */
  int64_t* landed; /* [n_sources]    DotHitStats::landed                      */
  double* image;   /* [W*H] ImageBuffer::data, row 0 = top; only written when
                      accumulate_image != 0                                    */
  /* RunReport */
  int64_t emitted;
  int64_t landed_total;
  int64_t lost;
  int64_t blocked_aperture;
  int64_t blocked_miss;
  int64_t blocked_tir;
  int64_t blocked_sensor_miss;
  double wall_seconds;
  int32_t threads; /* devices used (RunReport::threads)                         */
  int32_t k1_kernel; /* out: the render kernel that ran: 1 render_emitters, 2 render_warps
                        (0: no sources, or rb_trace_stats_fp64's validation kernel) */
  uint64_t config_hash;
  /* instrumentation (not in the reference report) */
  int64_t total_steps;     /* sum of RK4 steps over all rays                   */
  double kernel_ms;        /* device time of the render kernel(s), max over devices */
  /* optional render tail on device (render, engine.cpp:513-514): when
   * `quantized` is non-NULL and accumulate_image is set, it receives
   * quantize(image, bit_depth, gain) (sensor.cpp:124-135), W*H uint16 */
  uint16_t* quantized;
  double gain;
  int32_t bit_depth;
  int32_t kernel_launches; /* out: CUDA kernels this call launched (all devices) */
  /* optional device-resident result (ABI 2): when non-NULL and accumulate_image
   * is set, the reduced fixed-point image (W*H uint64, radiance * 2^31, the
   * integer ImageBuffer before rb_image_from_fixed's conversion) is left in
   * this DEVICE buffer, which lives on the context's first device (rank 0 in
   * rank mode); `image` and `quantized` may then be NULL to skip host copies. */
  uint64_t* image_fixed;
} rb_trace_out;

typedef struct rb_ctx rb_ctx;

/* ---- lifecycle ---------------------------------------------------------- */
/* n_devices <= 0: all visible devices.  first_device: ordinal of the first
 * device to use (devices first_device .. first_device+n-1).  With more than one
 * device the context renders on all of them from this process (one host thread
 * per device) and owns one NCCL communicator per device (ncclCommInitAll):
 * this is what raybos::run_trace's worker pool (engine.cpp:442-490) becomes on
 * an 8-GPU node.  NCCL is dlopen'ed (libnccl.so.2; RAYBOS_NCCL_LIB overrides). */
int rb_create(int n_devices, int first_device, rb_ctx** out, char* err, size_t errlen);
/* The same over an explicit list of device ordinals. */
int rb_create_devices(const int* devices, int n_devices, rb_ctx** out, char* err, size_t errlen);

/* ---- one process per GPU (torchrun / MPI style launchers) --------------- */
/* rank 0 creates the communicator id and hands the bytes to the other ranks
 * (any out-of-band channel, e.g. a torch.distributed broadcast); every rank then
 * calls rb_create_rank.  In a rank context rb_trace / rb_trace_bos_pair trace
 * this rank's shard of the SAME scene (all ranks pass the same scene), the
 * library sums the partial images onto rank 0 with one ncclReduce and
 * all-reduces the per-source stats and counters, so every rank returns the
 * whole call's DotHitStats and RunReport and rank 0 also returns the image.
 * With world == 1 an id is optional; given one, the one-rank job still runs
 * the NCCL exchange (a single-GPU check of the collective path). */
#define RB_NCCL_UNIQUE_ID_BYTES 128
int rb_nccl_unique_id(void* id, size_t len, char* err, size_t errlen);
int rb_create_rank(int device, int rank, int world, const void* id, size_t len, rb_ctx** out,
                   char* err, size_t errlen);
/* This context's place in the job: rank/world (1 unless rank mode), the number
 * of ranks its NCCL communicator spans (1 without one) and NCCL's version code. */
int rb_comm_info(const rb_ctx* ctx, int* rank, int* world, int* comm_ranks, int* nccl_version);
void rb_destroy(rb_ctx* ctx);
const char* rb_last_error(const rb_ctx* ctx);
int rb_abi_version(void);
int rb_device_count(const rb_ctx* ctx);

/* rb_trace caches its shard plan (the Z-order of the sources, the per-device
 * work lists and the device copies of the sources) and reuses it while the
 * sources, stream ids and pupil axis are bit-identical to the previous call's.
 * rb_plan_reset drops it, so the next call re-plans and re-uploads (a caller
 * timing a cold call, or one that freed the sources' memory). */
int rb_plan_reset(rb_ctx* ctx);
/* Page-locked host memory (cudaHostAlloc, portable): output buffers allocated
 * here are copied to at full PCIe / C2C bandwidth instead of through the
 * driver's pageable staging (a 2 MB FP64 image: ~40 us instead of ~160 us). */
void* rb_host_alloc(size_t bytes);
void rb_host_free(void* p);

/* ---- density grid ------------------------------------------------------- */
/* From GriddedField's own node values (node_n / node_grad, scene.hpp:88-92),
 * FP64 SoA x-fastest, as the reference stores them (scene.hpp:102).  Packed on
 * device into float4 (n-1, dn/dx, dn/dy, dn/dz). */
int rb_set_field_nodes(rb_ctx* ctx, const rb_field_desc* desc, const double* n, const double* gx,
                       const double* gy, const double* gz);
/* From the density volume itself (DensityVolume, scene.hpp:25-40): the
 * GriddedField constructor (scene.cpp:53-92) runs on device — n = K*rho + 1 and
 * the central / one-sided differences in FP64 — and packs the same float4 grid. */
int rb_set_field_density(rb_ctx* ctx, const rb_field_desc* desc, const float* rho,
                         double gladstone_dale_k);
/* A GVOL file (load_density_volume, scene.cpp:212-240: "GVOL1 nx ny nz dx dy dz
 * ox oy oz\n" + little-endian float32, x fastest) streamed to the devices in
 * z-slabs of at most `slab_bytes` (<= 0: 64 MiB) through two pinned buffers, so
 * host memory stays at two slabs for any volume size; the GriddedField ctor then
 * runs on device as in rb_set_field_density.  `z_center` non-NULL recentres the
 * volume on (0, 0, *z_center) like build_medium_volume (engine.cpp:27-37).  The
 * resolved grid geometry is written to `desc_out` (may be NULL).  Error messages
 * and their order are the reference's. */
int rb_set_field_gvol(rb_ctx* ctx, const char* path, const double* z_center,
                      double gladstone_dale_k, int64_t slab_bytes, rb_field_desc* desc_out);
int rb_clear_field(rb_ctx* ctx);
/* Bytes of device memory held by the packed grid (and its per-cell coefficient
 * table, when one was built) on each device. */
int64_t rb_field_bytes(const rb_ctx* ctx);

/* ---- the hot path -------------------------------------------------------- */
/* run_trace(setup, with_field, accumulate_image, run).  Sources are split over
 * the context's devices (and ranks); the partial fixed-point images are summed
 * with one NCCL reduce when more than one device takes part, and every device
 * takes part in it, including those whose shard is empty.  Bit-identical
 * results for any device count.  Fails with RB_E_RUNTIME, rather than
 * returning a wrapped sum, if a landed ray's sensor-plane coordinate exceeds
 * the fixed-point range of hit_sum (2^22 m / rays_per_source). */
int rb_trace(rb_ctx* ctx, const rb_scene* scene, int with_field, int accumulate_image,
             rb_trace_out* out);

/* Host-only (needs no device): the shard of every source under
 * rb_trace_shard(.., shard_index, shard_count, ..).  Sources are ordered along a
 * Z-order curve of their position projected on the pupil plane (neighbouring
 * cones cross the same part of the grid) and dealt to shards in tiles of 32
 * consecutive sources, which balances volume-crossing against missing cones.
 * rb_trace splits sources over its devices with the same plan. */
int rb_plan_shards(const rb_scene* scene, int64_t shard_count, int32_t* shard_of_source);

/* One shard of run_trace for multi-process drivers (one process per GPU):
 * traces the sources rb_plan_shards assigns to shard_index, on device 0 of the
 * context.  image_fixed, if non-NULL, is a DEVICE pointer to W*H uint64 that
 * the partial fixed-point image (radiance * 2^31) is added into; the caller
 * reduces those buffers across ranks (one NCCL sum).  The library's stream first
 * waits for work already queued on the device's legacy default stream (e.g. the
 * caller zeroing the buffer); work on other caller streams must be synchronized
 * by the caller.  The call returns after the image is complete.  Stats are written only
 * for the owned sources; counters cover only the owned sources.  out->image is
 * ignored. */
int rb_trace_shard(rb_ctx* ctx, const rb_scene* scene, int with_field, int accumulate_image,
                   int64_t shard_index, int64_t shard_count, uint64_t* image_fixed,
                   rb_trace_out* out);

/* Converts a device fixed-point image (uint64, radiance * 2^31) to FP64 host
 * radiance (ImageBuffer::data). */
int rb_image_from_fixed(rb_ctx* ctx, const uint64_t* image_fixed_device, int64_t n_pixels,
                        double* image_host);

/* Fixed-point scale of the device image accumulator: 2^31 per unit radiance. */
#define RB_IMAGE_FIXED_SCALE 2147483648.0

/* Per-ray replay of process_source (engine.cpp:107-140) for a list of
 * (source index, ray index) pairs: sensor (u, v), outcome (RB_RAY_*) and RK4
 * steps.  Used by the parity harness and by trace-debug style tooling. */
int rb_trace_rays(rb_ctx* ctx, const rb_scene* scene, int with_field, int64_t n_rays,
                  const int64_t* source_index, const int32_t* ray_index, double* uv,
                  int32_t* status, int32_t* steps);

/* ---- FP64 validation build ------------------------------------------------ */
/* The per-ray pipeline in FP64 with the reference's operation order and no FMA
 * contraction: GRIN samples the FP64 GriddedField nodes exactly like
 * GriddedField::sample (scene.cpp:99-135) and integrates trace_through_volume
 * (grin.cpp:74-134) literally.  Results are bit-identical to the reference
 * except where the device sin/cos in concentric_disk_map (raygen.cpp:24) differ
 * from glibc's by an ulp.  Needs the FP64 node copy the context keeps for grids
 * of at most RB_FP64_MAX_NODES nodes.  Validation only (one thread per ray). */
#define RB_FP64_MAX_NODES (1LL << 26)
int rb_trace_rays_fp64(rb_ctx* ctx, const rb_scene* scene, int with_field, int64_t n_rays,
                       const int64_t* source_index, const int32_t* ray_index, double* uv,
                       int32_t* status, int32_t* steps);
/* Per-source DotHitStats and counters of the FP64 validation build, rays summed
 * in the reference's order (engine.cpp:112-137): hit_sum / landed / counters
 * bit-identical to the reference under the same sin/cos caveat.  No image. */
int rb_trace_stats_fp64(rb_ctx* ctx, const rb_scene* scene, int with_field, rb_trace_out* out);

/* bos_run's two traces (engine.cpp:539-540: run_trace without, then with the
 * field, identical seeds) in one call: on the node grid every ray is generated
 * once and followed both straight (reference leg) and through the density grid
 * (gradient leg); with the per-cell table the two legs run as two passes (the
 * field kernel's occupancy makes that faster).  Per-dot DotHitStats and
 * counters for both legs, no images (bos_run only needs images when
 * write_images is set; use rb_trace for those).  Bit-identical to two
 * rb_trace(accumulate_image = 0) calls. */
int rb_trace_bos_pair(rb_ctx* ctx, const rb_scene* scene, rb_trace_out* out_reference,
                      rb_trace_out* out_gradient);

/* trace_debug (engine.cpp:605-624): the per-step trajectory of one ray, as the
 * StepObserver (grin.hpp:64-66) records it — (xi, r, t) after the volume entry,
 * after every accepted RK4 step and at the cut-back exit — 7 doubles per record
 * (xi, rx, ry, rz, tx, ty, tz).  Runs the FP64 validation build, so the records
 * follow the reference's arithmetic.  *n_records receives the total count even
 * when it exceeds max_records (only the first max_records are written). */
int rb_trace_debug(rb_ctx* ctx, const rb_scene* scene, int64_t source_index, int32_t ray_index,
                   double* records, int64_t max_records, int64_t* n_records);

#ifdef __cplusplus
}
#endif

#endif /* RAYBOS_GPU_H_ */
