#!/usr/bin/env python
"""Benchmark: rays/s for the 1e9-ray Tomo-PIV image through a density grid.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scene tomo]

One JSON line on rank 0.  A step is one full render of the scene's image (all
emitters, all rays: ray generation -> GRIN RK4 -> optics -> sensor deposition)
through the library's public call rb_trace, with the emitters sharded over N
GPUs and the partial 64-bit fixed-point images summed by the library's own NCCL
reduce (strong scaling: the 1e9-ray image is fixed, N GPUs share it).

N GPUs, either way the driver launches it:
  * torchrun --nproc-per-node N bench.py --gpus N: one process per GPU; each
    rank creates its context with rb_create_rank (rank 0's ncclUniqueId is
    broadcast over torch.distributed, which is used for nothing else but the
    barriers and the max-over-ranks of the timings); WORLD_SIZE must equal N.
  * python bench.py --gpus N: one process drives N GPUs (rb_create(N): one
    host thread and one NCCL communicator per device) — what the C++ drop-in
    raybos_gpu::run_trace does on an 8-GPU node.

  value       device-resident throughput: density grid resident in HBM, the
              step = rb_trace leaving the reduced fixed-point image on the
              device (rb_trace_out.image_fixed; per-source stats, 24 B/source,
              and counters still come back), L2 flushed (256 MiB write) before
              every timed step, CUDA events on the launching device around the
              synchronous call; max over ranks.
  e2e         the same call with HOST buffers: the FP64 image and the stats
              copied to the host every step (sources H2D every step in both).
  roofline    K1 (render_emitters / render_warps, as the call reports): scenes with a medium against the box's
              measured FP32 FFMA peak (tools/peaks.cu; MEASURED_PEAKS.json
              has no CUDA-core figure), algorithmic work 360 flops per RK4
              step + 700 per ray; scenes without a medium
              against the measured shared-memory RED.ADD throughput, at one
              RED per pixel of each landed ray's spot window (SURVEY §8(d) rows
              0 and 3: the deposition binds).  traffic from the committed ncu
              capture.
  cpu_baseline  the unmodified reference run_trace (oracle/_ref) on this host's
              cores, on a bounded random sample of the same emitters.
  gpu_launches  kernels the library launched in the timed steps (its own count).
  image_checksum  the last timed step's fixed-point image sum, and whether it
              equals a warm-up step's (bit-reproducibility).
  configs     (N=1 default run) the other BASELINE.json configs — piv, bos,
              optics and one GPU's 1/8 share of the large 1024^3 image — each
              with its own value / e2e / roofline / cpu_baseline.
--impl reference times only that CPU path (rank 0), same metric/config.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "rays/sec at 1/2/4/8 B200 for 1e9-ray image through density grid; % of roofline"
FLOPS_PER_STEP = 360.0
FLOPS_PER_RAY = 700.0
GATHER_BYTES_PER_STEP = 384.0
SCENES = ["piv", "bos", "tomo", "optics", "large"]
# BASELINE.json configs[i] of each scene
BASELINE_CONFIG = {"piv": 0, "bos": 1, "tomo": 2, "optics": 3, "large": 4}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, indices):
        self.indices = ",".join(str(i) for i in sorted(set(indices)))
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "200", "-i", self.indices, "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1]))
                    mx = float(p[2])
                except ValueError:
                    continue
                for n, v in zip(names, p[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


_PEAKS = {}


def measure_peaks(device: int) -> dict:
    """The roofline denominators, measured on this box (tools/peaks.cu), with
    the SM clocks sampled while the microbenchmarks ran."""
    if device in _PEAKS:
        return _PEAKS[device]
    sampler = ClockSampler([device])
    sampler.start()
    time.sleep(0.3)
    from paper_1812_05902_b200 import build as b
    lib = C.CDLL(b.PEAKS_LIB)
    for fn in ("rbp_ffma_tflops",):
        getattr(lib, fn).restype = C.c_double
        getattr(lib, fn).argtypes = [C.c_int, C.c_int]
    lib.rbp_l2_gather_gbs.restype = C.c_double
    lib.rbp_l2_gather_gbs.argtypes = [C.c_int, C.c_double]
    for fn in ("rbp_red_shared_gops", "rbp_dfma_tflops"):
        getattr(lib, fn).restype = C.c_double
        getattr(lib, fn).argtypes = [C.c_int]
    reg = lib.rbp_ffma_tflops(device, 0)
    imm = lib.rbp_ffma_tflops(device, 1)
    pk2 = lib.rbp_ffma_tflops(device, 2)   # packed FFMA2, which K1's Horner evaluation uses
    _PEAKS[device] = {"ffma_reg_tflops": reg, "ffma_imm_tflops": imm, "ffma2_tflops": pk2,
                      "ffma_tflops": max(reg, imm, pk2),
                      "l2_gather_gbs": lib.rbp_l2_gather_gbs(device, 64.0),
                      "red_shared_gops": lib.rbp_red_shared_gops(device),
                      "dfma_tflops": lib.rbp_dfma_tflops(device)}
    _PEAKS[device]["clocks"] = sampler.stop()
    return _PEAKS[device]


# rb_trace_out::k1_kernel -> the render kernel that ran (include/raybos_gpu.h)
K1_NAMES = {1: "render_emitters", 2: "render_warps"}


def profiled_traffic(scene: str, rays: float):
    """dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch of this
    scene from the committed ncu capture (profiles/k1_traffic.json), scaled to
    `rays` when the capture traced fewer (the 1024^3 share), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            t = json.load(f).get(scene)
    except OSError:
        return None
    if not t:
        return None
    return t["dram_bytes_per_launch"] * rays / t.get("rays_per_launch", rays)


def profiled_instructions(scene: str):
    """K1 warp instructions per ray of this scene from the committed ncu capture
    (profiles/k1_instructions.json: smsp__inst_executed.sum / rays of one launch)."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_instructions.json")) as f:
            return json.load(f).get(scene)
    except OSError:
        return None


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f).get("hbm_gbs")
    except OSError:
        return None


# ------------------------------------------------------------ CPU reference
def cpu_reference(scene, grid, target_s: float, seed: int = 0):
    """Times the unmodified reference run_trace (oracle/_ref) — all host threads,
    deterministic tiled mode, image accumulation — on a random sample of the
    scene's emitters sized to about target_s seconds.  Falls back to the C
    restatement (single thread) when the reference library is absent."""
    from oracle.oracle import COracle, Reference, reference_available
    rng = np.random.default_rng(seed)
    perm = rng.permutation(scene.n_sources)
    if reference_available():
        tiny = json.dumps({"scene": {"source": {"type": "dots", "count": 1}},
                           "optics": [{"type": "thin_lens", "focal_length_m": 0.105,
                                       "diameter_m": 0.03}],
                           "sensor": {"gain": 1.0}})
        ref = Reference(json_text=tiny)
        ref.set_flat(scene)
        if grid is not None:
            ref.set_field_density(grid)
        else:
            ref.clear_field()

        def run(m):
            ref.set_sources(scene.sources[perm[:m]])
            r = ref.run_trace(with_field=True, accumulate_image=True, threads=0)
            return r.report["wall_seconds"], r.report["threads"]

        kind, cores = "reference", os.cpu_count()
    else:
        orc = COracle()
        field = orc.field_from_density(grid) if grid is not None else None

        def run(m):
            t0 = time.perf_counter()
            orc.trace(scene.subset(perm[:m]), field, True, True)
            return time.perf_counter() - t0, 1

        kind, cores = "port", 1
    m0 = int(min(scene.n_sources, 2 * max(cores, 1)))
    t, thr = run(m0)
    m = int(min(scene.n_sources, max(m0, m0 * target_s / max(t, 1e-3))))
    return run, m, kind, thr


def cpu_baseline_entry(scene, grid, target_s: float):
    run, m, kind, thr = cpu_reference(scene, grid, target_s)
    t, thr = run(m)
    rays = m * scene.rays_per_source
    # the measured sample rate and its linear extrapolation to
    # the whole image (emitters are drawn at random, so the sample is unbiased)
    return {"value": rays / t, "unit": "rays/s", "cores": thr, "kind": kind,
            "sample": f"{m} of {scene.n_sources} emitters x {scene.rays_per_source} rays "
                      f"({rays:.3g} rays, {t:.1f} s), same grid/optics/sensor, image accumulated",
            "extrapolated_s_per_image": scene.n_sources * scene.rays_per_source / (rays / t)}


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scene", default="tomo", choices=SCENES)
    ap.add_argument("--scale", type=float, default=None,
                    help="emitter-count scale (default 1; 'large' defaults to 1/8 = one GPU's "
                         "share of the 8-GPU image)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true",
                    help="N=1: skip the other four BASELINE configs")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if world > 1 and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; launch one rank per GPU",
              file=sys.stderr)
        return 2
    if args.impl == "reference":
        return main_reference(args, rank, world)
    return main_ours(args, rank, world, local)


def default_scale(name, scale):
    if scale is not None:
        return scale
    return 0.125 if name == "large" else 1.0


def workload_config(name, scene, desc, info, n_gpus):
    share = ""
    if name == "large":
        share = (f" (one GPU's 1/8 share of the {8 * scene.n_sources} x "
                 f"{scene.rays_per_source} = {8 * scene.n_sources * scene.rays_per_source:.3g}-ray "
                 "8-GPU image)")
    return {"workload": f"{name}: {scene.n_sources} emitters x {scene.rays_per_source} rays "
                        f"({scene.n_sources * scene.rays_per_source:.3g} rays/image){share}, "
                        f"{scene.width}x{scene.height} sensor" +
                        (f", {desc['field']}" if "field" in desc else ", no medium"),
            "baseline_config": BASELINE_CONFIG[name],
            "scene": name, "emitters": scene.n_sources,
            "rays_per_emitter": scene.rays_per_source,
            "rays_per_image": scene.n_sources * scene.rays_per_source,
            "sensor": [scene.width, scene.height], "delta_xi_m": scene.delta_xi,
            "d_tau_m": scene.d_tau, "magnification": info.magnification,
            "parallelism": f"emitter shards x{n_gpus}, NCCL reduce of int64 image",
            "l2": "256 MiB L2 flush before every timed step"}


def main_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_1812_05902_b200 import scenes
    from oracle.oracle import COracle
    orc = COracle()

    def calibrate(sc):
        return orc.trace(sc, None, with_field=False, accumulate_image=True).image

    scale = default_scale(args.scene, args.scale)
    scene, grid, info, desc = scenes.build(args.scene, calibrate=calibrate, scale=scale)
    run, m, kind, thr = cpu_reference(scene, grid, args.cpu_seconds)
    for _ in range(args.warmup):
        run(max(1, m // 8))
    ts = []
    for _ in range(args.steps):
        t, thr = run(m)
        ts.append(t)
    rays = m * scene.rays_per_source
    value = rays / (sum(ts) / len(ts))
    cfg = workload_config(args.scene, scene, desc, info, args.gpus)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(ts) / len(ts), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            # what one timed step actually traced: a random sample of the
            # workload's emitters (the rate is unbiased; the image is not whole)
            "timed_rays_per_step": rays, "timed_emitters_per_step": m,
            "cpu_baseline": {"value": value, "unit": "rays/s", "cores": thr, "kind": kind,
                             "sample": f"{m} of {scene.n_sources} emitters x "
                                       f"{scene.rays_per_source} rays per step"},
            "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


class Job:
    """The process's place in the N-GPU job and its collectives (timing only)."""

    def __init__(self, args, rank, world, local):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.gpus = rank, world, args.gpus
        # RAYBOS_BENCH_BACKEND=gloo is a path check only: it lets the torchrun
        # (N>1) code run on a one-GPU box (ranks share the device, the library's
        # NCCL replaced by tests/fake_nccl through RAYBOS_NCCL_LIB); its
        # numbers are not a measurement.
        self.backend = os.environ.get("RAYBOS_BENCH_BACKEND", "nccl")
        ndev = torch.cuda.device_count()
        self.device = local if self.backend == "nccl" else local % ndev
        torch.cuda.set_device(self.device)
        from paper_1812_05902_b200.engine import GpuTracer, nccl_unique_id
        if world > 1 or "WORLD_SIZE" in os.environ:
            # launched by torchrun: one process per GPU, the library's rank mode —
            # also for a one-process run, so every N of a scaling curve goes
            # through the same rb_create_rank + NCCL exchange path
            if world > 1:
                if self.backend == "nccl":
                    dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
                else:
                    dist.init_process_group(self.backend)
                uid = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
            else:
                uid = [nccl_unique_id()]
            self.tracer = GpuTracer.for_rank(self.device, rank, world, uid[0])
            self.devices = [self.device]
            self.mode = "ranks"
        elif args.gpus > 1:
            # RAYBOS_BENCH_DEVICES (path check only, e.g. "0,0" on a one-GPU box
            # with the NCCL stand-in) names the devices; default 0..N-1
            env = os.environ.get("RAYBOS_BENCH_DEVICES")
            self.devices = ([int(x) for x in env.split(",")] if env else list(range(args.gpus)))
            assert len(self.devices) == args.gpus
            self.tracer = GpuTracer(devices=self.devices)
            self.mode = "in-process"
        else:
            self.tracer = GpuTracer(n_devices=1, first_device=self.device)
            self.devices = [self.device]
            self.mode = "single"
        self.comm = self.tracer.comm_info()
        print(f"raybos: rank {rank} of {world} process(es), devices {self.devices}, NCCL "
              f"communicator spans {self.comm['comm_ranks']} rank(s)"
              f" (NCCL version code {self.comm['nccl_version']})", file=sys.stderr, flush=True)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        for d in sorted(set(self.devices)):
            self.torch.cuda.synchronize(d)

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64,
                              device="cuda" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        self.tracer.close()
        if self.world > 1:
            self.dist.barrier()
            self.dist.destroy_process_group()


def spot_reds_per_ray(scene):
    """Shared-memory REDs per landed ray of the deposition: the spot window is
    floor(c + hw) - floor(c - hw) + 1 pixels a side (sensor.cpp:44-55), i.e.
    2 hw + 1 on average over sub-pixel centres."""
    sigma = 0.25 * scene.d_tau
    hw = scene.sensor.window_sigmas * sigma / scene.sensor.pitch
    if sigma < 1e-3 * scene.sensor.pitch:
        return 1.0
    return (2.0 * hw + 1.0) ** 2


def bench_scene(job, name, scale, steps, warmup, args, want_cpu, want_e2e):
    """One BASELINE config through rb_trace; returns the JSON entry (rank 0)."""
    torch = job.torch
    from paper_1812_05902_b200 import scenes
    tracer = job.tracer

    def calibrate(sc):  # the gain-calibration dot (engine.cpp:396-412); image on rank 0 only
        img = tracer.run_trace(sc, with_field=False, accumulate_image=True, host_image=True).image
        return img if img is not None else np.zeros(1)

    scene, grid, info, desc = scenes.build(name, calibrate=calibrate, scale=scale)
    t0 = time.perf_counter()
    tracer.set_field(grid)
    field_s = time.perf_counter() - t0
    W, H = scene.width, scene.height
    rays_total = scene.n_sources * scene.rays_per_source
    dev0 = job.devices[0]
    img = torch.zeros(W * H, dtype=torch.int64, device=f"cuda:{dev0}") if job.rank == 0 else None
    flush = [torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{d}")
             for d in sorted(set(job.devices))]

    def step():
        return tracer.run_trace(scene, True, True, host_image=False,
                                image_fixed_ptr=img.data_ptr() if img is not None else 0)

    for _ in range(warmup):
        step()
    checksum_warm = int(img.sum().item()) if img is not None else 0
    sampler = ClockSampler(job.devices)
    job.barrier()
    sampler.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream(dev0)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    total_ms, kernel_ms, launches, res = 0.0, [], 0, None
    for k in range(steps):
        for f in flush:
            f.fill_(k & 0xFF)
        job.barrier()
        with torch.cuda.device(dev0):
            ev0.record(stream)
            res = step()
            ev1.record(stream)
        torch.cuda.synchronize(dev0)
        total_ms += ev0.elapsed_time(ev1)
        kernel_ms.append(res.report["kernel_ms"])
        launches += res.report["kernel_launches"]
    clocks = sampler.stop()
    checksum_last = int(img.sum().item()) if img is not None else 0
    ms_per_step = job.max_over_ranks(total_ms / steps)
    kms = job.max_over_ranks(sum(kernel_ms) / len(kernel_ms))
    value = rays_total / (ms_per_step * 1e-3)
    steps_sum = res.report["total_steps"]          # whole call (all ranks, all devices)

    e2e = None
    if want_e2e:
        # Every step re-plans and re-uploads the scene's sources from host memory
        # (rb_plan_reset: the shard-plan cache the value steps reuse is dropped),
        # and the FP64 image + per-emitter stats come back to the host; the image
        # lands in a page-locked buffer (rb_host_alloc) as an application
        # streaming frames would keep one.
        n_src = scene.n_sources
        h2d = n_src * (3 * 8 + 4)                  # source positions + work order
        d2h = W * H * 8 + n_src * (2 * 8 + 8) + 6 * 8   # FP64 image + stats + counters
        host_img = tracer.pinned((H, W)) if job.rank == 0 else None
        e2e_ms = []
        tracer.reset_plan()
        tracer.run_trace(scene, True, True, image_out=host_img, host_image=(job.rank == 0))
        for _ in range(steps):
            job.barrier()
            s0 = time.perf_counter()
            tracer.reset_plan()
            tracer.run_trace(scene, True, True, image_out=host_img, host_image=(job.rank == 0))
            job.barrier()
            e2e_ms.append(1e3 * (time.perf_counter() - s0))
        te = job.max_over_ranks(sum(e2e_ms) / len(e2e_ms))
        e2e = {"value": rays_total / (te * 1e-3), "unit": "rays/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": te,
               "path": "rb_trace (C-ABI, host buffers; shard plan and sources rebuilt and "
                       "uploaded every step, image into page-locked memory)"}
    if job.rank != 0:
        return None

    peaks = measure_peaks(dev0)
    n_gpus = len(job.devices) * job.world
    ins = profiled_instructions(name)
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    sms = job.torch.cuda.get_device_properties(dev0).multi_processor_count
    peak_issue = 4.0 * sms * sm_mhz * 1e6 / 1e9  # G warp-instructions / s
    issue = None
    if ins:
        ach = ins["warp_inst_per_ray"] * rays_total / n_gpus / (kms * 1e-3) / 1e9
        issue = {"achieved": ach, "peak": peak_issue, "unit": "Gwarp-inst/s",
                 "frac": ach / peak_issue,
                 "per_ray": f"{ins['warp_inst_per_ray']:.1f} warp-instructions per ray "
                            f"({ins['source']})",
                 "peak_source": f"4 warp-instructions/clk/SM x {sms} SMs x {sm_mhz:.0f} MHz "
                                "(the SM clock sampled during the timed steps)"}
    if grid is not None:
        flops = FLOPS_PER_STEP * steps_sum + FLOPS_PER_RAY * rays_total
        achieved = flops / n_gpus / (kms * 1e-3) / 1e12
        gather = GATHER_BYTES_PER_STEP * steps_sum / n_gpus / (kms * 1e-3) / 1e9
        roofline = {"bound": "fp32", "achieved": achieved, "peak": peaks["ffma_tflops"],
                    "unit": "TFLOP/s", "frac": achieved / peaks["ffma_tflops"],
                    "per_ray": f"{FLOPS_PER_STEP:.0f} flops/RK4 step + {FLOPS_PER_RAY:.0f}; "
                               f"{steps_sum / max(rays_total, 1):.1f} steps/ray measured",
                    "peak_source": "measured on this box: FFMA microbenchmark "
                                   "(tools/peaks.cu), max of register / immediate / packed-FFMA2",
                    # what the samples would move if each gathered its 8 corners
                    # (3 x 8 x 16 B per step): above the measured L2 gather peak,
                    # which is why K1 caches the cell in registers instead
                    "gather": {"uncached_equivalent_gbs": gather,
                               "l2_gather_peak_gbs": peaks["l2_gather_gbs"],
                               "bytes_per_step": GATHER_BYTES_PER_STEP},
                    "issue": issue}
    else:
        # Without a medium K1 is instruction-issue bound (SURVEY §8(d) names the
        # deposition, but its shared REDs run at < 10% of their measured peak):
        # the roof is the SMs' issue rate, 4 warp-instructions per clock per SM
        # at the clock measured during the timed steps, and the work is the
        # committed ncu count of warp-instructions per ray of this scene.
        landed = res.report["landed"]
        reds = spot_reds_per_ray(scene) * landed
        red_ach = reds / n_gpus / (kms * 1e-3) / 1e9
        deposition = {"achieved": red_ach, "peak": peaks["red_shared_gops"], "unit": "Gop/s",
                      "frac": red_ach / peaks["red_shared_gops"],
                      "per_ray": f"{spot_reds_per_ray(scene):.1f} shared-memory RED.ADD.U32 per "
                                 f"landed ray (spot window (2 hw + 1)^2); {landed} of "
                                 f"{rays_total} rays landed",
                      "peak_source": "measured on this box: conflict-free red.shared.add.u32 "
                                     "microbenchmark (tools/peaks.cu)"}
        if issue:
            roofline = dict(issue, bound="issue", deposition=deposition)
        else:
            roofline = dict(deposition, bound="smem_red")
    roofline.update({"traffic": profiled_traffic(name, rays_total) if n_gpus == 1 else None,
                     "traffic_source": "profiles/k1_traffic.json (ncu --set full of one K1 "
                                       "launch, per ray x this launch's rays)",
                     "kernel": K1_NAMES.get(res.report.get("k1_kernel", 1), "render_emitters"),
                     "kernel_ms": kms,
                     "ffma_reg_tflops": peaks["ffma_reg_tflops"],
                     "ffma_imm_tflops": peaks["ffma_imm_tflops"],
                     "ffma2_tflops": peaks["ffma2_tflops"],
                     "red_shared_gops": peaks["red_shared_gops"],
                     "dfma_tflops": peaks["dfma_tflops"],
                     "hbm_gbs_measured": measured_hbm(),
                     "peak_clocks": peaks["clocks"],   # during the peak microbenchmarks
                     "kernel_clocks": clocks})         # during the timed steps
    cpu = None
    if want_cpu:
        try:
            cpu = cpu_baseline_entry(scene, grid, args.cpu_seconds)
        except Exception as e:  # report, never hide
            cpu = {"value": None, "unit": "rays/s", "cores": None, "kind": "reference",
                   "sample": f"failed: {e}"}
    return {"value": value, "ms_per_step": ms_per_step, "steps": steps, "warmup": warmup,
            "config": workload_config(name, scene, desc, info, n_gpus),
            "setup": {"field_upload_s": field_s,
                      "steps_per_ray": steps_sum / max(rays_total, 1)},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": launches,
            "image_checksum": {"fixed_point_sum": checksum_last,
                               "identical_to_warmup": checksum_last == checksum_warm}}


def main_ours(args, rank, world, local):
    job = Job(args, rank, world, local)
    n_gpus = len(job.devices) * job.world
    single = n_gpus == 1
    head = bench_scene(job, args.scene, default_scale(args.scene, args.scale), args.steps,
                       args.warmup, args, want_cpu=single and not args.no_cpu_baseline,
                       want_e2e=not args.no_e2e)
    extras = {}
    if single and not args.no_extra_configs and args.scene == "tomo" and args.scale is None:
        # the other BASELINE configs, at a few steps each (inside the default run)
        for name in ("piv", "bos", "optics", "large"):
            try:
                e = bench_scene(job, name, default_scale(name, None), min(args.steps, 3),
                                max(3, min(args.warmup, 3)), args,
                                want_cpu=not args.no_cpu_baseline, want_e2e=not args.no_e2e)
            except Exception as ex:  # report, never hide
                e = {"error": f"{type(ex).__name__}: {ex}"}
            extras[name] = e
            job.tracer.set_field(None)
    if rank == 0:
        line = {"metric": METRIC, "value": head["value"], "unit": "rays/s", "n_gpus": n_gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 GRIN + f64 raygen/optics/sensor", "data": "synthetic",
                "config": head["config"], "setup": head["setup"], "e2e": head["e2e"],
                "roofline": head["roofline"], "cpu_baseline": head["cpu_baseline"],
                "clocks": head["clocks"], "gpu_launches": head["gpu_launches"],
                "image_checksum": head["image_checksum"],
                "comm": dict(job.comm, mode=job.mode,
                             processes=job.world, devices_per_process=len(job.devices))}
        if extras:
            line["configs"] = extras
        print(json.dumps(line), flush=True)
    job.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
