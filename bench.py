#!/usr/bin/env python
"""Benchmark: rays/s for the 1e9-ray Tomo-PIV image through a density grid.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scene tomo]

One JSON line on rank 0.  A step is one full render of the scene's image (all
emitters, all rays: ray generation -> GRIN RK4 -> optics -> sensor deposition),
with the emitters sharded over the N ranks and the partial 64-bit fixed-point
images summed with one NCCL reduce (strong scaling: the 1e9-ray image is fixed,
N GPUs share it).

  value       device-resident throughput: density grid resident in HBM, the
              step = rb_trace_shard (K1 render) + NCCL reduce, timed with CUDA
              events between barriers, L2 flushed (256 MiB write) before every
              timed step; max over ranks.
  e2e         the same image through the public C-ABI with HOST buffers: scene
              sources H2D, render, reduce, FP64 image + per-emitter stats D2H
              (rb_trace at N=1; rb_trace_shard + reduce + rb_image_from_fixed at N>1).
  roofline    K1 render_emitters against the box's measured FP32 peak (best of
              FFMA register / immediate / packed FFMA2 forms; MEASURED_PEAKS.json
              has no CUDA-core number, measured here with tools/peaks.cu).
              Algorithmic work per ray = 360 flops per RK4 step + 700 (SURVEY.md
              §8(a)); traffic from the committed ncu capture.
  cpu_baseline  the unmodified reference run_trace (oracle/_ref) on this host's
              cores, on a bounded random sample of the same emitters (plus the
              extrapolated whole-image time).
  gpu_launches  kernels the library launched in the timed steps (its own count).
  image_checksum  the last timed step's fixed-point image sum, and whether it
              equals a warm-up step's (bit-reproducibility).
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


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "200", "-i", str(self.index), "-f", self.path],
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


def measure_peaks(device: int) -> dict:
    from paper_1812_05902_b200 import build as b
    lib = C.CDLL(b.PEAKS_LIB)
    lib.rbp_ffma_tflops.restype = C.c_double
    lib.rbp_ffma_tflops.argtypes = [C.c_int, C.c_int]
    lib.rbp_l2_gather_gbs.restype = C.c_double
    lib.rbp_l2_gather_gbs.argtypes = [C.c_int, C.c_double]
    reg = lib.rbp_ffma_tflops(device, 0)
    imm = lib.rbp_ffma_tflops(device, 1)
    pk2 = lib.rbp_ffma_tflops(device, 2)   # packed FFMA2, which K1's Horner evaluation uses
    return {"ffma_reg_tflops": reg, "ffma_imm_tflops": imm, "ffma2_tflops": pk2,
            "ffma_tflops": max(reg, imm, pk2),
            "l2_gather_gbs": lib.rbp_l2_gather_gbs(device, 64.0)}


def profiled_traffic(scene: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch of this
    scene, from the committed ncu capture (profiles/k1_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_traffic.json")) as f:
            return json.load(f).get(scene, {}).get("dram_bytes_per_launch")
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
    ap.add_argument("--scene", default="tomo", choices=["piv", "bos", "tomo", "optics", "large"])
    ap.add_argument("--scale", type=float, default=1.0, help="emitter-count scale (tests only)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return main_reference(args, rank, world)
    return main_ours(args, rank, world, local)


def workload_config(args, scene, desc, info, world):
    return {"workload": f"{args.scene}: {scene.n_sources} emitters x {scene.rays_per_source} rays "
                        f"({scene.n_sources * scene.rays_per_source:.3g} rays/image), "
                        f"{scene.width}x{scene.height} sensor" +
                        (f", {desc['field']}" if "field" in desc else ", no medium"),
            "scene": args.scene, "emitters": scene.n_sources,
            "rays_per_emitter": scene.rays_per_source,
            "rays_per_step": scene.n_sources * scene.rays_per_source,
            "sensor": [scene.width, scene.height], "delta_xi_m": scene.delta_xi,
            "d_tau_m": scene.d_tau, "magnification": info.magnification,
            "parallelism": f"emitter shards x{world}, NCCL reduce of int64 image",
            "l2": "256 MiB L2 flush before every timed step"}


def main_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_1812_05902_b200 import scenes
    from oracle.oracle import COracle
    orc = COracle()

    def calibrate(sc):
        return orc.trace(sc, None, with_field=False, accumulate_image=True).image

    scene, grid, info, desc = scenes.build(args.scene, calibrate=calibrate, scale=args.scale)
    run, m, kind, thr = cpu_reference(scene, grid, args.cpu_seconds)
    for _ in range(args.warmup):
        run(max(1, m // 8))
    ts = []
    for _ in range(args.steps):
        t, thr = run(m)
        ts.append(t)
    rays = m * scene.rays_per_source
    value = rays / (sum(ts) / len(ts))
    cfg = workload_config(args, scene, desc, info, world)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(ts) / len(ts), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": value, "unit": "rays/s", "cores": thr, "kind": kind,
                             "sample": f"{m} of {scene.n_sources} emitters x "
                                       f"{scene.rays_per_source} rays per step"},
            "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_1812_05902_b200 import scenes
    from paper_1812_05902_b200.engine import GpuTracer

    # RAYBOS_BENCH_BACKEND=gloo is a path check only: it lets the torchrun
    # (N>1) code run on a one-GPU box (ranks share the device, collectives go
    # through host memory); its numbers are not a measurement.
    backend = os.environ.get("RAYBOS_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    def reduce_to_root(x):
        if backend == "nccl":
            dist.reduce(x, 0)
        else:
            h = x.cpu()
            dist.reduce(h, 0)
            x.copy_(h)

    def max_over_ranks(x):
        if backend == "nccl":
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
        else:
            h = x.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX)
            x.copy_(h)
    tracer = GpuTracer(n_devices=1, first_device=local)

    def calibrate(sc):
        return tracer.run_trace(sc, with_field=False, accumulate_image=True).image

    scene, grid, info, desc = scenes.build(args.scene, calibrate=calibrate, scale=args.scale)
    t0 = time.perf_counter()
    tracer.set_field(grid)
    field_s = time.perf_counter() - t0
    W, H = scene.width, scene.height
    rays_total = scene.n_sources * scene.rays_per_source
    img = torch.zeros(W * H, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        img.zero_()
        torch.cuda.current_stream().synchronize()   # the library runs on its own stream
        rep = tracer.trace_shard(scene, True, True, rank, world, img.data_ptr())
        if world > 1:
            reduce_to_root(img)
        return rep

    for _ in range(args.warmup):
        step()
    # determinism evidence: the reduced fixed-point image of a warm-up step and of
    # the last timed step must be the same integers (checked on rank 0 after the loop)
    checksum_warm = int(img.sum().item()) if rank == 0 else 0
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    total_ms, kernel_ms, steps_sum, rays_local, launches = 0.0, [], 0, 0, 0
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        barrier()
        ev0.record()
        rep = step()
        ev1.record()
        torch.cuda.synchronize()
        total_ms += ev0.elapsed_time(ev1)
        kernel_ms.append(rep["kernel_ms"])
        launches += rep["kernel_launches"]  # render + split-stats kernels (library count)
        steps_sum = rep["total_steps"]
        rays_local = rep["emitted"]
    clocks = sampler.stop()
    checksum_last = int(img.sum().item()) if rank == 0 else 0
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        max_over_ranks(t)
    ms_per_step = t.item() / args.steps
    value = rays_total / (ms_per_step * 1e-3)

    # e2e through the public C-ABI with host buffers
    e2e = None
    if not args.no_e2e:
        n_src = scene.n_sources
        h2d = n_src * (3 * 8 + 4)                  # source positions + work order
        d2h = W * H * 8 + n_src * (2 * 8 + 8) + 6 * 8   # FP64 image + stats + counters
        if world == 1:
            tracer.run_trace(scene, True, True)
        e2e_ms = []
        for _ in range(args.steps):
            barrier()
            s0 = time.perf_counter()
            if world == 1:
                tracer.run_trace(scene, True, True)
            else:
                img.zero_()
                torch.cuda.current_stream().synchronize()
                tracer.trace_shard(scene, True, True, rank, world, img.data_ptr())
                reduce_to_root(img)
                if rank == 0:
                    tracer.image_from_fixed(img.data_ptr(), (H, W))
            barrier()
            e2e_ms.append(1e3 * (time.perf_counter() - s0))
        te = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            max_over_ranks(te)
        e2e = {"value": rays_total / (te.item() * 1e-3), "unit": "rays/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": te.item(),
               "path": "rb_trace (C-ABI, host buffers)" if world == 1 else
                       "rb_trace_shard + NCCL reduce + rb_image_from_fixed (host buffers)"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peaks = measure_peaks(local)
    kms = sum(kernel_ms) / len(kernel_ms)
    flops = FLOPS_PER_STEP * steps_sum + FLOPS_PER_RAY * rays_local
    achieved = flops / (kms * 1e-3) / 1e12
    gather = GATHER_BYTES_PER_STEP * steps_sum / (kms * 1e-3) / 1e9
    roofline = {"bound": "fp32", "achieved": achieved, "peak": peaks["ffma_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["ffma_tflops"],
                "traffic": profiled_traffic(args.scene) if world == 1 else None,
                "traffic_source": "profiles/k1_traffic.json (ncu --set full, one launch)",
                "kernel": "render_emitters", "kernel_ms": kms,
                "peak_source": "measured on this box: FFMA microbenchmark (tools/peaks.cu), "
                               "max of register / immediate / packed-FFMA2 forms",
                "per_ray": f"{FLOPS_PER_STEP:.0f} flops/RK4 step + {FLOPS_PER_RAY:.0f}; "
                           f"{steps_sum / max(rays_local, 1):.1f} steps/ray measured",
                # what the samples would move if each gathered its 8 corners
                # (3 x 8 x 16 B per step): above the measured L2 gather peak,
                # which is why K1 caches the cell in registers instead
                "gather": {"uncached_equivalent_gbs": gather,
                           "l2_gather_peak_gbs": peaks["l2_gather_gbs"],
                           "bytes_per_step": GATHER_BYTES_PER_STEP},
                "ffma_reg_tflops": peaks["ffma_reg_tflops"],
                "ffma_imm_tflops": peaks["ffma_imm_tflops"],
                "ffma2_tflops": peaks["ffma2_tflops"], "hbm_gbs_measured": measured_hbm()}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_entry(scene, grid, args.cpu_seconds)
        except Exception as e:  # report, never hide
            cpu = {"value": None, "unit": "rays/s", "cores": None, "kind": "reference",
                   "sample": f"failed: {e}"}
    line = {"metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 GRIN + f64 raygen/optics/sensor", "data": "synthetic",
            "config": dict(workload_config(args, scene, desc, info, world),
                           field_upload_s=field_s, steps_per_ray=steps_sum / max(rays_local, 1)),
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": launches,
            "image_checksum": {"fixed_point_sum": checksum_last,
                               "identical_to_warmup": checksum_last == checksum_warm}}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
