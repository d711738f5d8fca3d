#!/usr/bin/env python3
"""Headline benchmark: FPS of a 1920x1080 sphere-traced KiloNeuS frame (primary rays + FD normals
+ colour pass) on the random-init 16^3 field of SPEC.md defaults -- BASELINE.json config 3.

    python bench.py --gpus 1 --steps 20 --warmup 3           # our arm, one GPU
    torchrun --nproc-per-node N ... bench.py --gpus N ...    # one rank per GPU, views sharded (weak scaling)
    torchrun ... bench.py --gpus N --shard rows              # one frame per step split into interleaved row bands (strong scaling)
    python bench.py --impl reference --gpus 1 ...            # the reference's own CPU renderer (oracle/_ref: the unmodified
                                                             # kilofield package, installed by oracle/build_ref.py), all host threads

One "step" = every rank renders one orbit view (view = step * N + rank) with the field resident in
HBM, then the finished buffers (colour, depth, normal, hit) are all-gathered over NCCL.  Prints ONE JSON line (rank 0).
At N = 1 the line also carries the other BASELINE.json configs (`configs`: 2 orbit, 4 batched forward, 5 4K path trace).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SM_COUNT = 148
FFMA_LANES_PER_SM = 128
FLOP_PER_SDF_EVAL = 5120  # 2 * (39*32 + 32*32 + 32*9), SURVEY 8(d)
FLOP_PER_COLOR_EVAL = 4864
ROUTE_BYTES_PER_REQUEST = 16.25  # scatter reads cell+rank+offset (12 B) and writes perm (4 B) per routed request, + 16 B tile per 64
ROUTE_BYTES_PER_CELL = 16      # scan: count read + zeroed, offset + tile base written, per cell per wavefront
ORBIT_VIEWS, ORBIT_RADIUS, ORBIT_ELEV, FOV = 100, 2.5, 0.2, np.deg2rad(40.0)


PREHEAT_FRAMES = int(os.environ.get("BENCH_PREHEAT", "48"))  # untimed, before the W warm-up steps (BENCH_PREHEAT=0 for ncu launch lists)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """Samples SM clocks and throttle reasons during the timed region (B200_PROFILING.md 'clocks' line).

    Uses NVML in-process (nvidia_ml_py) every 250 ms: spawning one nvidia-smi per sample was measured to
    slow the timed frames by ~25 % (driver-lock contention), a long-lived `nvidia-smi -lms` is the fallback.
    """

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._stop, self._t, self._proc = index, [], threading.Event(), None, None
        self.nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index(index))
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)  # ~40 ms: once, outside the timed region
        except Exception:
            self.nvml = None

    @staticmethod
    def _physical_index(index):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[index])
            except Exception:
                return index
        return index

    def _nvml_row(self):
        n = self.nvml
        sm = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
        mx = self.max_sm
        try:
            mask = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
        except Exception:
            mask = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
        flags = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}
        return sm, mx, [k for k, bit in flags.items() if mask & bit]

    def _run(self):
        while not self._stop.is_set():
            try:
                self.rows.append(self._nvml_row())
            except Exception:
                pass
            self._stop.wait(0.25)

    def __enter__(self):
        if self.nvml is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        else:
            try:
                self._proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                               "-lms", "250"], stdout=subprocess.PIPE, text=True)
            except Exception:
                self._proc = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=3)
        if self._proc is not None:
            self._proc.terminate()
            try:
                out = self._proc.communicate(timeout=3)[0]
            except Exception:
                out = ""
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in out.splitlines():
                c = [x.strip() for x in line.split(",")]
                if len(c) >= 7 and c[0].replace(".", "").isdigit():
                    self.rows.append((float(c[0]), float(c[1]), [n for n, v in zip(names, c[3:7]) if v.lower().startswith("active")]))

    def summary(self):
        sm = [float(r[0]) for r in self.rows]
        mx = [float(r[1]) for r in self.rows]
        reasons = sorted({x for r in self.rows for x in r[2]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi -lms"}


def orbit_view(k: int, width: int, height: int):
    from paper_2206_10885_b200.cameras import orbit_pose

    return orbit_pose(k % ORBIT_VIEWS, ORBIT_VIEWS, ORBIT_RADIUS, ORBIT_ELEV, FOV, width, height)


def _reference_package():
    """The unmodified reference (kilofield) installed in oracle/_ref by oracle/build_ref.py, or None."""
    try:
        from oracle import build_ref

        return build_ref.import_reference() if build_ref.available() else None
    except Exception:
        return None


_REF_CACHE: dict = {}


def cpu_frame_seconds(width: int, height: int, view: int, threads: int):
    """One (width x height) frame of the SAME camera and field on the host CPU: the reference's own
    kilofield.surface.render_frame (kind "reference") when oracle/_ref is installed, else the oracle port of it
    (kind "port").  Returns (seconds, kind, hit_fraction).  KNF_THREADS is the reference's own knob (surface.py:32-39)."""
    pose = orbit_view(view, width, height)
    kf = _reference_package()
    os.environ["KNF_THREADS"] = str(max(1, int(threads)))
    if kf is not None:
        if "ref" not in _REF_CACHE:
            field = kf.grid.field_init(kf.grid.GridConfig(), seed=0)
            _REF_CACHE["ref"] = kf.surface.FieldSurface(field)
        cam = kf.cameras.CameraPose(np.asarray(pose.position, dtype=np.float64), np.asarray(pose.rotation, dtype=np.float64),
                                    float(pose.fov_y), int(width), int(height))
        t0 = time.perf_counter()
        fb = kf.surface.render_frame(_REF_CACHE["ref"], cam, kf.surface.RenderSettings())
        return time.perf_counter() - t0, "reference", float(fb.hit.mean())
    import oracle

    if "port" not in _REF_CACHE:
        _REF_CACHE["port"] = oracle.FieldTraceable(oracle.make_random_field(oracle.FieldSpec(resolution=16), seed=0))
    cam = oracle.Camera(pose.position, pose.rotation, pose.fov_y, width, height)
    t0 = time.perf_counter()
    frame = oracle.render(_REF_CACHE["port"], cam, oracle.MarchSettings())
    return time.perf_counter() - t0, "port", float(frame.hit.mean())


def sample_raster(budget_rays: float):
    """A 16:9 raster with about `budget_rays` rays, between 64x36 and 480x270."""
    h = int(np.clip(np.sqrt(budget_rays * 9 / 16), 36, 270))
    return (h * 16) // 9, h


def host_description():
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cpus": os.cpu_count(), "cpu_model": model, "numpy": np.__version__}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU renderer on this box's host cores, rank 0 only.

    Timed steps: each step renders ONE bounded sample raster (same orbit view, same field, same settings) with
    KNF_THREADS = all host cores -- `ms_per_step` is the time of exactly those steps.  `value` (frames/s at WxH) comes from
    ONE full WxH frame rendered un-extrapolated after the steps (BENCH_REF_FULL=0 skips it and scales the sample per
    ray instead, labelled as such); the 1-thread figure (BASELINE.md section 3 asks for both) is measured on the sample raster."""
    if rank != 0:
        return
    W, H = args.width, args.height
    total = args.steps + args.warmup
    ncpu = os.cpu_count() or 1
    w, h = sample_raster(48.0 * 20000.0 / max(total, 1))  # ~20 krays/s on one core: ~48 s for all the steps together
    times, kind = [], "port"
    for s in range(total):
        dt, kind, _ = cpu_frame_seconds(w, h, s, ncpu)
        if s >= args.warmup:
            times.append(dt)
    sec = float(np.sum(times))
    sample_rps_all = len(times) * w * h / sec
    one = [cpu_frame_seconds(w, h, args.warmup, 1)[0] for _ in range(2)]
    sample_rps_one = w * h / min(one)
    full = None
    if os.environ.get("BENCH_REF_FULL", "1") != "0":
        # The reference's own threading (KNF_THREADS row bands, each calling multi-threaded BLAS) helps on small rasters and HURTS on
        # the full frame: measured on this pool, 16 threads give 1.5x on the 480x270 sample but 0.5x at 1920x1080 (155-168 s vs
        # 83 s, profiles/bench_r2_reference.json / bench_reference_r2_final2.json).  The full frame is rendered with the setting
        # that is the reference's best there: all threads only if they at least double the sample rate.
        threads_full = ncpu if sample_rps_all >= 2.0 * sample_rps_one else 1
        dt, kind, hitf = cpu_frame_seconds(W, H, args.warmup, threads_full)
        full = {"seconds": dt, "threads": threads_full, "hit_fraction": hitf, "fps": 1.0 / dt, "krays_per_s": W * H / dt / 1e3}
    fps = full["fps"] if full else max(sample_rps_all, sample_rps_one) / (W * H)
    what = "kilofield.surface.render_frame of the unmodified reference package (oracle/_ref)" if kind == "reference" else \
        "oracle.render, the NumPy restatement of the reference renderer (oracle/_ref not installed on this box)"
    sample = (f"{what}; value = one full {W}x{H} frame, un-extrapolated ({full['seconds']:.1f} s, KNF_THREADS={full['threads']})" if full else
              f"{what}; value extrapolated per ray from the {w}x{h} sample raster (BENCH_REF_FULL=0)")
    sample += (f"; the {args.steps} timed steps are {w}x{h} rasters of the same orbit views at KNF_THREADS={ncpu} ({sample_rps_all / 1e3:.1f} krays/s; "
               f"{sample_rps_one / 1e3:.1f} krays/s at KNF_THREADS=1)")
    line = {
        "impl": "reference", "metric": f"fps_{W}x{H}_sphere_traced", "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / max(len(times), 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(W, H, world, args.shard),
        "ms_per_step_is": f"one {w}x{h} sample raster per step (what the timed steps rendered); a {W}x{H} frame takes 1e3 / value ms",
        "cpu_baseline": dict({"value": fps, "unit": "frames/s", "cores": (full["threads"] if full else ncpu), "kind": kind, "sample": sample,
                              "full_frame": full, "sample_raster": [w, h], "sample_krays_per_s_all_threads": sample_rps_all / 1e3,
                              "sample_krays_per_s_1_thread": sample_rps_one / 1e3}, **host_description()),
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(W, H, world, shard="views"):
    """The SAME dict in both arms (the reference arm renders the same views of the same field with the same settings)."""
    return {
        "workload": f"{W}x{H} sphere-traced colour pass (primary rays, secant refinement, FD normals, colour MLP) of a "
                    "random-init 16^3 KiloNeuS grid (seed 0, MLPs 39-32-32-9 / 41-32-32-3), RenderSettings defaults "
                    "(eps 1e-3, 128 steps, scale 0.8), orbit views r=2.5 el=0.2 fov 40deg (BASELINE config 3)",
        "views_per_step": world if shard == "views" else 1,
        "parallelism": (f"view-sharded x{world}" if shard == "views" else f"one frame per step in interleaved 32-row bands x{world}") +
                       ", field replicated, final all_gather of the colour / depth / normal / hit buffers (overlapped with the next step's render)",
        "preheat": f"{PREHEAT_FRAMES} untimed frames before the warm-up steps (idle B200 clocks need 1-2 s of load to settle)",
        "l2": "no explicit flush: the per-step working set (ray state + request buffers, >400 MB) exceeds the 126 MB L2; "
              "the 45 MB SDF weight blobs are meant to stay L2-resident",
    }


def ncu_route_traffic():
    """Measured DRAM bytes per frame of the emit / scan / scatter kernels (profiles/ncu_traffic.json "route"), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh).get("route")
    except Exception:
        return None


def ncu_traffic(which: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture (profiles/ncu_traffic.json:
    {"filter": {"kernel": ..., "dram_bytes_per_launch": ...}, ...}); None when absent or captured from another kernel."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            ent = json.load(fh).get(which)
        if ent and (which != "filter" or ent.get("kernel") == filter_kernel_name()):
            return float(ent["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


_FILTER_KERNEL = {"name": "march_tc5_kernel"}


def filter_kernel_name():
    return _FILTER_KERNEL["name"]


def _event_ms(fn, warm=1, it=3):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(it):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def other_configs(fs, field, peaks, ffma_peak, tensor_peak):
    """BASELINE.json configs 2, 4 and 5 on one GPU, device-resident, CUDA-event timed (median of 3 after a warm-up).
    Reported next to the headline so every config has a driver-run number; not part of `value`."""
    import torch

    from paper_2206_10885_b200 import cameras, grid, pathtrace, surface
    from paper_2206_10885_b200.modelio import load_model

    out = {}
    dev = fs.dev
    settings = surface.RenderSettings()
    # config 4: batched multi-network forward, uniform points over all cells (cli.py:177-178), per precision mode
    fwd = {}
    for M in (1_000_000, 1 << 24):
        pts = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (M, 3)).astype(np.float32), device=f"cuda:{dev.device}")
        for mode in ("fp32_chain", "tensor_bf16x3", "tensor_fp16x2"):
            try:
                dev.set_precision(mode)
            except Exception:
                continue
            ms = _event_ms(lambda: grid.sdf_query(dev, pts))
            tf = M * FLOP_PER_SDF_EVAL / ms / 1e9
            peak = ffma_peak if mode == "fp32_chain" else tensor_peak
            fwd[f"sdf_{mode}_{M}"] = {"ms": ms, "Gq_per_s": M / ms / 1e6, "tflops": tf, "frac_of_peak": tf / peak,
                                      "peak": peak, "bound": "fp32" if mode == "fp32_chain" else "tensor"}
        dev.set_precision("fp32_chain")
        z = grid.sdf_query(dev, pts).features.contiguous()
        v = torch.nn.functional.normalize(torch.randn(M, 3, device=pts.device), dim=1)
        ms = _event_ms(lambda: grid.color_query(dev, pts, v, v, z))
        tf = M * FLOP_PER_COLOR_EVAL / ms / 1e9
        fwd[f"color_fp32_chain_{M}"] = {"ms": ms, "Gq_per_s": M / ms / 1e6, "tflops": tf, "frac_of_peak": tf / ffma_peak, "peak": ffma_peak, "bound": "fp32"}
        del pts, z, v
    out["config4_batched_forward"] = dict(fwd, note="uniform points over all 4096 cells (244 and 4096 per cell); 5120 / 4864 flop per query; I/O 12 B in + 36 B out (SDF)")
    # config 2: 800x800 orbit, primary rays + normals + colour, 25 of the 100 views (every 4th)
    def orbit(surf, views=25):
        for k in range(views):
            surface.render_rows(surf, cameras.orbit_pose(4 * k, 100, ORBIT_RADIUS, ORBIT_ELEV, FOV, 800, 800), settings, (1, 1, 1), 1, 0, 800, device_out=True)
    ms = _event_ms(lambda: orbit(fs), warm=1, it=1)
    out["config2_orbit_800x800_random_init_16"] = {"views": 25, "ms_total": ms, "fps": 25e3 / ms, "mrays_per_s": 25 * 640000 / ms / 1e3}
    trained = {}
    r8 = os.path.join(ROOT, "tests", "golden", "sphere_stripes_r8_distilled.knf")
    if os.path.exists(r8):
        f8 = load_model(r8)
        # the 12 000-step distilled 8^3 field refined onto the 16^3 grid of the BASELINE configs (same function, 4096 MLPs)
        trained["trained_16_refined_from_r8_distilled"] = surface.FieldSurface(grid.refine_field(f8, 2))
        trained["trained_8_distilled_12k"] = surface.FieldSurface(f8)
    for name, surf in trained.items():
        ms = _event_ms(lambda: orbit(surf), warm=1, it=1)
        out[f"config2_orbit_800x800_{name}"] = {"views": 25, "ms_total": ms, "fps": 25e3 / ms, "mrays_per_s": 25 * 640000 / ms / 1e3}
        pose = orbit_view(3, 1920, 1080)
        surf.dev.reset_stats()
        ms = _event_ms(lambda: surface.render_rows(surf, pose, settings, (1, 1, 1), 1, 0, 1080, device_out=True), warm=2, it=5)
        st = surf.dev.stats()
        out[f"config3_1920x1080_{name}"] = {"ms": ms, "fps": 1e3 / ms, "sdf_evals_per_ray": st["sdf_evals"] / max(st["rays"], 1),
                                            "hit_fraction": st["hits"] / max(st["rays"], 1),
                                            "note": "trained field: rays never crawl, the decision filter switches itself off -- this is the exact FP32 path"}
    # config 5: 3840x2160 path tracing, floor quad + neural object, 1 spp, 8 bounces
    pose = cameras.look_at_pose((0.5, 0.8, 3.2), (0, -0.2, 0), (0, 1, 0), np.deg2rad(45), 3840, 2160)
    quad = pathtrace.QuadObj((-3, -1.0, -3), (6, 0, 0), (0, 0, 6), pathtrace.Lambertian((0.7, 0.7, 0.7)))
    surfs = {"random_init_16": fs}
    surfs.update({k: v for k, v in list(trained.items())[:1]})
    for name, surf in surfs.items():
        scene = pathtrace.Scene([quad, pathtrace.NeuralObject(surf)], pathtrace.ConstantEnv((1, 1, 1)))
        ms = _event_ms(lambda: pathtrace.pathtrace_rows(scene, pose, 1, 0, 8, 0, 0, 2160, device_out=True), warm=1, it=2)
        out[f"config5_pathtrace_3840x2160_spp1_{name}"] = {"ms": ms, "Mpaths_per_s": 3840 * 2160 / ms / 1e3}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="views", choices=["views", "rows"],
                    help="N > 1: one view per rank and step (weak scaling) or one frame per step in interleaved row bands (strong)")
    ap.add_argument("--no-extras", action="store_true", help="skip the other BASELINE configs (2, 4, 5) appended at N = 1")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return 0

    import torch
    import torch.distributed as dist

    from paper_2206_10885_b200 import _native as N  # noqa: F401
    from paper_2206_10885_b200 import dist as kdist
    from paper_2206_10885_b200 import grid, surface

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: there is no CPU fallback for the product path")
    torch.cuda.set_device(local)
    use_dist = world > 1 or "RANK" in os.environ  # under torchrun even a single rank goes through NCCL
    if use_dist:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the communicator / rank log (stdout, before the JSON line, which stays last)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))

    W, H = args.width, args.height
    field = grid.field_init(grid.GridConfig(resolution=16), seed=0)
    fs = surface.FieldSurface(field, device=local)
    _FILTER_KERNEL["name"] = fs.dev.filter_kernel()
    # one-time field set-up beside the upload: the sub-box refinement of the per-cell Lipschitz bounds (csrc/knf_bounds.cuh) that
    # the first filtered march would otherwise trigger; timed here so that the line can report it
    lip_closed, lip_refined, lip_ms = fs.dev.lipschitz()
    settings = surface.RenderSettings()
    dev = torch.device("cuda", local)
    rows_mode = args.shard == "rows" and world > 1
    BAND = 32
    my_bands = kdist.shard_rows_interleaved(H, rank, world, BAND) if rows_mode else [(0, H)]
    my_rows = sum(b[1] - b[0] for b in my_bands)
    bufs = (torch.empty((my_rows, W, 3), dtype=torch.float32, device=dev), torch.empty((my_rows, W), dtype=torch.float32, device=dev),
            torch.empty((my_rows, W, 3), dtype=torch.float32, device=dev), torch.empty((my_rows, W), dtype=torch.uint8, device=dev))
    # one all_gather per step moves all four finished buffers: 29 B per pixel packed into one byte tensor
    PIX_BYTES = 12 + 4 + 12 + 1
    tallest = max(sum(b[1] - b[0] for b in kdist.shard_rows_interleaved(H, r, world, BAND)) for r in range(world)) if rows_mode else H
    # double-buffered: the gather of step s runs on NCCL's stream while step s + 1 renders (frames are independent; the
    # timed region closes with a barrier + synchronize, so every gather it started has finished inside it)
    packed = [torch.empty((tallest * W * PIX_BYTES,), dtype=torch.uint8, device=dev) for _ in range(2)] if use_dist else None
    gathered = [torch.empty((world * tallest * W * PIX_BYTES,), dtype=torch.uint8, device=dev) for _ in range(2)] if use_dist else None
    pending = [None, None]

    def render_mine(view, out):
        at = 0
        for r0, r1 in my_bands:
            sub = tuple(o[at : at + (r1 - r0)] for o in out)
            surface.render_rows(fs, orbit_view(view, W, H), settings, (1.0, 1.0, 1.0), 1, r0, r1, out=sub, device_out=True)
            at += r1 - r0

    def resident_step(s):
        render_mine(s if rows_mode else s * world + rank, bufs)
        if use_dist:
            k = s & 1
            if pending[k] is not None:
                pending[k].wait()  # the gather that last used this buffer pair (two steps ago)
            at = 0
            for b in bufs:
                nb = b.numel() * b.element_size()
                packed[k][at : at + nb].copy_(b.reshape(-1).view(torch.uint8))
                at += nb
            pending[k] = dist.all_gather_into_tensor(gathered[k], packed[k], async_op=True)

    def drain():
        # make the current stream wait for the gathers still in flight (so an event recorded next covers them)
        for k in range(2):
            if pending[k] is not None:
                pending[k].wait()
                pending[k] = None

    def barrier():
        if use_dist:
            drain()
            dist.barrier()
        torch.cuda.synchronize()

    # Pre-heat: a B200 that has been idle needs 1-2 s of sustained load before its SM clock settles at the
    # boost clock (measured: the first 20 frames after a 3-frame warm-up ran at 40-80 ms instead of 32 ms).
    # A fixed frame count keeps the collective call pattern identical on every rank.
    for s in range(PREHEAT_FRAMES):
        resident_step(s)
    barrier()
    fs.dev.set_profiling(True)
    for s in range(args.warmup):
        resident_step(s)
    barrier()
    fs.dev.reset_stats()

    # ---- timed region 1: device-resident frames ------------------------------------------------------
    with ClockSampler(local) as clocks:
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(args.steps):
            resident_step(args.warmup + s)
        drain()
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1)
        if use_dist:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
    stats = fs.dev.stats()
    fs.dev.set_profiling(False)

    # ---- timed region 2: end to end through the NumPy plugin API, host buffers ------------------------
    pinned = (torch.empty((my_rows, W, 3), dtype=torch.float32).pin_memory(), torch.empty((my_rows, W), dtype=torch.float32).pin_memory(),
              torch.empty((my_rows, W, 3), dtype=torch.float32).pin_memory(), torch.empty((my_rows, W), dtype=torch.uint8).pin_memory())
    host_out = tuple(p.numpy() for p in pinned)

    def e2e_step(s):
        at = 0
        for r0, r1 in my_bands:
            sub = tuple(o[at : at + (r1 - r0)] for o in host_out)
            surface.render_rows(fs, orbit_view(s if rows_mode else s * world + rank, W, H), settings, (1.0, 1.0, 1.0), 1, r0, r1, out=sub)
            at += r1 - r0
        return float(host_out[0][my_rows // 2, W // 2, 0])  # touch the host result

    for s in range(2):
        e2e_step(s)
    barrier()
    t0 = time.perf_counter()
    for s in range(args.steps):
        e2e_step(args.warmup + s)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if use_dist:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    final_line = None
    if rank == 0:
        peaks, peak_src = measured_peaks()
        frames_per_step = 1 if rows_mode else world
        fps = args.steps * frames_per_step / (ms / 1e3)
        e2e_fps = args.steps * frames_per_step / e2e_s
        ck = clocks.summary()
        ffma_peak = SM_COUNT * FFMA_LANES_PER_SM * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        tensor_peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0)))
        exact_tflops = stats["sdf_evals"] * FLOP_PER_SDF_EVAL / (stats["sdf_mlp_ms"] * 1e-3) / 1e12 if stats["sdf_mlp_ms"] > 0 else None
        filter_tflops = stats["filter_evals"] * FLOP_PER_SDF_EVAL / (stats["filter_ms"] * 1e-3) / 1e12 if stats["filter_ms"] > 0 else None
        route_bytes = stats["march_routed_requests"] * ROUTE_BYTES_PER_REQUEST + stats["wavefronts"] * 4096 * ROUTE_BYTES_PER_CELL + stats["rays"] * 100
        route_gbs = route_bytes / (stats["route_ms"] * 1e-3) / 1e9 if stats["route_ms"] > 0 else None
        # what the reference evaluates for the same frames: every crawl step the filter decided or certified counts once
        ref_evals = stats["sdf_evals"] + stats["filter_evals"] - stats["filter_deferred"] + stats["filter_skipped"]
        clock_hz = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        roof_exact = {
            "kernel": "march_warp_kernel / march_small_kernel / march_tail_kernel / mlp_warp_kernel (fused encode + 3-layer SDF MLP as k-ordered fp32 FMA chains + NumPy-exact softplus + sphere-trace step)",
            "bound": "fp32", "achieved": exact_tflops, "peak": ffma_peak, "unit": "TFLOP/s", "frac": (exact_tflops / ffma_peak) if exact_tflops else None,
            "peak_source": f"derived: {SM_COUNT} SMs x {FFMA_LANES_PER_SM} FFMA lanes x 2 x sm_max_mhz ({peak_src} MEASURED_PEAKS.json holds HBM and bf16-tensor "
                           "peaks only); measured attainable FP32 rates on this pool: 71.0 TFLOP/s packed FFMA2, 52.0 with one LDS.128 per 16 FFMA2 (profiles/ffma_peak_micro_r1.txt)",
            "evals": int(stats["sdf_evals"]), "launches": int(stats["sdf_mlp_launches"]), "avg_launch_ms": stats["sdf_mlp_ms"] / max(stats["sdf_mlp_launches"], 1),
            "elapsed_share_of_step": stats["sdf_mlp_ms"] / ms, "tile_fill": stats["sdf_evals"] / max(stats["march_lane_slots"], 1),
            "note": "these launches run on a side stream CONCURRENTLY with the filter kernel (sparse, latency-bound tiles): their summed elapsed time overlaps the filter's and "
                    "is not a share of the step; achieved = useful evaluations x 5120 flop over that elapsed time, so it understates the kernels alone "
                    "(dense batched forward, config 4: see configs.config4_batched_forward)",
        }
        tc5 = filter_kernel_name() == "march_tc5_kernel"
        filter_evals_per_s = stats["filter_evals"] / (stats["filter_ms"] * 1e-3) if stats["filter_ms"] > 0 else None
        mufu_per_eval = 64.0 if tc5 else 128.0  # tcgen05 filter: one MUFU.EX2 per softplus (ln(1 + e) is a polynomial); mma.sync filter: ex2 + lg2
        xu_peak_evals = SM_COUNT * 16 * clock_hz / mufu_per_eval  # 16 MUFU lanes per SM and clock
        roof_filter = {
            "kernel": ("march_tc5_kernel (decision filter: Fourier features + fp16x2 operand split in the threads, tcgen05.mma M128 N64/N32 K16 issued by one thread, "
                       "accumulators in TMEM read back with tcgen05.ld, MUFU softplus, sphere-trace crawl step + certified skipping)") if tc5 else
                      "march_mma_kernel<2, filter> (decision filter on mma.sync.m16n8k16)",
            "bound": "tensor", "achieved": filter_tflops, "peak": tensor_peak, "unit": "TFLOP/s", "frac": (filter_tflops / tensor_peak) if filter_tflops else None,
            "traffic": ncu_traffic("filter"),
            "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per dense launch of the filter kernel, from the committed ncu --set full capture "
                            "(profiles/ncu_traffic.json; null when that file holds another kernel than the one this build runs); weights and ray state are L2-resident",
            "peak_source": f"{peak_src} MEASURED_PEAKS.json bf16_tflops_sustained (cuBLAS, tcgen05 path)",
            "algorithmic_flop_per_launch": stats["filter_evals"] * FLOP_PER_SDF_EVAL / max(stats["filter_launches"], 1),
            "avg_launch_ms": stats["filter_ms"] / max(stats["filter_launches"], 1), "launches": int(stats["filter_launches"]),
            "share_of_step": stats["filter_ms"] / ms,
            "tensor_flop_issued_per_eval": 15360,
            "tensor_issued_tflops": (stats["filter_evals"] * 15360 / (stats["filter_ms"] * 1e-3) / 1e12) if stats["filter_ms"] > 0 else None,
            "evals_per_s": filter_evals_per_s,
            "binding_pipe": {"name": "instruction issue (CUDA-core work around the MMAs: 64 softplus, 71 operand splits, 39 Fourier features, the fp64 march step and the certified-skip runs)",
                             "issue_slots_busy_ncu": 0.51, "fma_pipe_busy_ncu": 0.35, "alu_pipe_busy_ncu": 0.27, "xu_pipe_busy_ncu": 0.27, "tensor_pipe_busy_ncu": 0.09,
                             "top_stalls_per_issue_ncu": {"barrier": 2.72, "wait": 1.68, "long_scoreboard": 1.49},
                             "xu_roof_evals_per_s": xu_peak_evals, "frac_of_xu_roof": (filter_evals_per_s / xu_peak_evals) if filter_evals_per_s else None,
                             "note": "ncu --set full of a dense launch (profiles/ncu_r2_final2_tc5_filter.summary.txt): ~1200 CUDA-core instructions per evaluation surround 10 "
                                     "tcgen05.mma per 128 evaluations, and since the refined Lipschitz bounds each evaluation is followed by ~9 certified crawl steps "
                                     "(closed-form run + per-sample checks) that cost issue slots and no flop -- the fraction of tensor peak is not what limits this kernel"},
            "certified_steps_per_evaluation": stats["filter_skipped"] / max(stats["filter_evals"], 1),
            "note": "achieved = filter evaluations x 5120 algorithmic flop / summed CUDA-event time of the filter launches; each evaluation issues 3 fp16 piece products "
                    "over K padded to 48 + 32 (15360 tensor flop); the certified steps the same launches take without evaluating are NOT counted as flop",
        }
        dominant = roof_filter if stats["filter_ms"] >= 0.3 * ms else roof_exact  # the exact launches overlap the filter's: their elapsed sum is not a share
        line = {
            "metric": f"fps_{W}x{H}_sphere_traced", "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong" if rows_mode else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload_config(W, H, world, args.shard),
            "engine": {"precision": fs.dev.get_precision(), "decision_filter": "auto (results bit-identical to filter off)",
                       "filter_kernel": filter_kernel_name()},
            "mrays_per_s": fps * W * H / 1e6,
            "sdf_evals_per_s": ref_evals * world / (ms / 1e3),
            "sdf_evals_per_ray": ref_evals / max(stats["rays"], 1),
            "sdf_evals_executed_per_s": (stats["sdf_evals"] + stats["filter_evals"]) * world / (ms / 1e3),  # network evaluations actually run (exact + filter)
            "sdf_evals_breakdown": {"exact_fp32_chain": int(stats["sdf_evals"]), "filter_tensor": int(stats["filter_evals"]),
                                    "filter_undecided_re_evaluated": int(stats["filter_deferred"]), "certified_without_evaluation": int(stats["filter_skipped"]),
                                    "note": "sdf_evals_per_s / per_ray count what the reference evaluates for these frames (exact + filter - undecided + certified)"},
            "hit_fraction": stats["hits"] / max(stats["rays"], 1),
            "clocks": ck,
            "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": 160 * world * len(my_bands),
                    "d2h_bytes_per_step": int(sum(a.nbytes for a in host_out)) * world,
                    "note": "surface.render_frame-equivalent C-ABI call (KNF_MEM_HOST) into pinned host buffers; the only "
                            "per-step input is the camera/settings structs, the field is uploaded once like the reference loads it once"},
            "gpu_launches": int(stats["kernel_launches"]),
            "field_setup": {"lipschitz_refinement_ms": lip_ms, "closed_form_over_refined_bound": float(np.mean(lip_closed / lip_refined)),
                            "note": "once per field handle, outside the timed regions like the weight upload: per-cell Lipschitz bounds of the SDF networks by sub-box bound "
                                    "propagation (lip_bound_kernel); certified skipping reaches that many times further than with the closed-form bounds"},
            "roofline": dominant,
            "roofline_exact": roof_exact,
            "roofline_filter": roof_filter,
            "roofline_route": {
                "kernel": "march_init (emit) / route_scan / route_scatter", "bound": "hbm", "achieved": route_gbs,
                "algorithmic_bytes": "16.25 B per routed request + 16 B per cell per wavefront + 100 B per ray (init: t_near/t_far/o/d read, state + request written)",
                "routed_fraction_of_march_evals": stats["march_routed_requests"] / max(ref_evals, 1),
                "peak": float(peaks["hbm_gbs"]), "unit": "GB/s", "frac": (route_gbs / float(peaks["hbm_gbs"])) if route_gbs else None,
                "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs", "share_of_step": stats["route_ms"] / ms,
                "launches": int(stats["route_launches"]),
                "traffic": (ncu_route_traffic() or {}).get("dram_bytes_per_step"),
                "traffic_per_kernel_ncu": (ncu_route_traffic() or {}).get("per_kernel"),
                "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per 1080p frame of march_init / route_scan2 / route_scatter2 from the committed ncu capture "
                                "(profiles/route_traffic_r2_final.csv): march_init streams at 2.5 TB/s (39 % of the HBM peak), the scatter at 1.2 TB/s, the scans are "
                                "one-CTA latency-bound launches (8.7 us each)",
            },
        }
        if world == 1 and not args.no_extras:
            line["configs"] = other_configs(fs, field, peaks, ffma_peak, tensor_peak)
        if world == 1 and not args.no_cpu_baseline:
            # the reference's own renderer on this box's host cores, one bounded raster at 1 thread and at all cores
            w, h = 384, 216
            ncpu = os.cpu_count() or 1
            dt1, kind, _ = cpu_frame_seconds(w, h, args.warmup, 1)
            dtn, kind, _ = cpu_frame_seconds(w, h, args.warmup, ncpu)
            best, cores = (dt1, 1) if dt1 <= dtn else (dtn, ncpu)
            line["cpu_baseline"] = dict({"value": w * h / best / (W * H), "unit": "frames/s", "cores": cores, "kind": kind,
                                         "sample": f"one {w}x{h} frame of the same camera/field by "
                                                   f"{'kilofield.surface.render_frame (unmodified reference, oracle/_ref)' if kind == 'reference' else 'oracle.render (port)'}: "
                                                   f"{dt1:.1f} s at KNF_THREADS=1, {dtn:.1f} s at KNF_THREADS={ncpu}; scaled per ray to {W}x{H} "
                                                   "(bench.py --impl reference renders the full frame un-extrapolated)",
                                         "krays_per_s_1_thread": w * h / dt1 / 1e3, "krays_per_s_all_threads": w * h / dtn / 1e3}, **host_description())
        final_line = json.dumps(line)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        sys.stdout.flush()
        print(final_line, flush=True)  # after the process group is gone: the JSON line is the last thing on stdout (NCCL's INFO log comes before)
    return 0


if __name__ == "__main__":
    sys.exit(main())
