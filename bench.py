#!/usr/bin/env python
"""Frame-render benchmark of the B200-native ray tracer (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one frame of the workload `--config` (default C2: the paper's
benchmark scene, 1280x720, 200 soft-shadow samples, 3 reflection bounces —
BASELINE.json configs[1]).  `value` is frames/s with the scene resident in
HBM (device-timed render kernels, CUDA events on the launching stream,
L2 flushed between frames); `e2e` is frames/s through the public
`render_frame` into a host Framebuffer (the reference's call, bench.py:65-78
methodology: wall clock around the synchronous call, frame copied back).
With N > 1 (torchrun, one process per GPU) every rank renders its
interleaved 8-row blocks straight into rank 0's framebuffer over NVLink
(CUDA IPC), and the step time is the max over ranks.

`--impl reference` times the reference algorithm on the host CPU: the
float64 C port of `render_frame` (oracle/, bit-identical to the reference's
numba path) with every host thread, on a bounded row sample of the same
workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # SMs x FP32 lanes x FMA x max SM clock
# instruction issue: 148 SMs x 4 schedulers x 1 warp instruction per cycle at 1965 MHz
ISSUE_PEAK_WARP_INST_PER_S = 148 * 4 * 1.965e9
L2_FLUSH_BYTES = 256 << 20
EXTRA_CONFIGS = ("C1", "P720", "P1080", "P4K", "C3", "C4", "C5", "C5_512")


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default=None, help="workload (default: C2 on one GPU, C4 in row bands on several)")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--no-extra", action="store_true", help="skip the other configurations' fps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU-baseline sample budget")
    return ap.parse_args(argv)


def work_counts():
    with open(os.path.join(ROOT, "paper_2305_07450_b200", "work_counts.json")) as f:
        return json.load(f)["configs"]


# --- clocks during the timed region ------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax = float(parts[2])
                except ValueError:
                    continue
                for name, flag in zip(names, parts[5:9]):
                    if flag.lower() == "active":
                        reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# --- CPU: the reference algorithm on the host cores -------------------------------
def cpu_reference_sample(cfg, budget_s, threads=0):
    """Time the float64 C port of render_frame (oracle/, bit-identical to the
    reference) on every `step`-th row of the workload; returns frames/s."""
    import oracle
    from paper_2305_07450_b200 import pack_scene

    scene, cam = cfg.scene(), cfg.camera()
    ps = vars(pack_scene(scene))

    def run(step):
        t = time.perf_counter()
        oracle.render(ps, cam.position, cam.yaw, cam.pitch, cam.fov, cfg.width, cfg.height, cfg.samples, cfg.bounces,
                      row0=step // 2, row_step=step, threads=threads)
        return time.perf_counter() - t

    step = max(1, cfg.height // 8)
    dt = run(step)
    # rows sampled scale linearly: pick the stride that fills the budget
    rows = len(range(step // 2, cfg.height, step))
    per_row = dt / rows
    want_rows = max(1, int(budget_s / max(per_row, 1e-9)))
    if want_rows >= cfg.height:  # whole frames fit: render as many as the budget allows
        frames = max(1, min(100, int(want_rows / cfg.height)))
        t = time.perf_counter()
        for _ in range(frames):
            run(1)
        dt = time.perf_counter() - t
        return frames / dt, dict(rows=cfg.height * frames, row_step=1, frames=frames, seconds=dt,
                                 threads=threads or oracle.max_threads())
    step = max(1, cfg.height // want_rows)
    dt = run(step)
    rows = len(range(step // 2, cfg.height, step))
    frac = rows / cfg.height
    return frac / dt, dict(rows=rows, row_step=step, frames=0, seconds=dt, threads=threads or oracle.max_threads())


def run_reference(args):
    from paper_2305_07450_b200 import CONFIGS
    import oracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # the same workload as this run's own arm (run_ours)
    args.config = args.config or ("C2" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "C4")
    cfg = CONFIGS[args.config]
    threads = oracle.max_threads()
    per_step = max(2.0, args.cpu_seconds / max(1, args.steps))
    vals = []
    meta = None
    for i in range(args.warmup + args.steps):
        budget = 0.5 if i < args.warmup else per_step
        v, meta_i = cpu_reference_sample(cfg, budget, threads)
        if i >= args.warmup:
            vals.append(v)
            meta = meta_i
    fps = statistics.mean(vals)
    wc = work_counts()[args.config]
    what = (f"{meta['frames']} whole frames" if meta["frames"] else
            f"every {meta['row_step']}th row ({meta['rows']} of {cfg.height} rows)")
    sample = (f"{what} of {cfg.name} per step, float64 C port of render_frame (oracle/rt_oracle.c, "
              f"bit-identical to the reference), OpenMP dynamic rows")
    line = {
        "impl": "reference",
        "metric": "frames/s",
        "value": fps,
        "unit": "frames/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 / fps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (the paper's benchmark scene, sceneio.py:314-333)",
        "config": {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "samples": cfg.samples,
                   "bounces": cfg.bounces, "sky": cfg.sky},
        "mrays_per_s": wc["rays"] * fps / 1e6,
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": meta["threads"], "kind": "port",
                         "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    # the reference's own numba render_frame on the same cores, for context:
    # the C port above is the conservative (faster) stand-in
    nb = numba_reference(args.config)
    if nb:
        line["numba_reference"] = nb
    print(json.dumps(line), flush=True)
    return 0


# --- GPU ----------------------------------------------------------------------------
def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


# CPU baseline protocol per configuration: the paper's 100
# warm-up + 10 measured frames (reference bench.py:24-25) where a CPU frame
# is short, 1 + 3 whole frames for the soft-shadow configurations, and C5 on
# a 384x216 frame scaled by the pixel count (a 4K C5 frame is ~20 CPU-minutes)
CPU_PROTOCOL = {"C1": (100, 10, None), "P720": (100, 10, None), "P1080": (100, 10, None), "P4K": (100, 10, None),
                "C2": (1, 3, None), "C3": (1, 3, None), "C4": (1, 3, None), "C5": (1, 3, (384, 216)),
                "C5_512": (1, 3, (384, 216))}


# whole frames of the reference's numba render_frame timed per extra configuration (no-sky rows only:
# the reference's sceneio builds them; ~2-20 s each on 16 cores)
NUMBA_FRAMES = {"C1": 10, "P720": 10, "P1080": 5, "P4K": 2}


def numba_reference(key, frames=2, timeout=240):
    """The unmodified reference's own render_frame (numba, pip-installed into
    baseline/_ref) on all host cores, in a subprocess (tools/
    numba_reference_time.py): whole frames after the JIT warm-up.  None when
    the reference is not installed or the configuration has no counterpart
    built by the reference's sceneio (skybox configurations)."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "raytracer")):
        return None
    try:
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "numba_reference_time.py"), key,
                              str(frames)], capture_output=True, text=True, timeout=timeout, cwd=ROOT)
        lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
        return json.loads(lines[-1]) if out.returncode == 0 and lines else None
    except (subprocess.TimeoutExpired, OSError, ValueError):
        return None


def cpu_frames(key, threads=0):
    """The reference algorithm (float64 C port of render_frame, oracle/,
    bit-identical to the reference) on the host cores, per CPU_PROTOCOL."""
    import oracle
    from paper_2305_07450_b200 import CONFIGS, pack_scene

    cfg = CONFIGS[key]
    warm, meas, sub = CPU_PROTOCOL[key]
    w, h = sub or (cfg.width, cfg.height)
    scene, cam = cfg.scene(), cfg.camera()
    ps = vars(pack_scene(scene))

    def one():
        oracle.render(ps, cam.position, cam.yaw, cam.pitch, cam.fov, w, h, cfg.samples, cfg.bounces, threads=threads)

    for _ in range(warm):
        one()
    t = time.perf_counter()
    for _ in range(meas):
        one()
    dt = time.perf_counter() - t
    scale = (w * h) / (cfg.width * cfg.height)
    fps = meas / dt * scale
    what = f"{warm} warm-up + {meas} measured frames"
    if sub:
        what += f" at {w}x{h}, scaled by the pixel count to {cfg.width}x{cfg.height}"
    return fps, {"value": fps, "unit": "frames/s", "cores": threads or oracle.max_threads(), "kind": "port",
                 "sample": f"{what} of {cfg.name}; float64 C port of render_frame (oracle/rt_oracle.c, "
                           f"bit-identical to the reference), OpenMP dynamic rows, {dt:.1f} s"}


def run_ours(args):
    import numpy as np
    import torch

    import paper_2305_07450_b200 as rt
    from paper_2305_07450_b200 import _native, bands

    world, rank, local = _dist_env()
    if world != args.gpus:
        args.gpus = world
    # the headline workload: BASELINE.json configs[1] (C2) on one GPU; with
    # several, configs[3] (C4, 4K) split in row bands across them
    key = args.config or ("C2" if world == 1 else "C4")
    # B200RT_BENCH_SHARE_GPU=1: every rank on GPU 0 with host (gloo)
    # collectives — a functional check of the N > 1 code path on a one-GPU
    # box (no kernel waits on another rank's), never a measurement
    share = world > 1 and os.environ.get("B200RT_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    lib = _native.load()
    ctx = _native.Context((local,))
    cfg = rt.CONFIGS[key]
    prec = _native.PRECISIONS[args.precision]
    wc = work_counts()

    def set_scene(scene):
        ps = rt.pack_scene(scene)
        P = _native.ptr
        _native.check(lib.rt_set_scene_v1(ctx.handle, ps.n_bodies, P(ps.kinds), P(ps.positions), P(ps.sizes),
                                          P(ps.colors), P(ps.refls), P(ps.light_pos), ps.light_radius,
                                          P(ps.light_color), ps.ambient, ps.max_refl, P(ps.sky), ps.sky_w, ps.sky_h,
                                          int(ps.has_sky)), "rt_set_scene_v1")
        return ps

    # a dedicated stream: the legacy default stream's handle is NULL, which the
    # C ABI reads as "the library's own stream" (not ordered with our events)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)

    # framebuffer: rank 0 owns it (sized for the largest frame measured);
    # other ranks map it over NVLink (CUDA IPC) and render their rows into it
    extra_keys = () if (args.no_extra or world > 1) else tuple(k for k in EXTRA_CONFIGS if k != key)
    size_keys = (key, *extra_keys, "C2", "C4")
    max_px = max(rt.CONFIGS[k].width * rt.CONFIGS[k].height for k in size_keys)
    exchange = bands.torch_exchange if world > 1 else (lambda blob: blob)
    ipc = bands.IpcFrame(local, 1, max_px, rank, exchange)
    fb_ptr = ipc.ptr
    tiny = torch.zeros(1, device=dev)
    d_local = ctypes.c_void_p()
    if world > 1:  # each rank's own device frame (whole-frame sharding, shared-host-frame gather)
        _native.check(lib.rt_device_malloc(local, 4 * max_px, ctypes.byref(d_local)), "rt_device_malloc")
    cur = {"prec": prec, "mode": "bands" if world > 1 else "frames"}

    def render_cfg(c, part=None, n_parts=None, out=None, sync=True):
        bands_mode = world > 1 and cur["mode"] == "bands"
        if part is None:
            part, n_parts = (rank, world) if bands_mode else (0, 1)
        if out is None:
            out = fb_ptr if (world == 1 or bands_mode) else d_local
        cam = c.camera()
        cp = np.array(cam.position, dtype=np.float64)
        rc = lib.rt_render_device_v1(ctx.handle, 0, out, c.width, None, c.width, c.height, _native.ptr(cp),
                                     float(cam.yaw), float(cam.pitch), rt.camera_viewport_distance(cam.fov),
                                     c.samples, c.bounces, part, n_parts, 8, cur["prec"],
                                     ctypes.c_void_p(stream.cuda_stream))
        _native.check(rc, "rt_render_device_v1")
        if bands_mode and sync:
            import torch.distributed as dist
            dist.all_reduce(tiny)  # completes once every rank's rows have landed in rank 0's frame

    def time_config(c, warmup, steps, sample_clocks=False):
        set_scene(c.scene())
        for _ in range(warmup):
            render_cfg(c)
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        clocks = None
        if sample_clocks:  # nvidia-smi samples every 100 ms: keep the GPU loaded >= 1 s around the region
            clocks = ClockSampler(local).start()
            t_load = time.perf_counter()
            while time.perf_counter() - t_load < 1.0:
                for _ in range(8):
                    render_cfg(c)
                torch.cuda.synchronize()
        n0 = ctx.launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for e0, e1 in evs:
            flush.zero_()  # L2 flush between frames (outside the event pair)
            e0.record(stream)
            render_cfg(c)
            e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        launches = ctx.launch_count() - n0
        if clocks:
            t_load = time.perf_counter()
            while time.perf_counter() - t_load < 0.5:
                for _ in range(8):
                    render_cfg(c)
                torch.cuda.synchronize()
        clk = clocks.stop() if clocks else None
        ms = [a.elapsed_time(b) for a, b in evs]
        total = sum(ms)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([total], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total = float(t.item())
        return dict(ms=ms, total_ms=total, wall_s=wall, launches=launches, clocks=clk)

    def measure(c, warmup, steps, sample_clocks=False):
        """Frames/s, per-kernel device shares and executed work of config c."""
        r = time_config(c, warmup, steps, sample_clocks)
        # whole-job frames/s: every rank rendered len(ms) whole frames
        # ("frames" mode), or the ranks rendered len(ms) frames together ("bands")
        per = world if (world > 1 and cur["mode"] == "frames") else 1
        fps_c = per * len(r["ms"]) / (r["total_ms"] / 1e3)
        # per-kernel shares: CUDA events between the kernels on their launch
        # stream, averaged over as many frames as were timed (events cost
        # ~2.5 us each, so they stay out of the timed region itself)
        ctx.set_option("phases", 1)
        acc = {}
        n_ph = max(3, min(steps, 50))
        for _ in range(n_ph):
            render_cfg(c)
            torch.cuda.synchronize()
            for k, v in ctx.phase_ms().items():
                acc[k] = acc.get(k, 0.0) + v / n_ph
        ctx.set_option("phases", 0)
        ctx.set_option("count_work", 1)
        ctx.work_counts(reset=True)
        render_cfg(c)
        torch.cuda.synchronize()
        work = ctx.work_counts(reset=True)
        ctx.set_option("count_work", 0)
        return r, fps_c, acc, work

    def e2e_sync(c, steps):
        """render_frame (the reference's call) into a host Framebuffer, a new
        camera every step; wall clock around each synchronous call."""
        scene, cam, params = c.scene(), c.camera(), c.params()
        fb = rt.Framebuffer.create(c.width, c.height)
        for _ in range(max(3, args.warmup)):
            rt.render_frame(scene, cam, params, fb, precision=args.precision)
        # every step a new camera (the frame loop's moving view): the scene
        # arrays and camera cross the C ABI, the library compares the scene
        # (and the sky's texels) with its copies and uploads only what changed
        cams = [rt.Camera(position=cam.position, yaw=cam.yaw + 1e-4 * (i % 2), pitch=cam.pitch, fov=cam.fov)
                for i in range(2)]
        ts = []
        d2h = 0
        ctx1 = _native.context(1)
        for i in range(steps):
            t = time.perf_counter()
            rt.render_frame(scene, cams[i % 2], params, fb, precision=args.precision)
            ts.append(time.perf_counter() - t)
            d2h += ctx1.last_d2h_bytes()  # (outside the timed call)
        ps = rt.pack_scene(scene)
        # kinds, positions, sizes, colours, reflectivities, light, ambient, max_refl + camera (f64, i32)
        h2d = int(4 * len(ps.kinds) + 8 * (3 + 1 + 3 + 1) * len(ps.kinds) + 8 * (3 + 1 + 3 + 2) + 8 * 6)
        codec = bool(_native.get_options().get("codec", 1))
        return {"value": steps / sum(ts), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h // steps, "d2h_frame_bytes": 4 * c.width * c.height,
                "ms_per_step": 1e3 * statistics.mean(ts), "ms_median": 1e3 * statistics.median(ts),
                "transfer": ("compressed (option codec): the encode kernel's row runs into mapped host memory, "
                             "expanded by host threads into the framebuffer, bit-exact; d2h_bytes_per_step as "
                             "moved over PCIe (rt_last_d2h_bytes)") if codec else "raw frame copy",
                "path": "paper_2305_07450_b200.render_frame -> rt_render_v1 (C ABI), host framebuffer"}

    line = {"metric": "frames/s", "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "f64",
            "data": "synthetic (the paper's benchmark scene and camera, sceneio.py:314-333)"}
    if world == 1:
        # headline: device-resident frames/s on the default path (wavefront + exact culling)
        main, fps, phases, work = measure(cfg, max(3, args.warmup), args.steps, sample_clocks=True)
        ms_frame = statistics.mean(main["ms"])
        wcc = wc[key]
        peak_meas = _native.fp32_peak_tflops(local)
        roof = roofline(wcc, phases, work, ms_frame, cfg.samples, peak_meas, config_key=key)
        e2e = e2e_sync(cfg, args.steps)
        # the same call with the frame copied raw (option codec off), for comparison
        _native.set_options(codec=0)
        raw = e2e_sync(cfg, args.steps)
        _native.set_options(codec=1)
        e2e["raw_copy"] = {k: raw[k] for k in ("value", "unit", "d2h_bytes_per_step", "ms_median")}
        # the frame server's loop: frames back to back through FramePipeline,
        # each frame's copy overlapping the next frame's kernels; every frame
        # still lands whole in a host framebuffer before it is counted
        scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
        cams = [rt.Camera(position=cam.position, yaw=cam.yaw + 1e-4 * (i % 2), pitch=cam.pitch, fov=cam.fov)
                for i in range(2)]
        depth = 3
        pipe = rt.FramePipeline(depth, precision=args.precision)
        fbs = [rt.Framebuffer.create(cfg.width, cfg.height) for _ in range(depth)]
        for i in range(max(3, args.warmup)):
            pipe.submit(scene, cam, params, fbs[i % depth])
        pipe.drain()
        t = time.perf_counter()
        for i in range(args.steps):
            pipe.submit(scene, cams[i % 2], params, fbs[i % depth])
        pipe.drain()
        dt = time.perf_counter() - t
        pipe_d2h = pipe.ctx.last_d2h_bytes()  # (the last frame's)
        pipe.close()
        e2e["pipelined"] = {"value": args.steps / dt, "unit": "frames/s",
                            "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                            "d2h_bytes_per_step": pipe_d2h, "ms_per_step": 1e3 * dt / args.steps,
                            "path": "paper_2305_07450_b200.FramePipeline (rt_render_async_v1 / rt_frame_wait_v1), "
                                    "depth 3, host framebuffers"}
        line.update({
            "value": fps, "ms_per_step": main["total_ms"] / args.steps, "scaling": "weak",
            # config: the workload keys both arms share (--impl reference prints the same)
            "config": {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "samples": cfg.samples,
                       "bounces": cfg.bounces, "sky": cfg.sky},
            "run": {"parallelism": "one GPU", "path": "wavefront + exact per-hit occluder culling (default)",
                    "l2": "flushed between timed frames (256 MiB memset outside the event pair)"},
            **ray_rates(wcc, work, fps),
            "mrays_definition": "reference_equivalent: the rays the reference's control flow traces for the frame "
                                "(closest-hit + every shadow sample) / time; executed: closest-hit rays + the shadow "
                                "rays the culled pass sampled",
            "e2e": e2e, "gpu_launches": main["launches"], "clocks": main["clocks"], "roofline": roof,
            "framebuffer_write": framebuffer_writes(cfg, main["total_ms"] / args.steps, key),
            "phases_ms": phases, "executed_work": work})
        if not args.no_extra:
            extra = {}
            for k in extra_keys:
                c = rt.CONFIGS[k]
                r, f, ph, wk = measure(c, 3, 10 if k not in ("C4", "C5", "C5_512") else 5)
                km = statistics.mean(r["ms"])
                extra[k] = {"workload": c.name, "fps": f, "ms_per_frame": km, **ray_rates(wc[k], wk, f),
                            "phases_ms": ph,
                            "roofline": roofline(wc[k], ph, wk, km, c.samples, peak_meas, config_key=k),
                            "e2e": e2e_sync(c, 10 if c.width * c.height < 4_000_000 else 5)}
                if k in rt.workloads.PAPER_FPS:
                    extra[k]["paper_fps_rtx2060"] = rt.workloads.PAPER_FPS[k]
                if not args.no_cpu_baseline and k in CPU_PROTOCOL:
                    extra[k]["cpu_baseline"] = cpu_frames(k)[1]
                    nb = numba_reference(k, frames=NUMBA_FRAMES.get(k, 0)) if k in NUMBA_FRAMES else None
                    if nb:  # the reference's own numba render_frame on the same cores
                        extra[k]["cpu_baseline"]["numba_reference"] = nb
            # ablation on the headline config: the same frame without culling, and as one megakernel
            for name, opts in (("no_cull", dict(wave=1, cull=0)), ("megakernel", dict(wave=0, cull=0))):
                for o, v in opts.items():
                    ctx.set_option(o, v)
                r, f, ph, wk = measure(cfg, 3, args.steps)
                km = statistics.mean(r["ms"])
                extra[f"{key}_{name}"] = {"fps": f, "ms_per_frame": km, "phases_ms": ph,
                                          "roofline": roofline(wcc, ph, wk, km, cfg.samples, peak_meas,
                                                               culled=False)}
            for o, v in dict(wave=1, cull=1).items():
                ctx.set_option(o, v)
            # the bit-identical mode (float64 in the reference's operation order)
            cur["prec"] = _native.RT_PREC_FP64
            for k in (key, "P720", "P1080", "P4K"):
                c = rt.CONFIGS[k]
                r = time_config(c, 3, 10)
                f = len(r["ms"]) / (r["total_ms"] / 1e3)
                extra[f"{k}_fp64_bit_exact"] = {"workload": c.name, "fps": f, "ms_per_frame": statistics.mean(r["ms"]),
                                                "precision": "fp64, bit-identical to the reference"}
            cur["prec"] = prec
            line["extra"] = extra
        if not args.no_cpu_baseline:
            if key in CPU_PROTOCOL:
                line["cpu_baseline"] = cpu_frames(key)[1]
                nb = numba_reference(key)
                if nb:  # the reference's own numba render_frame on the same cores
                    line["cpu_baseline"]["numba_reference"] = nb
            else:
                v, meta = cpu_reference_sample(cfg, args.cpu_seconds)
                line["cpu_baseline"] = {"value": v, "unit": "frames/s", "cores": meta["threads"], "kind": "port",
                                        "sample": f"{meta['rows']} rows of {cfg.name}"}
    else:
        import torch.distributed as dist

        # headline: one frame of C4 in row bands (8-row blocks round-robin,
        # SURVEY.md §8e), every rank storing its rows into rank 0's device
        # frame over NVLink (CUDA IPC) — the gather fused into the render; the
        # all-reduce completes once every band has landed (strong scaling)
        cur["mode"] = "bands"
        main, fps, phases, work = measure(cfg, max(3, args.warmup), args.steps, sample_clocks=True)
        peak_meas = _native.fp32_peak_tflops(local)
        # per GPU: rank 0's kernels did ~1/world of the frame's work (balanced
        # row blocks) in its frame time
        work_frame = {k: v * world for k, v in work.items()}
        roof = roofline(wc[key], phases, work_frame, world * statistics.mean(main["ms"]), cfg.samples, peak_meas,
                        config_key=key)
        roof["per"] = "GPU (rank 0's share of the frame)"
        frame_bytes = 4 * cfg.width * cfg.height

        def e2e_run(step, frames_per_step):
            ts = []
            for i in range(max(3, args.warmup) + args.steps):
                dist.barrier()
                t = time.perf_counter()
                step()
                torch.cuda.synchronize()
                dist.barrier()
                if i >= max(3, args.warmup):
                    ts.append(time.perf_counter() - t)
            t = torch.tensor([sum(ts)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return frames_per_step * args.steps / float(t.item())

        # e2e (1): every rank renders its rows into its own device frame and
        # copies them into a page-locked host frame shared by the node's ranks
        # over its own PCIe link — the frame is whole in host
        # memory when the closing barrier passes
        set_scene(cfg.scene())
        shm = bands.ShmFrame(ctx, cfg.width, cfg.height, rank, bands.torch_exchange)

        def shm_step():
            render_cfg(cfg, part=rank, n_parts=world, out=d_local, sync=False)
            shm.copy_rows(d_local, rank, world, ctypes.c_void_p(stream.cuda_stream))

        fps_shm = e2e_run(shm_step, 1)
        # e2e (2): the NVLink gather into rank 0's device frame + one D2H on rank 0
        host = torch.empty(cfg.width * cfg.height, dtype=torch.int32, pin_memory=True) if rank == 0 else None

        def ipc_step():
            render_cfg(cfg)  # its all-reduce orders "every band landed"
            if rank == 0:
                _native.check(lib.rt_copy_to_host(ctx.handle, 0, ctypes.c_void_p(host.data_ptr()), fb_ptr,
                                                  frame_bytes, ctypes.c_void_p(stream.cuda_stream)),
                              "rt_copy_to_host")

        fps_ipc = e2e_run(ipc_step, 1)
        # both host frames against one GPU rendering the whole frame
        ok_shm = ok_ipc = True
        if rank == 0:
            ref = np.empty(cfg.width * cfg.height, dtype=np.uint32)
            render_cfg(cfg, part=0, n_parts=1, out=d_local, sync=False)
            _native.check(lib.rt_copy_to_host(ctx.handle, 0, _native.ptr(ref), d_local, frame_bytes,
                                              ctypes.c_void_p(stream.cuda_stream)), "rt_copy_to_host")
        dist.barrier()
        if rank == 0:
            ok_shm = bool(np.array_equal(ref, shm.pixels))
            ok_ipc = bool(np.array_equal(ref, host.numpy().view(np.uint32)))
        shm.close()
        e2e = {"value": fps_shm, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": frame_bytes,
               "path": f"one {cfg.name} frame in row bands over {world} ranks (rt_render_device_v1), each rank's rows "
                       "copied into a page-locked host frame shared by the ranks over its own PCIe link "
                       "(rt_copy_partition_to_host), barrier",
               "frame_matches_single_gpu_render": ok_shm,
               "ipc_gather": {"value": fps_ipc, "unit": "frames/s", "d2h_bytes_per_step": frame_bytes,
                              "path": "row bands stored into rank 0's device frame over NVLink (CUDA IPC) + one D2H "
                                      "on rank 0",
                              "frame_matches_single_gpu_render": ok_ipc}}
        # whole frames sharded across the GPUs (each rank its own frames, no
        # collective: weak scaling) — the alternative split, reported alongside
        cur["mode"] = "frames"
        whole = {}
        for k in ("C2", "C4"):
            c = rt.CONFIGS[k]
            r = time_config(c, 3, args.steps)
            whole[k] = {"workload": c.name, "fps": world * len(r["ms"]) / (r["total_ms"] / 1e3),
                        "ms_per_frame": r["total_ms"] / len(r["ms"]), "scaling": "weak",
                        "path": "rt_render_device_v1 whole frames, one per rank per step, no collective"}
        cur["mode"] = "bands"
        line.update({
            "value": fps, "ms_per_step": main["total_ms"] / args.steps, "scaling": "strong",
            "config": {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "samples": cfg.samples,
                       "bounces": cfg.bounces, "sky": cfg.sky},
            "run": {"parallelism": f"row bands x{world} (8-row blocks round-robin), gathered into rank 0's frame "
                                   "over NVLink",
                    "path": "wavefront + exact per-hit occluder culling (default)",
                    "l2": "flushed between timed frames (256 MiB memset outside the event pair)"},
            **ray_rates(wc[key], work, fps),
            "e2e": e2e, "gpu_launches": main["launches"], "clocks": main["clocks"], "roofline": roof,
            "phases_ms": phases, "whole_frames": whole})
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ipc.close()
    if d_local:
        lib.rt_device_free(d_local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


# FLOPs per unit of the SURVEY.md §8d cost model (FMA = 2, add/mul/sqrt/div = 1)
FLOP_SPHERE_TCA = 8     # a sphere test that exits at tca < 0
FLOP_SPHERE_DISC = 17   # ... at the discriminant
FLOP_SPHERE_FULL = 19   # ... evaluated to the end
FLOP_PLANE = 2
FLOP_SHADOW_SETUP = 33  # sample point from the table, normalise, limit (n > 1); 21 for n = 1
FLOP_HIT = 60           # hit point, normal, to-light, Lambert/Blinn inputs
FLOP_BASIS = 39         # disc basis per hit (n > 1)
FLOP_PRIMARY = 36       # primary direction + pack
FLOP_REFLECT = 18
FLOP_SHADE = 45
# units of the culled path (no reference counterpart), weighted by the FP32
# operations of their code (FMA = 2): reconciled against the ncu FP32
# instruction counters in profiles/ncu_flops.json (bench line: model_over_counter)
FLOP_CULL = 40          # one body's cone classification (centre offset, axial/radial split, 2 sqrt, compares)
FLOP_CONIC = 17         # one silhouette-form sample test (|w|^2, x, y, d: 7 FMA + 1 add; culled sampler)
FLOP_CONIC_Z = 4        # its terminator test z > 0 (2 FMA), when the sphere is not wholly in front
FLOP_CONIC_SETUP = 120  # shadow frame, cone and the six coefficients of one (hit, sphere) pair


def _sphere_flops(tca, disc, full):
    return tca * FLOP_SPHERE_TCA + disc * FLOP_SPHERE_DISC + full * FLOP_SPHERE_FULL


def _load_profile(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def roofline(wcc, phases, work, ms_frame, samples, peak, culled=True, config_key=None):
    """Roofline of the dominant kernel: its algorithmic FLOPs (SURVEY.md §8d
    units x the counts of one launch: the reference's control flow, or the
    culled pass's own tallies) over its device time.  The kernels' shares of
    the frame come from CUDA events between them (phases); the kernel time is
    that share of the frame time measured without them, so the events' own
    cost (~2.5 us each) does not inflate it."""
    c = wcc["counts"]
    setup = FLOP_SHADOW_SETUP if samples > 1 else 21
    flops = {
        "trace": _sphere_flops(c["CH_TCA"], c["CH_DISC"], c["CH_FULL"]) + c["CH_PLANE"] * FLOP_PLANE
        + c["HITS"] * FLOP_HIT + c["PIX"] * FLOP_PRIMARY + c["REFL"] * FLOP_REFLECT,
        "shade": c["SHADE"] * FLOP_SHADE,
    }
    if culled and work.get("hits"):
        # the culled (fused) path: the trace kernel classifies its hits; the
        # sampler runs silhouette-form tests, and ray-form ones for the rest
        flops["trace"] += work["cull_tests"] * FLOP_CULL
        flops["classify"] = 0
        conic_hits, conic_tests = work.get("conic_hits", 0), work.get("conic_tests", 0)
        ray_hits = work["sampled_hits"] - conic_hits
        ray_rays = ray_hits * samples
        flops["shadow"] = (conic_tests * FLOP_CONIC + work.get("conic_z_tests", 0) * FLOP_CONIC_Z
                           + conic_hits * FLOP_CONIC_SETUP
                           + ray_rays * setup + ray_hits * (FLOP_BASIS if samples > 1 else 0)
                           + (work["sphere_tests"] - conic_tests) * FLOP_SPHERE_FULL
                           + work["plane_tests"] * FLOP_PLANE)
    else:
        flops["classify"] = 0
        flops["shadow"] = (c["SH_RAYS"] * setup + c["HITS"] * (FLOP_BASIS if samples > 1 else 0)
                           + _sphere_flops(c["SH_TCA"], c["SH_DISC"], c["SH_FULL"]) + c["SH_PLANE"] * FLOP_PLANE)
    real = {k: v for k, v in (phases or {}).items() if v > 0.005}  # phases of a few us are event gaps
    if real:
        total = sum(real.values())
        shares = {k: v / total for k, v in real.items()}
        kernel = max(shares, key=shares.get)
        share = shares[kernel]
        kms = share * ms_frame
    else:  # megakernel: one kernel does everything
        kernel, kms, share = "megakernel", ms_frame, 1.0
        shares = {kernel: 1.0}
        flops = {"megakernel": sum(flops.values())}
    achieved = flops[kernel] / (kms * 1e-3) / 1e12 if kms > 0 else 0.0
    # DRAM traffic per launch of that kernel, from the committed ncu capture
    # (profiles/ncu_traffic.json); null when there is none for this config
    traffic, traffic_src = None, None
    tr = _load_profile("ncu_traffic.json")
    t = tr.get(config_key, {}).get(kernel) if tr else None
    if t:
        traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
        traffic_src = tr.get("_source")
    # executed operations per launch from ncu's instruction counters
    # (profiles/ncu_flops.json): FP32 (FFMA x 2 + FADD + FMUL, the paired
    # forms x 2 per component) plus FP64 (DFMA x 2 + DADD + DMUL) — the trace
    # kernel carries each ray's origin and direction in float64, so part of
    # the model's work runs on the FP64 pipe
    counters = _load_profile("ncu_flops.json").get(config_key, {})
    per_kernel = {}
    for k, sh in shares.items():
        ms = sh * ms_frame
        if flops.get(k) and ms > 0:
            a = flops[k] / (ms * 1e-3) / 1e12
            per_kernel[k] = {"ms": ms, "share_of_frame": sh, "flops": flops[k], "achieved": a,
                             "frac": a / peak if peak else None}
            cf = counters.get(k, {}).get("flops")
            if cf:
                c64 = counters.get(k, {}).get("fp64_ops", 0.0)
                per_kernel[k]["counter_flops"] = cf + c64
                per_kernel[k]["counter_flops_fp32"] = cf
                per_kernel[k]["counter_flops_fp64"] = c64
                per_kernel[k]["counter_achieved"] = (cf + c64) / (ms * 1e-3) / 1e12
                per_kernel[k]["model_over_counter"] = flops[k] / (cf + c64)
            wi = counters.get(k, {}).get("warp_inst")
            if wi:  # the instruction-issue roofline (what bounds a divergent per-pixel chain)
                per_kernel[k]["issue"] = {"warp_inst_per_launch": wi, "achieved": wi / (ms * 1e-3),
                                          "peak": ISSUE_PEAK_WARP_INST_PER_S, "unit": "warp inst/s",
                                          "frac": wi / (ms * 1e-3) / ISSUE_PEAK_WARP_INST_PER_S}
    out = {
        "bound": "fp32",
        "kernel": kernel,
        "achieved": achieved,
        "peak": peak,
        "unit": "TFLOP/s",
        "frac": achieved / peak if peak else None,
        "traffic": traffic,
        "traffic_source": traffic_src,
        "kernel_ms": kms,
        "kernel_share_of_frame": share,
        "flops_per_launch": flops[kernel],
        "flops_definition": "algorithmic: SURVEY.md §8d units (sphere test 8/17/19 by exit, plane 2, hit 60, "
                            "primary 36, reflection 18, shade 45, shadow-ray setup 33) x this launch's counts, "
                            "plus the culled path's own units (cone class 40, silhouette test 17 + 4 with the "
                            "terminator test, its setup 120)",
        "peak_source": "measured dependent-free FFMA stream on this GPU (rt_fp32_peak_tflops); "
                       "MEASURED_PEAKS.json has no FP32 CUDA-core figure",
        "peak_nominal": NOMINAL_FP32_TFLOPS,
        "reference_equivalent_tflops": wcc["flops"] / (ms_frame * 1e-3) / 1e12,
        "kernels": per_kernel,
    }
    if per_kernel.get(kernel, {}).get("counter_flops"):
        out["counter_flops_per_launch"] = per_kernel[kernel]["counter_flops"]
        out["counter_achieved"] = per_kernel[kernel]["counter_achieved"]
        out["model_over_counter"] = per_kernel[kernel]["model_over_counter"]
        out["counter_source"] = counters.get("_source") or _load_profile("ncu_flops.json").get("_source")
    if per_kernel.get(kernel, {}).get("issue"):
        # beside the FP32 roofline: the same kernel against instruction issue
        # (148 SMs x 4 schedulers x 1 warp instruction per cycle) — its FP32
        # fraction is bounded by its instruction mix, its issue
        # fraction by latency
        iss = per_kernel[kernel]["issue"]
        out["issue_roofline"] = {"bound": "instruction issue", "kernel": kernel, "achieved": iss["achieved"],
                                 "peak": iss["peak"], "unit": "warp inst/s", "frac": iss["frac"],
                                 "warp_inst_per_launch": iss["warp_inst_per_launch"],
                                 "source": "smsp__inst_executed from profiles/ncu_flops.json (per launch) over "
                                           "this run's kernel time; peak 148 x 4 x 1.965 GHz"}
    return out


def framebuffer_writes(cfg, ms_frame, cfg_key=None):
    """The framebuffer's store traffic (north star: "framebuffer write
    GB/s"): 4 B per pixel (one 0xAARRGGBB word per thread, coalesced into the
    warp's 8x4 patch rows), over the frame's device time, against the
    measured HBM copy bandwidth — a few percent: the frame is written once,
    into L2 (ncu: DRAM writes of the kernels ~0.1 MB per C2 frame), and read
    back over PCIe."""
    bpf = 4 * cfg.width * cfg.height
    gbs = bpf / (ms_frame * 1e-3) / 1e9 if ms_frame > 0 else 0.0
    peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = json.load(f).get("hbm_gbs")
    except (OSError, ValueError):
        pass
    out = {"bytes_per_frame": bpf, "gbs": gbs, "store": "one 32-bit word per pixel, 32 B row segments per warp"}
    if peak:
        out.update({"hbm_peak_gbs": peak, "frac_of_hbm": gbs / peak})
    # ncu's dram__bytes_write.sum of the frame's kernels (profiles/ncu_flops.json;
    # ncu flushes caches between kernels, so this is the frame leaving L2)
    ctr = _load_profile("ncu_flops.json").get(cfg_key or "", {})
    dw = sum(v.get("dram_write_bytes", 0.0) for v in ctr.values() if isinstance(v, dict))
    if dw and ms_frame > 0:
        out.update({"ncu_dram_write_bytes_per_frame": dw, "ncu_dram_write_gbs": dw / (ms_frame * 1e-3) / 1e9,
                    "ncu_source": "profiles/ncu_flops.json (tools/ncu_counters.sh)"})
    return out


def ray_rates(wcc, work, fps):
    """Mrays/s two ways: reference-equivalent (the rays the reference's
    control flow traces for this frame) and executed (the
    closest-hit rays plus the shadow rays the culled pass actually sampled)."""
    c = wcc["counts"]
    out = {"mrays_per_s_reference_equivalent": wcc["rays"] * fps / 1e6}
    if work.get("hits"):
        out["mrays_per_s_executed"] = (c["CH_RAYS"] + work.get("shadow_rays", 0)) * fps / 1e6
    else:
        out["mrays_per_s_executed"] = out["mrays_per_s_reference_equivalent"]
    return out


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
