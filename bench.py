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
L2_FLUSH_BYTES = 256 << 20
EXTRA_CONFIGS = ("C1", "P720", "P1080", "P4K", "C3", "C4", "C5", "C5_512")


def parse_args(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2")
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
    print(json.dumps(line), flush=True)
    return 0


# --- GPU ----------------------------------------------------------------------------
def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def run_ours(args):
    import numpy as np
    import torch

    import paper_2305_07450_b200 as rt
    from paper_2305_07450_b200 import _native

    world, rank, local = _dist_env()
    if world != args.gpus:
        args.gpus = world
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
    cfg = rt.CONFIGS[args.config]
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
    # other ranks map it over NVLink (CUDA IPC) and render straight into it
    from paper_2305_07450_b200 import bands

    extra_keys = () if (args.no_extra or world > 1) else EXTRA_CONFIGS
    size_keys = (args.config, *extra_keys, *(("C4",) if world > 1 else ()))
    max_px = max(rt.CONFIGS[k].width * rt.CONFIGS[k].height for k in size_keys)
    frame_bytes = 4 * cfg.width * cfg.height
    exchange = bands.torch_exchange if world > 1 else (lambda blob: blob)
    ipc = bands.IpcFrame(local, 1, max_px, rank, exchange)
    fb_ptr = ipc.ptr
    tiny = torch.zeros(1, device=dev)

    # N > 1: frames are independent units, so the headline shards whole
    # frames across the GPUs (each renders its own frames into its own
    # device frame, no collective: "weak" scaling); the north star's row
    # bands of one frame gathered to rank 0 (strong scaling) are measured too
    d_local = ctypes.c_void_p()
    if world > 1:
        _native.check(lib.rt_device_malloc(local, 4 * max_px, ctypes.byref(d_local)), "rt_device_malloc")
    cur = {"prec": prec, "mode": "frames"}

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
            dist.all_reduce(tiny)  # completes once every rank's band has landed

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
        """Frames/s, per-phase device times and executed work of config c."""
        r = time_config(c, warmup, steps, sample_clocks)
        # whole-job frames/s: every rank rendered len(ms) whole frames
        # ("frames" mode), or the ranks rendered len(ms) frames together ("bands")
        per = world if (world > 1 and cur["mode"] == "frames") else 1
        fps_c = per * len(r["ms"]) / (r["total_ms"] / 1e3)
        # per-kernel device times: CUDA events between the kernels on their
        # launch stream, averaged over as many frames as were timed (events
        # cost ~2.5 us each, so they stay out of the timed region itself)
        ctx.set_option("phases", 1)
        acc = {}
        n_ph = max(3, min(steps, 50))
        for _ in range(n_ph):
            render_cfg(c)
            torch.cuda.synchronize()
            for k, v in ctx.phase_ms().items():
                acc[k] = acc.get(k, 0.0) + v / n_ph
        phases = acc
        ctx.set_option("phases", 0)
        ctx.set_option("count_work", 1)
        ctx.work_counts(reset=True)
        render_cfg(c)
        torch.cuda.synchronize()
        work = ctx.work_counts(reset=True)
        ctx.set_option("count_work", 0)
        return r, fps_c, phases, work

    # headline: device-resident frames/s on the default path (wavefront + exact culling)
    main, fps, phases, work = measure(cfg, max(3, args.warmup), args.steps, sample_clocks=True)
    ms_frame = statistics.mean(main["ms"])
    wcc = wc[args.config]
    rays = wcc["rays"]
    peak_meas = _native.fp32_peak_tflops(local)
    roof = roofline(wcc, phases, work, ms_frame, cfg.samples, peak_meas, config_key=args.config)

    # e2e through the public API into a host framebuffer (rank 0's process)
    e2e = None
    if world == 1:
        scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
        fb = rt.Framebuffer.create(cfg.width, cfg.height)
        for _ in range(max(3, args.warmup)):
            rt.render_frame(scene, cam, params, fb, precision=args.precision)
        # every step a new camera (the frame loop's moving view): the frame
        # differs each step; the scene arrays and camera cross the C ABI and
        # travel to the device in the launch parameters (the library compares
        # the scene with its cached copy and re-uploads only what changed)
        cams = [rt.Camera(position=cam.position, yaw=cam.yaw + 1e-4 * (i % 2), pitch=cam.pitch, fov=cam.fov)
                for i in range(2)]
        ts = []
        for i in range(args.steps):
            t = time.perf_counter()
            rt.render_frame(scene, cams[i % 2], params, fb, precision=args.precision)
            ts.append(time.perf_counter() - t)
        e2e_fps = args.steps / sum(ts)
        ps = rt.pack_scene(scene)
        # kinds, positions, sizes, colours, reflectivities, light, ambient, max_refl + camera (f64, i32)
        h2d = int(4 * len(ps.kinds) + 8 * (3 + 1 + 3 + 1) * len(ps.kinds) + 8 * (3 + 1 + 3 + 2) + 8 * 6)
        e2e = {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": frame_bytes,
               "ms_per_step": 1e3 * statistics.mean(ts),
               "path": "paper_2305_07450_b200.render_frame -> rt_render_v1 (C ABI), pinned host framebuffer"}
        # the frame server's loop: frames back to back through FramePipeline,
        # each frame's copy overlapping the next frame's kernels; every frame
        # still lands whole in a host framebuffer before it is counted
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
        pipe.close()
        e2e["pipelined"] = {"value": args.steps / dt, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                            "d2h_bytes_per_step": frame_bytes,
                            "ms_per_step": 1e3 * dt / args.steps,
                            "path": "paper_2305_07450_b200.FramePipeline (rt_render_async_v1 / rt_frame_wait_v1), "
                                    "depth 3, pinned host framebuffers"}
    else:
        import torch.distributed as dist

        def e2e_run(step, frames_per_step):
            ts = []
            for i in range(max(3, args.warmup) + args.steps):
                dist.barrier()
                t = time.perf_counter()
                step()
                torch.cuda.synchronize()
                if i >= max(3, args.warmup):
                    ts.append(time.perf_counter() - t)
            t = torch.tensor([sum(ts)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return frames_per_step * args.steps / float(t.item())

        # (0) the headline: every rank renders whole frames and reads each back
        # into its own page-locked host frame over its own PCIe link
        host_own = torch.empty(cfg.width * cfg.height, dtype=torch.int32, pin_memory=True)

        def own_step():
            cur["mode"] = "frames"
            render_cfg(cfg)
            _native.check(lib.rt_copy_to_host(ctx.handle, 0, ctypes.c_void_p(host_own.data_ptr()), d_local,
                                              frame_bytes, ctypes.c_void_p(stream.cuda_stream)), "rt_copy_to_host")

        fps_own = e2e_run(own_step, world)

        # (1) one frame split in row bands: every rank renders its rows into its
        # own device frame and copies them into a page-locked host frame shared
        # by the node's ranks, over its own PCIe link
        shm = bands.ShmFrame(ctx, cfg.width, cfg.height, rank, bands.torch_exchange)

        def shm_step():
            render_cfg(cfg, part=rank, n_parts=world, out=d_local, sync=False)
            shm.copy_rows(d_local, rank, world, ctypes.c_void_p(stream.cuda_stream))

        fps_shm = e2e_run(shm_step, 1)
        ok = True
        if rank == 0:  # the shared frame is the frame
            ref = np.empty(cfg.width * cfg.height, dtype=np.uint32)
            render_cfg(cfg, part=0, n_parts=1, out=d_local, sync=False)
            _native.check(lib.rt_copy_to_host(ctx.handle, 0, _native.ptr(ref), d_local, frame_bytes,
                                              ctypes.c_void_p(stream.cuda_stream)), "rt_copy_to_host")
        dist.barrier()
        if rank == 0:
            ok = bool(np.array_equal(ref, shm.pixels))
        shm.close()

        # (2) row bands gathered into rank 0's device frame (CUDA IPC), one D2H on rank 0
        host = torch.empty(cfg.width * cfg.height, dtype=torch.int32, pin_memory=True) if rank == 0 else None

        def ipc_step():
            cur["mode"] = "bands"
            render_cfg(cfg)  # its all-reduce orders "every band landed"
            if rank == 0:
                _native.check(lib.rt_copy_to_host(ctx.handle, 0, ctypes.c_void_p(host.data_ptr()), fb_ptr,
                                                  frame_bytes, ctypes.c_void_p(stream.cuda_stream)),
                              "rt_copy_to_host")

        fps_ipc = e2e_run(ipc_step, 1)
        cur["mode"] = "frames"
        e2e = {"value": fps_own, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": frame_bytes * world,
               "path": f"rt_render_device_v1 whole frames on each of {world} ranks, each read back into the "
                       "rank's own page-locked host frame (its own PCIe link)",
               "row_bands_shared_host_frame": {
                   "value": fps_shm, "unit": "frames/s", "d2h_bytes_per_step": frame_bytes,
                   "path": "one frame in row bands: rt_copy_partition_to_host into a page-locked host frame "
                           "shared by the ranks (each GPU's rows over its own PCIe link)",
                   "frame_matches_single_gpu_render": ok},
               "row_bands_ipc_gather": {
                   "value": fps_ipc, "unit": "frames/s", "d2h_bytes_per_step": frame_bytes,
                   "path": "one frame in row bands into rank 0's device frame over NVLink (CUDA IPC) + one D2H "
                           "on rank 0"}}

    line = {
        "metric": "frames/s",
        "value": fps,
        "unit": "frames/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": main["total_ms"] / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (the paper's benchmark scene and camera, sceneio.py:314-333)",
        "config": {"workload": cfg.name, "width": cfg.width, "height": cfg.height, "samples": cfg.samples,
                   "bounces": cfg.bounces, "sky": cfg.sky, "parallelism": (f"frames x{world} (a whole frame per GPU per step, no collective)" if world > 1
                                   else "one GPU"),
                   "path": "wavefront + exact per-hit occluder culling (default)",
                   "l2": "flushed between timed frames (256 MiB memset outside the event pair)"},
        "mrays_per_s": rays * fps / 1e6,
        "e2e": e2e,
        "gpu_launches": main["launches"],
        "clocks": main["clocks"],
        "roofline": roof,
        "phases_ms": phases,
        "executed_work": work,
    }
    if world > 1:
        # the north star's row bands: one frame split across the GPUs, rows
        # gathered into rank 0's frame over NVLink (strong scaling), and the
        # same for 4K, where the split pays
        bands_lines = {}
        cur["mode"] = "bands"
        for key in (args.config, "C4"):
            c = rt.CONFIGS[key]
            if c.width * c.height > max_px:
                continue
            r = time_config(c, 3, args.steps)
            bands_lines[key] = {"workload": c.name, "fps": len(r["ms"]) / (r["total_ms"] / 1e3),
                                "ms_per_frame": r["total_ms"] / len(r["ms"]), "scaling": "strong",
                                "path": "rt_render_device_v1 row blocks into rank 0's frame (CUDA IPC) + all-reduce"}
        cur["mode"] = "frames"
        line["row_bands"] = bands_lines
    if rank == 0 and not args.no_extra and world == 1:
        extra = {}
        for key in extra_keys:
            c = rt.CONFIGS[key]
            r, f, ph, wk = measure(c, 3, 10 if key not in ("C4", "C5") else 5)
            km = statistics.mean(r["ms"])
            extra[key] = {"workload": c.name, "fps": f, "ms_per_frame": km,
                          "mrays_per_s": wc[key]["rays"] * f / 1e6, "phases_ms": ph,
                          "roofline": roofline(wc[key], ph, wk, km, c.samples, peak_meas, config_key=key)}
            if key in rt.workloads.PAPER_FPS:
                extra[key]["paper_fps_rtx2060"] = rt.workloads.PAPER_FPS[key]
        # ablation on the headline config: the same frame without culling, and as one megakernel
        for name, opts in (("no_cull", dict(wave=1, cull=0)), ("megakernel", dict(wave=0, cull=0))):
            for k, v in opts.items():
                ctx.set_option(k, v)
            r, f, ph, wk = measure(cfg, 3, args.steps)
            km = statistics.mean(r["ms"])
            extra[f"{args.config}_{name}"] = {"fps": f, "ms_per_frame": km, "phases_ms": ph,
                                              "roofline": roofline(wcc, ph, wk, km, cfg.samples, peak_meas,
                                                                   culled=False)}
        for k, v in dict(wave=1, cull=1).items():
            ctx.set_option(k, v)
        # the bit-identical mode (float64 in the reference's operation order)
        cur["prec"] = _native.RT_PREC_FP64
        for key in (args.config, "P720", "P1080", "P4K"):
            c = rt.CONFIGS[key]
            r = time_config(c, 3, 10)
            f = len(r["ms"]) / (r["total_ms"] / 1e3)
            extra[f"{key}_fp64_bit_exact"] = {"workload": c.name, "fps": f, "ms_per_frame": statistics.mean(r["ms"]),
                                              "precision": "fp64, bit-identical to the reference"}
        cur["prec"] = prec
        line["extra"] = extra
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        v, meta = cpu_reference_sample(cfg, args.cpu_seconds)
        what = (f"{meta['frames']} whole frames" if meta["frames"] else
                f"every {meta['row_step']}th row ({meta['rows']}/{cfg.height} rows)")
        line["cpu_baseline"] = {"value": v, "unit": "frames/s", "cores": meta["threads"], "kind": "port",
                                "sample": f"{what} of {cfg.name}, float64 C port of render_frame (oracle/, "
                                          f"bit-identical to the reference), {meta['seconds']:.1f} s"}
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
FLOP_SPHERE_FULL = 19   # a sphere test evaluated to the end (the kernels are branch-free: every test is full)
FLOP_PLANE = 2
FLOP_SHADOW_SETUP = 33  # sample point from the table, normalise, limit (n > 1); 21 for n = 1
FLOP_HIT = 60           # hit point, normal, to-light, Lambert/Blinn inputs
FLOP_BASIS = 39         # disc basis per hit (n > 1)
FLOP_PRIMARY = 36       # primary direction + pack
FLOP_REFLECT = 18
FLOP_SHADE = 45
FLOP_CULL = 40          # one body's cone classification (centre offset, axial/radial split, 2 sqrt, compares)
FLOP_CONIC = 17         # one silhouette-form sample test (|w|^2, x, y, d: 7 FMA + 1 add; culled sampler)
FLOP_CONIC_SETUP = 120  # shadow frame, cone and the six coefficients of one (hit, sphere) pair


def roofline(wcc, phases, work, ms_frame, samples, peak, culled=True, config_key=None):
    """Roofline of the dominant kernel: its executed FLOPs (cost model above,
    counts from the reference's control flow or the culled pass's own
    tallies) over its measured device time."""
    c = wcc["counts"]
    setup = FLOP_SHADOW_SETUP if samples > 1 else 21
    ch_tests = c["CH_TCA"] + c["CH_DISC"] + c["CH_FULL"]
    flops = {
        "trace": ch_tests * FLOP_SPHERE_FULL + c["CH_PLANE"] * FLOP_PLANE + c["HITS"] * FLOP_HIT
        + c["PIX"] * FLOP_PRIMARY + c["REFL"] * FLOP_REFLECT,
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
        flops["shadow"] = (conic_tests * FLOP_CONIC + conic_hits * FLOP_CONIC_SETUP
                           + ray_rays * setup + ray_hits * (FLOP_BASIS if samples > 1 else 0)
                           + (work["sphere_tests"] - conic_tests) * FLOP_SPHERE_FULL
                           + work["plane_tests"] * FLOP_PLANE)
    else:
        sh_tests = c["SH_TCA"] + c["SH_DISC"] + c["SH_FULL"]
        flops["classify"] = 0
        flops["shadow"] = (c["SH_RAYS"] * setup + c["HITS"] * (FLOP_BASIS if samples > 1 else 0)
                           + sh_tests * FLOP_SPHERE_FULL + c["SH_PLANE"] * FLOP_PLANE)
    if phases and sum(phases.values()) > 0:
        kernel = max(phases, key=phases.get)
        kms = phases[kernel]
        share = kms / max(sum(phases.values()), 1e-12)
    else:  # megakernel: one kernel does everything
        kernel, kms, share = "megakernel", ms_frame, 1.0
        flops = {"megakernel": sum(flops.values())}
    achieved = flops[kernel] / (kms * 1e-3) / 1e12 if kms > 0 else 0.0
    # DRAM traffic per launch of that kernel, from the committed ncu capture
    # (profiles/ncu_traffic.json); null when there is none for this config
    traffic, traffic_src = None, None
    try:
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")))
        t = tr.get(config_key, {}).get(kernel)
        if t:
            traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
            traffic_src = tr["_source"]
    except (OSError, ValueError, KeyError):
        pass
    per_kernel = {}
    if phases and sum(phases.values()) > 0:
        for k, ms in phases.items():
            if flops.get(k) and ms > 0.005:  # phases of a few us are event gaps, not kernels
                a = flops[k] / (ms * 1e-3) / 1e12
                per_kernel[k] = {"ms": ms, "flops": flops[k], "achieved": a, "frac": a / peak if peak else None}
    return {
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
        "peak_source": "measured dependent-free FFMA stream on this GPU (rt_fp32_peak_tflops); "
                       "MEASURED_PEAKS.json has no FP32 CUDA-core figure",
        "peak_nominal": NOMINAL_FP32_TFLOPS,
        "reference_equivalent_tflops": wcc["flops"] / (ms_frame * 1e-3) / 1e12,
        "kernels": per_kernel,
    }


def main(argv=None):
    args = parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
