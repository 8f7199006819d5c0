"""Row bands across ranks (paper_2305_07450_b200/bands.py).

CPU: the interleaved 8-row partition covers every row exactly once, and the
collective gather (`gather_bands`) reassembles a frame from per-rank compact
rows with world_size 2 over gloo — each rank's rows rendered by the oracle.
GPU: two processes sharing one B200 render their bands through
`rt_render_device_v1` straight into rank 0's framebuffer mapped with CUDA
IPC (the one-process-per-GPU product path), byte-identical to one render.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_cases as G
from paper_2305_07450_b200 import bands


@pytest.mark.parametrize("height", [1, 7, 8, 9, 72, 720, 1080, 2160, 2161])
@pytest.mark.parametrize("n_parts", [1, 2, 3, 4, 8])
def test_band_rows_partition_the_frame(height, n_parts):
    rows = np.concatenate([bands.band_rows(height, p, n_parts) for p in range(n_parts)])
    assert sorted(rows.tolist()) == list(range(height))
    counts = bands.band_row_counts(height, n_parts)
    assert sum(counts) == height and max(counts) - min(counts) <= bands.BLOCK_ROWS


def test_band_rows_balance_on_the_benchmark_camera():
    # interleaved 8-row blocks keep per-GPU row counts even
    counts = bands.band_row_counts(2160, 8)
    assert max(counts) / (sum(counts) / 8) <= 1.03


def test_band_rows_rejects_bad_partitions():
    with pytest.raises(ValueError):
        bands.band_rows(10, 2, 2)
    with pytest.raises(ValueError):
        bands.band_rows(10, 0, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, out_path):
    import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = G.frame_case("sweep_160x90_s16_b5_sky")
    cam = c["camera"]
    full = oracle.render(G.packed_scene(c), cam["position"], cam["yaw"], cam["pitch"], cam["fov"], c["width"],
                         c["height"], c["samples"], c["bounces"], threads=1)
    frame = torch.from_numpy(full.view(np.int32).reshape(c["height"], c["width"]).copy())
    mine = bands.compact_rows(frame, rank, world)
    out = torch.zeros_like(frame) if rank == 0 else None
    got = bands.gather_bands(mine, out, c["height"], rank, world)
    if rank == 0:
        np.save(out_path, got.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_bands_world_size_2_gloo(tmp_path):
    out = str(tmp_path / "frame.npy")
    mp.spawn(_gloo_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out).view(np.uint32).reshape(-1)
    np.testing.assert_array_equal(got, G.frame_pixels("sweep_160x90_s16_b5_sky"))


def _ipc_worker(rank, world, port, out_path):
    import ctypes

    import paper_2305_07450_b200 as rt
    from paper_2305_07450_b200 import _native

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = rt.CONFIGS["C2"]
    lib = _native.load()
    ctx = _native.Context((0,))
    ps = rt.pack_scene(cfg.scene())
    P = _native.ptr
    _native.check(lib.rt_set_scene_v1(ctx.handle, ps.n_bodies, P(ps.kinds), P(ps.positions), P(ps.sizes),
                                      P(ps.colors), P(ps.refls), P(ps.light_pos), ps.light_radius, P(ps.light_color),
                                      ps.ambient, ps.max_refl, P(ps.sky), ps.sky_w, ps.sky_h, int(ps.has_sky)),
                  "rt_set_scene_v1")
    frame = bands.IpcFrame(0, cfg.width, cfg.height, rank, bands.torch_exchange)
    cam = cfg.camera()
    cp = np.array(cam.position, dtype=np.float64)
    _native.check(lib.rt_render_device_v1(ctx.handle, 0, frame.ptr, cfg.width, None, cfg.width, cfg.height, P(cp),
                                          cam.yaw, cam.pitch, rt.camera_viewport_distance(cam.fov), cfg.samples,
                                          cfg.bounces, rank, world, bands.BLOCK_ROWS, _native.RT_PREC_FP32, None),
                  "rt_render_device_v1")
    host = np.zeros(cfg.width * cfg.height, dtype=np.uint32)
    # rt_copy_to_host synchronises the slot's stream: this rank's band has landed
    _native.check(lib.rt_copy_to_host(ctx.handle, 0, P(host), frame.ptr, host.nbytes, None), "rt_copy_to_host")
    dist.barrier()  # every band written
    if rank == 0:
        _native.check(lib.rt_copy_to_host(ctx.handle, 0, P(host), frame.ptr, host.nbytes, None), "rt_copy_to_host")
        np.save(out_path, host)
    dist.barrier()
    frame.close()
    dist.destroy_process_group()
    del ctypes


@pytest.mark.gpu
def test_ipc_row_bands_two_processes_one_gpu(tmp_path):
    """Two ranks on one GPU (nothing waits on another kernel: the only sync is
    a host barrier) write their interleaved bands into rank 0's IPC-mapped
    framebuffer; the frame equals a single-process render byte for byte."""
    import paper_2305_07450_b200 as rt

    out = str(tmp_path / "frame.npy")
    mp.spawn(_ipc_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    cfg = rt.CONFIGS["C2"]
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(cfg.scene(), cfg.camera(), cfg.params(), fb)
    np.testing.assert_array_equal(np.load(out), fb.pixels)


def _shm_worker(rank, world, port, out_path):
    import paper_2305_07450_b200 as rt
    from paper_2305_07450_b200 import _native

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = rt.CONFIGS["C2"]
    lib = _native.load()
    ctx = _native.Context((0,))
    ps = rt.pack_scene(cfg.scene())
    P = _native.ptr
    _native.check(lib.rt_set_scene_v1(ctx.handle, ps.n_bodies, P(ps.kinds), P(ps.positions), P(ps.sizes),
                                      P(ps.colors), P(ps.refls), P(ps.light_pos), ps.light_radius, P(ps.light_color),
                                      ps.ambient, ps.max_refl, P(ps.sky), ps.sky_w, ps.sky_h, int(ps.has_sky)),
                  "rt_set_scene_v1")
    # each rank renders its rows into its own device frame and copies them into the shared host frame
    d_frame = ctypes.c_void_p()
    _native.check(lib.rt_device_malloc(0, 4 * cfg.width * cfg.height, ctypes.byref(d_frame)), "rt_device_malloc")
    shm = bands.ShmFrame(ctx, cfg.width, cfg.height, rank, bands.torch_exchange)
    cam = cfg.camera()
    cp = np.array(cam.position, dtype=np.float64)
    _native.check(lib.rt_render_device_v1(ctx.handle, 0, d_frame, cfg.width, None, cfg.width, cfg.height, P(cp),
                                          cam.yaw, cam.pitch, rt.camera_viewport_distance(cam.fov), cfg.samples,
                                          cfg.bounces, rank, world, bands.BLOCK_ROWS, _native.RT_PREC_FP32, None),
                  "rt_render_device_v1")
    shm.copy_rows(d_frame, rank, world)
    dist.barrier()  # every rank's rows are in the shared frame
    if rank == 0:
        np.save(out_path, shm.pixels.copy())
    dist.barrier()
    shm.close()
    lib.rt_device_free(d_frame)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_shm_host_frame_two_processes_one_gpu(tmp_path):
    """The host-frame gather: two ranks copy their interleaved rows into a
    page-locked shared host frame over their own PCIe links; the frame equals
    a single-process render byte for byte."""
    import paper_2305_07450_b200 as rt

    out = str(tmp_path / "frame.npy")
    mp.spawn(_shm_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    cfg = rt.CONFIGS["C2"]
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(cfg.scene(), cfg.camera(), cfg.params(), fb)
    np.testing.assert_array_equal(np.load(out), fb.pixels)
