"""The compressed frame transfer (option "codec", frame_codec.h) on the GPU:
every frame it delivers equals the raw device-to-host copy bit for bit —
full-size configurations, ragged and tiny frames, every band count, FP64,
radiance alongside, the pipelined slots — and it moves fewer bytes."""

import numpy as np
import pytest

import paper_2305_07450_b200 as rt
from paper_2305_07450_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _restore_options():
    yield
    _native.set_options(codec=1, bands=0, codec_threads=0, codec_parts=0)


def _frame(scene, cam, params, precision=None, radiance=None, **opts):
    _native.set_options(**opts)
    fb = rt.Framebuffer.create(params.width, params.height)
    fb.pixels[:] = 0x5A5A5A5A  # a stale framebuffer: every pixel must be written
    rt.render_frame(scene, cam, params, fb, precision=precision, radiance=radiance)
    return fb.pixels.copy(), _native.context(1).last_d2h_bytes()


def _small(width, height, samples=16, bounces=2, sky=False):
    c = rt.CONFIGS["C3" if sky else "C2"]
    params = rt.RenderParams(width=width, height=height, shadow_samples=samples, bounce_limit=bounces)
    return c.scene(), c.camera(), params


@pytest.mark.parametrize("key", ["C1", "C2", "C3", "P720", "P1080"])
def test_codec_equals_raw_copy_full_size(key):
    c = rt.CONFIGS[key]
    scene, cam, params = c.scene(), c.camera(), c.params()
    raw, raw_bytes = _frame(scene, cam, params, codec=0)
    enc, enc_bytes = _frame(scene, cam, params, codec=1)
    np.testing.assert_array_equal(enc, raw)
    assert raw_bytes == 4 * c.width * c.height
    assert enc_bytes < raw_bytes / 2, (enc_bytes, raw_bytes)


@pytest.mark.parametrize("bands", [1, 2, 3, 6, 8])
def test_codec_every_band_count(bands):
    scene, cam, params = _small(333, 251, samples=32, bounces=3)
    raw, _ = _frame(scene, cam, params, codec=0, bands=bands)
    enc, _ = _frame(scene, cam, params, codec=1, bands=bands)
    np.testing.assert_array_equal(enc, raw)


@pytest.mark.parametrize("size", [(1, 1), (1, 9), (7, 3), (8, 8), (9, 17), (31, 5), (33, 40), (97, 61), (1000, 3)])
def test_codec_ragged_and_tiny_frames(size):
    w, h = size
    scene, cam, params = _small(w, h, samples=8, bounces=1, sky=True)
    raw, _ = _frame(scene, cam, params, codec=0)
    enc, _ = _frame(scene, cam, params, codec=1)
    np.testing.assert_array_equal(enc, raw)


def test_codec_fp64_and_radiance_alongside():
    scene, cam, params = _small(160, 90, samples=16, bounces=2, sky=True)
    raw_rad = np.zeros((160 * 90, 3), dtype=np.float64)
    enc_rad = np.zeros((160 * 90, 3), dtype=np.float64)
    raw, _ = _frame(scene, cam, params, precision="fp64", radiance=raw_rad, codec=0)
    enc, enc_bytes = _frame(scene, cam, params, precision="fp64", radiance=enc_rad, codec=1)
    np.testing.assert_array_equal(enc, raw)
    np.testing.assert_array_equal(enc_rad, raw_rad)
    assert enc_bytes >= raw_rad.nbytes  # the radiance still travels raw


@pytest.mark.parametrize("threads", [1, 2, 16])
def test_codec_thread_counts(threads):
    c = rt.CONFIGS["C2"]
    scene, cam, params = c.scene(), c.camera(), c.params()
    raw, _ = _frame(scene, cam, params, codec=0)
    enc, _ = _frame(scene, cam, params, codec=1, codec_threads=threads)
    np.testing.assert_array_equal(enc, raw)


def test_codec_pipelined_frames_equal_raw():
    c = rt.CONFIGS["C2"]
    scene, cam, params = c.scene(), c.camera(), c.params()
    cams = [rt.Camera(position=(0.3 * i, 1.4, -4.5), yaw=0.05 * i, pitch=-0.08, fov=60.0) for i in range(6)]
    want = []
    for cm in cams:
        raw, _ = _frame(scene, cm, params, codec=0)
        want.append(raw)
    _native.set_options(codec=1)
    pipe = rt.FramePipeline(depth=3)
    fbs = [rt.Framebuffer.create(c.width, c.height) for _ in cams]
    for cm, fb in zip(cams, fbs):
        pipe.submit(scene, cm, params, fb)  # (waits for the frame depth tickets back)
    pipe.drain()
    for fb, w in zip(fbs, want):
        np.testing.assert_array_equal(fb.pixels, w)


def test_codec_rgba_byte_order():
    """Option rgba (the frame server's R,G,B,A bytes): alpha is still the top
    byte, so rows travel packed; the frame equals the raw copy's."""
    scene, cam, params = _small(200, 120, samples=16, bounces=2, sky=True)
    try:
        raw, _ = _frame(scene, cam, params, codec=0, rgba=1)
        enc, enc_bytes = _frame(scene, cam, params, codec=1, rgba=1)
    finally:
        _native.set_options(rgba=0)
    np.testing.assert_array_equal(enc, raw)
    assert (enc >> 24 == 0xFF).all()
    assert enc_bytes < 200 * 120 * 4


def test_codec_pipeline_mixed_sizes_and_depth4():
    """Slots of different frame sizes in flight at once (each slot keeps its own
    mapped buffer and expands into its own framebuffer)."""
    c = rt.CONFIGS["C3"]
    scene = c.scene()
    sizes = [(320, 180), (97, 61), (640, 360), (1, 9), (333, 251), (160, 90)]
    cam = c.camera()
    want = []
    for w, h in sizes:
        p = rt.RenderParams(width=w, height=h, shadow_samples=16, bounce_limit=2)
        raw, _ = _frame(scene, cam, p, codec=0)
        want.append(raw)
    _native.set_options(codec=1)
    pipe = rt.FramePipeline(depth=4)
    fbs = []
    for w, h in sizes:
        p = rt.RenderParams(width=w, height=h, shadow_samples=16, bounce_limit=2)
        fb = rt.Framebuffer.create(w, h)
        fb.pixels[:] = 0x5A5A5A5A
        fbs.append(fb)
        pipe.submit(scene, cam, p, fb)
    pipe.drain()
    for fb, w in zip(fbs, want):
        np.testing.assert_array_equal(fb.pixels, w)


def test_codec_two_threads_two_contexts():
    """render_frame on the shared context and a FramePipeline (its own context)
    from two Python threads at once: each expansion team writes its own frame."""
    import threading

    c = rt.CONFIGS["C2"]
    scene, cam, params = c.scene(), c.camera(), c.params()
    want, _ = _frame(scene, cam, params, codec=0)
    _native.set_options(codec=1)
    errors = []

    def sync_loop():
        try:
            fb = rt.Framebuffer.create(c.width, c.height)
            for _ in range(20):
                fb.pixels[:] = 0
                rt.render_frame(scene, cam, params, fb)
                np.testing.assert_array_equal(fb.pixels, want)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    def pipe_loop():
        try:
            pipe = rt.FramePipeline(depth=2)
            fbs = [rt.Framebuffer.create(c.width, c.height) for _ in range(20)]
            for fb in fbs:
                pipe.submit(scene, cam, params, fb)
            pipe.drain()
            for fb in fbs:
                np.testing.assert_array_equal(fb.pixels, want)
            pipe.close()
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=sync_loop), threading.Thread(target=pipe_loop)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


def test_codec_reports_fewer_bytes_and_device_time():
    """rt_last_d2h_bytes: the compressed run's bytes; rt_last_kernel_ms still
    reports the frame's device time (read after the early return)."""
    c = rt.CONFIGS["C2"]
    scene, cam, params = c.scene(), c.camera(), c.params()
    _, enc_bytes = _frame(scene, cam, params, codec=1)
    ms = rt.last_kernel_ms()
    assert 0.01 < ms < 5.0
    assert 100_000 < enc_bytes < 1_000_000


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_codec_encode_parts(parts):
    """A one-band frame's encode cut into parts (option codec_parts), each
    expanded as it lands: the same frame."""
    c = rt.CONFIGS["C2"]
    scene, cam, params = c.scene(), c.camera(), c.params()
    raw, _ = _frame(scene, cam, params, codec=0)
    enc, _ = _frame(scene, cam, params, codec=1, bands=1, codec_parts=parts)
    np.testing.assert_array_equal(enc, raw)
    small = _small(97, 61, samples=8, bounces=1)
    raw, _ = _frame(*small, codec=0)
    enc, _ = _frame(*small, codec=1, bands=1, codec_parts=parts)
    np.testing.assert_array_equal(enc, raw)


@pytest.mark.parametrize("n_parts,size", [(1, (1280, 720)), (3, (1280, 720)), (2, (97, 61)), (5, (333, 19))])
def test_codec_partition_copies(n_parts, size):
    """rt_copy_partition_to_host (the multi-GPU host-frame gather) with the
    compressed transfer: each partition's interleaved 8-row blocks land in a
    host frame exactly as the raw 2-D copies put them."""
    import ctypes

    w, h = size
    lib = _native.load()
    ctx = _native.Context((0,))
    try:
        c = rt.CONFIGS["C2"]
        ps = rt.pack_scene(c.scene())
        P = _native.ptr
        _native.check(lib.rt_set_scene_v1(ctx.handle, ps.n_bodies, P(ps.kinds), P(ps.positions), P(ps.sizes),
                                          P(ps.colors), P(ps.refls), P(ps.light_pos), ps.light_radius,
                                          P(ps.light_color), ps.ambient, ps.max_refl, P(ps.sky), ps.sky_w, ps.sky_h,
                                          int(ps.has_sky)), "rt_set_scene_v1")
        d_frame = ctypes.c_void_p()
        _native.check(lib.rt_device_malloc(0, 4 * w * h, ctypes.byref(d_frame)), "rt_device_malloc")
        cam = c.camera()
        cp = np.array(cam.position, dtype=np.float64)
        _native.check(lib.rt_render_device_v1(ctx.handle, 0, d_frame, w, None, w, h, P(cp), cam.yaw, cam.pitch,
                                              rt.camera_viewport_distance(cam.fov), 16, 2, 0, 1, 8,
                                              _native.RT_PREC_FP32, None), "rt_render_device_v1")
        frames = []
        for codec in (0, 1):
            ctx.set_option("codec", codec)
            host = np.full(w * h, 0x5A5A5A5A, dtype=np.uint32)
            for part in range(n_parts):
                _native.check(lib.rt_copy_partition_to_host(ctx.handle, 0, P(host), d_frame, w, h, part, n_parts, 8,
                                                            None), "rt_copy_partition_to_host")
            frames.append(host)
        np.testing.assert_array_equal(frames[1], frames[0])
        assert (frames[0] != 0x5A5A5A5A).all()
        lib.rt_device_free(d_frame)
    finally:
        ctx.close()


def test_codec_partition_copy_from_an_offset_device_frame():
    """rt_copy_partition_to_host from a device frame that starts 4 bytes into
    its allocation (a caller's pointer need not be 16-byte aligned)."""
    import ctypes

    import torch

    w, h = 64, 24
    lib = _native.load()
    ctx = _native.Context((0,))
    try:
        frame = (np.arange(w * h, dtype=np.uint32) // 5) | np.uint32(0xFF000000)
        buf = torch.zeros(w * h + 4, dtype=torch.int32, device="cuda")
        buf[1:1 + w * h] = torch.from_numpy(frame.view(np.int32)).cuda()
        torch.cuda.synchronize()
        d_frame = ctypes.c_void_p(buf.data_ptr() + 4)
        for codec in (0, 1):
            ctx.set_option("codec", codec)
            host = np.zeros(w * h, dtype=np.uint32)
            for part in range(3):
                _native.check(lib.rt_copy_partition_to_host(ctx.handle, 0, _native.ptr(host), d_frame, w, h, part, 3,
                                                            8, None), "rt_copy_partition_to_host")
            np.testing.assert_array_equal(host, frame)
    finally:
        ctx.close()
