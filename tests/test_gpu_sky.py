"""The skybox is read by the reference on every frame (renderer.py:282-300):
an in-place edit of `Skybox.texels` between two frames must show in the
second frame.  The library hashes the caller's array in full on every frame
and compares the hash with that of the texels it uploaded (rt_host.cu:
sky_content_changed); the hash sees content and position, so swapped texels
are a change too."""

import math

import numpy as np
import pytest

import oracle
import parity
import paper_2305_07450_b200 as rt
from paper_2305_07450_b200 import FramePipeline

pytestmark = pytest.mark.gpu

W, H = 96, 54


def _texel_of(d, sw, sh):
    """renderer.py:60-74: the texel a unit direction samples."""
    u = 0.5 + math.atan2(d[0], d[2]) / (2 * math.pi)
    v = 0.5 - math.asin(max(-1.0, min(1.0, d[1]))) / math.pi
    tx = int(math.floor(u * sw)) % sw
    ty = min(max(int(math.floor(v * sh)), 0), sh - 1)
    return tx, ty


def _setup():
    cfg = rt.CONFIGS["C3"]
    scene, cam = cfg.scene(), cfg.camera()
    sky = scene.skybox
    # a sky pixel of the top row and the texel it samples, chosen so that its
    # float index is not on the round-1 sampled signature's stride (n / 4099)
    n = sky.texels.size
    stride = max(1, n // 4099)
    xs = np.arange(W, dtype=np.int32)
    dirs = oracle.primary_directions(xs, np.zeros(W, np.int32), W, H, cam.yaw, cam.pitch, cam.fov)
    for x, d in zip(xs, dirs):
        tx, ty = _texel_of(d, sky.width, sky.height)
        i = (ty * sky.width + tx) * 3
        if 0 < ty < sky.height - 1 and all((i + c) % stride for c in range(3)):
            return scene, cam, rt.RenderParams(8, 2, W, H), int(x), tx, ty
    raise AssertionError("no suitable sky pixel")


def _want(scene, cam, params):
    return oracle.render(vars(rt.pack_scene(scene)), cam.position, cam.yaw, cam.pitch, cam.fov, W, H,
                         params.shadow_samples, params.bounce_limit)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_in_place_texel_edit_is_rendered(precision):
    scene, cam, params, px, tx, ty = _setup()
    sky = scene.skybox
    fb = rt.Framebuffer.create(W, H)
    rt.render_frame(scene, cam, params, fb, precision=precision)
    before = fb.pixels.copy()
    sky.texels[ty, tx] = (0.91, 0.05, 0.61)  # one texel, in place (same array)
    want = _want(scene, cam, params)
    assert want[px] != before[px], "the edited texel is visible at the chosen pixel"
    rt.render_frame(scene, cam, params, fb, precision=precision)
    if precision == "fp64":
        np.testing.assert_array_equal(fb.pixels, want)
    else:
        parity.assert_byte_gate(fb.pixels, want, "sky edit")
        assert parity.byte_gate(fb.pixels[px:px + 1], want[px:px + 1])[1] <= 1
        assert fb.pixels[px] != before[px]
    # and back: the original texel returns
    sky.texels[ty, tx] = (tx / sky.width, ty / sky.height, 0.25)
    rt.render_frame(scene, cam, params, fb, precision=precision)
    np.testing.assert_array_equal(fb.pixels[px], before[px])


def test_in_place_texel_edit_pipelined():
    scene, cam, params, px, tx, ty = _setup()
    sky = scene.skybox
    pipe = FramePipeline(2)
    try:
        a, b = rt.Framebuffer.create(W, H), rt.Framebuffer.create(W, H)
        ta = pipe.submit(scene, cam, params, a)
        pipe.wait(ta)
        sky.texels[ty, tx] = (0.05, 0.95, 0.1)
        tb = pipe.submit(scene, cam, params, b)
        pipe.wait(tb)
    finally:
        pipe.close()
    want = _want(scene, cam, params)
    assert parity.byte_gate(b.pixels[px:px + 1], want[px:px + 1])[1] <= 1 and a.pixels[px] != b.pixels[px]
    parity.assert_byte_gate(b.pixels, want, "pipelined sky edit")


def test_swapped_texels_are_a_change():
    """Exchanging the sampled texel with another one (same multiset of
    values, new positions) must be seen: the hash is position-sensitive."""
    scene, cam, params, px, tx, ty = _setup()
    sky = scene.skybox
    fb = rt.Framebuffer.create(W, H)
    rt.render_frame(scene, cam, params, fb, precision="fp64")
    before = fb.pixels.copy()
    ox = (tx + sky.width // 2) % sky.width  # a texel no top-row pixel samples
    a, b = sky.texels[ty, tx].copy(), sky.texels[ty, ox].copy()
    assert not np.array_equal(a, b)
    sky.texels[ty, tx], sky.texels[ty, ox] = b, a
    want = _want(scene, cam, params)
    rt.render_frame(scene, cam, params, fb, precision="fp64")
    np.testing.assert_array_equal(fb.pixels, want)
    assert fb.pixels[px] != before[px]


def test_new_sky_array_after_the_old_one_is_freed():
    """The library keeps no copy of the texels: a frame after the caller
    replaced (and freed) its sky array renders the new one."""
    scene, cam, params, px, tx, ty = _setup()
    fb = rt.Framebuffer.create(W, H)
    rt.render_frame(scene, cam, params, fb, precision="fp64")
    old = scene.skybox
    t = old.texels.copy()
    t[ty, tx] = (0.2, 0.9, 0.3)
    scene.skybox = rt.Skybox(old.width, old.height, t)
    del old
    import gc

    gc.collect()
    rt.render_frame(scene, cam, params, fb, precision="fp64")
    np.testing.assert_array_equal(fb.pixels, _want(scene, cam, params))
