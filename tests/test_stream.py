"""The frame server's wire format (server.py:56-74): the host restatement
matches the reference's encode_frame bytes; the GPU renders the same message
directly (R,G,B,A packed by the kernels)."""

import pytest

import golden_cases as G
import paper_2305_07450_b200 as rt
from paper_2305_07450_b200 import stream


def _golden_fb():
    fb = rt.Framebuffer.create(128, 72)
    fb.pixels[:] = G.frame_pixels("bench_128x72_s200_b3")
    return fb


def test_encode_frame_matches_reference_bytes():
    want = G._frames()["encode/bench_128x72_s200_b3_id7"].tobytes()
    assert stream.encode_frame(7, _golden_fb()) == want


def test_decode_frame_header():
    msg = stream.encode_frame(0x1_0000_0005, _golden_fb())
    assert stream.decode_frame_header(msg) == (5, 128, 72, stream.FORMAT_RGBA8)
    with pytest.raises(ValueError):
        stream.decode_frame_header(b"\0" * 16)
    with pytest.raises(ValueError):
        stream.decode_frame_header(b"RAYF")


@pytest.mark.gpu
def test_frame_encoder_renders_the_wire_message():
    scene, cam = rt.build_benchmark_scene(), rt.benchmark_camera()
    enc = stream.FrameEncoder()
    try:
        msg = enc.render(scene, cam, rt.RenderParams(200, 3, 128, 72), 7, precision="fp64")
        assert bytes(msg) == G._frames()["encode/bench_128x72_s200_b3_id7"].tobytes()
        params = rt.RenderParams(200, 3, 1280, 720)
        fb = rt.Framebuffer.create(1280, 720)
        rt.render_frame(scene, cam, params, fb)
        for workers in (None, 3):
            msg = enc.render(scene, cam, params, 42, workers=workers)
            assert bytes(msg) == stream.encode_frame(42, fb)
    finally:
        enc.close()


@pytest.mark.gpu
def test_pipelined_frame_encoder_messages():
    """Several RAYF messages in flight: each equals the synchronous
    encoder's message for the same frame."""
    scene = rt.build_benchmark_scene()
    params = rt.RenderParams(32, 3, 320, 180)
    sync = stream.FrameEncoder()
    pipe = stream.PipelinedFrameEncoder(3)
    try:
        want, tickets = [], []
        for i in range(6):
            cam = rt.Camera(position=(0.1 * i, 1.4, -4.5), yaw=0.02 * i, pitch=-0.08, fov=60.0)
            want.append(bytes(sync.render(scene, cam, params, 100 + i)))
            tickets.append(pipe.submit(scene, cam, params, 100 + i))
            if i >= 2:  # consume with a lag of two frames, as a frame loop would
                assert bytes(pipe.wait(tickets[i - 2])) == want[i - 2]
        for i in (4, 5):
            assert bytes(pipe.wait(tickets[i])) == want[i]
    finally:
        pipe.close()
        sync.close()
