"""The reference CLI on the B200 backend (paper_2305_07450_b200.cli, the
`--backend b200` switch for `raytracer render | bench`, cli.py:59-83).

`render` writes its PPM with the reference's own write_ppm
(sceneio.py:170-179); in fp64 the bytes must equal the oracle's frame in
that format, in fp32 the pixels must pass the byte gate.  `bench` must print
the reference harness's report for the B200 renderer.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import parity
import paper_2305_07450_b200 as rt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu


def _run(args, tmp_path):
    if not os.path.isdir(os.path.join(REF, "raytracer")):
        pytest.skip("baseline/_ref not installed (bash tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, REF, env.get("PYTHONPATH", "")])
    proc = subprocess.run([sys.executable, "-m", "paper_2305_07450_b200.cli", *args], cwd=tmp_path, env=env,
                          capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stdout[-2000:] + proc.stderr[-2000:]
    return proc.stdout


def _ppm(pixels, w, h):
    p = pixels.reshape(-1)
    rgb = np.stack([(p >> 16) & 255, (p >> 8) & 255, p & 255], -1).astype(np.uint8)
    return b"P6\n%d %d\n255\n" % (w, h) + rgb.tobytes()


def _oracle_frame(w, h, s, b):
    scene, cam = rt.build_benchmark_scene(), rt.benchmark_camera()
    return oracle.render(vars(rt.pack_scene(scene)), cam.position, cam.yaw, cam.pitch, cam.fov, w, h, s, b)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_cli_render_ppm(precision, tmp_path):
    w, h, s, b = 320, 180, 200, 3
    out = tmp_path / "frame.ppm"
    stdout = _run(["--backend", "b200", "--precision", precision, "render", "--width", str(w), "--height", str(h),
                   "--samples", str(s), "--bounces", str(b), "--workers", "3", "--out", str(out)], tmp_path)
    assert f"wrote {w}x{h} frame" in stdout
    got = out.read_bytes()
    want = _oracle_frame(w, h, s, b)
    if precision == "fp64":
        assert got == _ppm(want, w, h)
    else:
        hdr = len(b"P6\n%d %d\n255\n" % (w, h))
        rgb = np.frombuffer(got[hdr:], np.uint8).reshape(h, w, 3).astype(np.uint32)
        pix = (0xFF << 24) | (rgb[..., 0] << 16) | (rgb[..., 1] << 8) | rgb[..., 2]
        parity.assert_byte_gate(pix.astype(np.uint32), want.reshape(h, w))


def test_cli_bench_reports_b200_fps(tmp_path):
    stdout = _run(["bench", "--resolution", "720p", "--samples", "1", "--bounces", "1", "--warmup", "2",
                   "--frames", "20"], tmp_path)
    assert "fps" in stdout.lower() or "frames" in stdout.lower(), stdout
