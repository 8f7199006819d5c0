"""INTEGRATION.md is executable: the ctypes stub a reference maintainer would
add (section 3) renders the reference's packed arguments through the C ABI,
and install() rebinds the reference package's importers (CPU test with a fake
package lives in test_host.py)."""

import os
import re

import numpy as np
import pytest

import golden_cases as G
import parity
from paper_2305_07450_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def stub_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 3."):]
    return re.search(r"```python\n(.*?)```", sec, re.S).group(1)


def test_stub_is_valid_python():
    compile(stub_source(), "INTEGRATION.md#3", "exec")


@pytest.mark.gpu
def test_stub_renders_the_golden_frame():
    src = stub_source().replace("/path/to/paper_2305_07450_b200/libb200rt.so", _native.LIB_PATH)
    ns = {}
    exec(compile(src, "INTEGRATION.md#3", "exec"), ns)
    c = G.frame_case("bench_128x72_s200_b3")
    ps = G.packed_scene(c)
    cam = c["camera"]
    import math

    vdist = 1.0 / math.tan(math.radians(cam["fov"]) / 2.0)
    pixels = np.zeros(c["width"] * c["height"], dtype=np.uint32)
    ns["_render_kernel_b200"](pixels, c["width"], c["height"], np.array(cam["position"]), cam["yaw"], cam["pitch"],
                              vdist, ps["kinds"], ps["positions"], ps["sizes"], ps["colors"], ps["refls"],
                              ps["light_pos"], ps["light_radius"], ps["light_color"], ps["ambient"], ps["max_refl"],
                              ps["sky"], ps["sky_w"], ps["sky_h"], ps["has_sky"], c["samples"], c["bounces"],
                              workers=2)
    parity.assert_byte_gate(pixels, G.frame_pixels(c["name"]), "INTEGRATION.md stub")
