"""A few synchronous render_frame calls with the compressed transfer on and
one band, for ncu captures of the encode kernel:

    ncu --metrics gpu__time_duration.sum -k regex:encode_rows -s 2 -c 2 python tools/codec_profile.py C2
"""
import sys
sys.path.insert(0, "/root/repo")
import paper_2305_07450_b200 as rt
from paper_2305_07450_b200 import _native
key = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = rt.CONFIGS[key]
_native.set_options(bands=1)
scene, cam, params = c.scene(), c.camera(), c.params()
fb = rt.Framebuffer.create(c.width, c.height)
for _ in range(5):
    rt.render_frame(scene, cam, params, fb)
