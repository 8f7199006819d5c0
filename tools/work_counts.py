"""Count the reference algorithm's work per frame for every configuration
(roofline numerators), with the oracle's counting build.

    python tools/work_counts.py   ->  paper_2305_07450_b200/work_counts.json

Rays = closest-hit rays (primary + reflection) + shadow rays under the
reference's control flow.  FLOPs use SURVEY.md §8d's cost model: FMA = 2,
add/mul/sqrt/div = 1, compares free; sphere test 8 / 17 / 19 by exit
(tca < 0 / outside the disc / full), plane test 2, shadow-ray setup 33
(n > 1) or 21 (n = 1), per hit 60 (+39 disc basis when n > 1), per primary
ray 30 + 6 pack, per reflection 18, per shade 45.  C5 is counted on every
8th row and scaled (a full 4K frame takes ~19 CPU-minutes).
"""

import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2305_07450_b200 import CONFIGS, camera_viewport_distance, pack_scene  # noqa: E402

KEYS = ["PIX", "CH_RAYS", "SH_RAYS", "HITS", "REFL", "SHADE", "CH_TCA", "CH_DISC", "CH_FULL", "CH_PLANE", "SH_TCA",
        "SH_DISC", "SH_FULL", "SH_PLANE", "MISS"]


def flops(c, samples):
    return (8 * (c["CH_TCA"] + c["SH_TCA"]) + 17 * (c["CH_DISC"] + c["SH_DISC"]) + 19 * (c["CH_FULL"] + c["SH_FULL"])
            + 2 * (c["CH_PLANE"] + c["SH_PLANE"]) + (33 if samples > 1 else 21) * c["SH_RAYS"]
            + (60 + (39 if samples > 1 else 0)) * c["HITS"] + 36 * c["PIX"] + 18 * c["REFL"] + 45 * c["SHADE"])


def count(cfg, row_step=1):
    oracle.build()
    L = ctypes.CDLL(os.path.join(ROOT, "oracle", "librt_oracle_count.so"))
    scene, cam = cfg.scene(), cfg.camera()
    ps = pack_scene(scene)
    out = np.zeros(len(KEYS), dtype=np.int64)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    cp = np.array(cam.position, dtype=np.float64)
    d = ctypes.c_double
    L.rto_count_work(P(out), cfg.width, cfg.height, P(cp), d(cam.yaw), d(cam.pitch), d(camera_viewport_distance(cam.fov)),
                     ps.n_bodies, P(ps.kinds), P(ps.positions), P(ps.sizes), P(ps.colors), P(ps.refls),
                     P(ps.light_pos), d(ps.light_radius), P(ps.light_color), d(ps.ambient), d(ps.max_refl),
                     P(ps.sky), ps.sky_w, ps.sky_h, int(ps.has_sky), cfg.samples, cfg.bounces, 0, row_step, 0)
    c = {k: int(v) * row_step for k, v in zip(KEYS, out)}
    return c


def main():
    # python tools/work_counts.py [KEY ...]: recount only those configurations
    path = os.path.join(ROOT, "paper_2305_07450_b200", "work_counts.json")
    only = sys.argv[1:]
    res = {"model": __doc__.split("\n\n")[1].replace("\n", " "), "configs": {}}
    if only and os.path.exists(path):
        res["configs"] = json.load(open(path))["configs"]
    for key, cfg in CONFIGS.items():
        if only and key not in only:
            continue
        t = time.time()
        step = 8 if cfg.stress else 1
        c = count(cfg, step)
        entry = dict(name=cfg.name, counts=c, rays=c["CH_RAYS"] + c["SH_RAYS"], flops=flops(c, cfg.samples),
                     row_sample_step=step)
        res["configs"][key] = entry
        print(f"{key}: rays {entry['rays']:.4g} flops {entry['flops']:.4g} ({time.time() - t:.1f}s)", flush=True)
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
