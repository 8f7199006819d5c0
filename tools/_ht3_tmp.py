import os, sys, time, statistics
os.environ["B200RT_HOST_TIMING"] = "1"
sys.path.insert(0, "/root/repo")
import paper_2305_07450_b200 as rt
key = sys.argv[1]
cfg = rt.CONFIGS[key]
scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
fb = rt.Framebuffer.create(cfg.width, cfg.height)
for _ in range(50):
    rt.render_frame(scene, cam, params, fb)
print("---", file=sys.stderr, flush=True)
ts = []
for _ in range(6):
    t = time.perf_counter(); rt.render_frame(scene, cam, params, fb); ts.append(time.perf_counter() - t)
print("python-side", [round(1e6 * x, 1) for x in ts], file=sys.stderr, flush=True)
