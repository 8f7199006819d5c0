"""C5 stress scenes (256 and 512 spheres): device frame time of the culled path, a quick A/B probe."""
import sys, time
sys.path.insert(0, '.')
import paper_2305_07450_b200 as rt
cfg = rt.CONFIGS["C5"]
for count in (256, 512):
    s = rt.stress_scene(count=count)
    cam = cfg.camera()
    p = rt.RenderParams(500, 8, 384, 216)
    fb = rt.Framebuffer.create(384, 216)
    rt.render_frame(s, cam, p, fb)
    t = time.perf_counter()
    rt.render_frame(s, cam, p, fb)
    print(count, "spheres 384x216 s500 b8:", round((time.perf_counter() - t) * 1e3, 2), "ms", rt.last_kernel_ms(), flush=True)
