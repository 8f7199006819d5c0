"""render_frame end to end with and without torch imported and its CUDA context active in the same process (the bench imports torch)."""
import sys, time, statistics, os
sys.path.insert(0, '/root/repo')
if len(sys.argv) > 1 and sys.argv[1] == 'torch':
    import torch
    x = torch.zeros(1 << 20, device='cuda'); x += 1; torch.cuda.synchronize()
    if len(sys.argv) > 2:
        y = torch.randn(1000, 1000); z = y @ y  # CPU op: wakes torch's intra-op pool
import paper_2305_07450_b200 as rt
cfg = rt.CONFIGS["C3"]
scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
fb = rt.Framebuffer.create(cfg.width, cfg.height)
cams = [rt.Camera(position=cam.position, yaw=cam.yaw + 1e-4 * (i % 2), pitch=cam.pitch, fov=cam.fov) for i in range(2)]
for i in range(5): rt.render_frame(scene, cam, params, fb)
ts = []
for i in range(50):
    t = time.perf_counter(); rt.render_frame(scene, cams[i % 2], params, fb); ts.append(time.perf_counter() - t)
print(sys.argv[1:], "median %.1f us" % (1e6 * statistics.median(ts)))
