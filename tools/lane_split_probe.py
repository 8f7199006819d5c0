"""Queue split of the culled FP32 path: hits sampled by the lane sampler (B1)
vs the warp sampler (B2), per configuration (option count_work)."""
import sys; sys.path.insert(0,'.')
import paper_2305_07450_b200 as rt
from paper_2305_07450_b200 import _native
for key in ["C2","C3","C4"]:
    cfg=rt.CONFIGS[key]; s,c,p=cfg.scene(),cfg.camera(),cfg.params()
    fb=rt.Framebuffer.create(cfg.width,cfg.height)
    _native.set_options(count_work=1)
    ctx=_native.context(1)
    rt.render_frame(s,c,p,fb); ctx.work_counts(reset=True)
    rt.render_frame(s,c,p,fb); w=ctx.work_counts(reset=True)
    _native.set_options(count_work=0)
    print(key, {k:w[k] for k in ("hits","sampled_hits","lane_hits","conic_hits","shadow_rays","sphere_tests")})
