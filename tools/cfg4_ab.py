import sys
sys.path.insert(0, "tests")
import numpy as np
import paper_2504_18001_b200 as P
from paper_2504_18001_b200.harness import OrbitTrajectory
from paper_2504_18001_b200.session import RenderSession, SessionConfig


def run(ranked, seed, impl, frames=8):
    dims = (2048, 2048, 2048)
    fld = P.make_procedural("shells", dims)
    cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(24, 24, 24)),
                        scheduler=P.SchedulerConfig(max_requests=40, ranking_enabled=ranked),
                        policy=P.LodPolicy(1.2, 8), settings=P.RenderSettings(base_step_scale=4.0), seed=seed)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 1.8, 240, width=1920, height=1080)
    sess = RenderSession(fld, P.warm_body(0.35, 0.9), traj.camera_at(seed * 7), cfg)
    sess.impl = impl
    out = []
    for f in range(frames):
        sess.set_camera(traj.camera_at(seed * 7 + f))
        img, rec = sess.render_frame()
        out.append((rec.samples, rec.true_misses, rec.exact_hits, float(np.abs(img).sum())))
    return out


for impl in (0, 9):
    print(impl, run(True, 1, impl))
