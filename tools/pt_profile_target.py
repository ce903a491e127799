"""Small driver for ncu: a few path-traced 1024^2 frames (config 2) and training steps."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import bench  # noqa: E402
import paper_2504_18001_b200 as P  # noqa: E402
from paper_2504_18001_b200.harness import OrbitTrajectory  # noqa: E402
from paper_2504_18001_b200.macrocell import MacroCellGrid, layout  # noqa: E402
from paper_2504_18001_b200.session import RenderSession, SessionConfig  # noqa: E402

what = sys.argv[1]
if what == "pt":
    vol = 512
    fld = bench.make_model(vol).as_field()
    vmin, vmax, _ = bench.load_macro(vol)
    grid, _, _ = layout((vol,) * 3, 16)
    mg = MacroCellGrid(16, (vol,) * 3, grid, vmin, vmax, np.ones_like(vmin))
    cfg = SessionConfig(cached=True, mode="pathtrace", samples_per_pixel=1, loader="inline",
                        cache=P.CacheConfig(brick_size=16, pool_dims=(32, 32, 32)),
                        scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20), seed=0)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
    sess = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
    for f in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
        sess.set_camera(traj.camera_at(f))
        sess.render_frame()
else:
    from paper_2504_18001_b200.train import train
    from scene_specs import smoothed_random_lattice

    f = P.RawLatticeField(smoothed_random_lattice((64, 64, 64), 9), P.FieldDomain((64, 64, 64)))
    m = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((64, 64, 64)), seed=0)
    train(m, f, steps=int(sys.argv[2]) if len(sys.argv) > 2 else 4, seed=1)
