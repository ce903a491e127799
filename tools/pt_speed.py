"""Path-trace frame time at the bench workload (config 2, 1024^2): device-timed."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2504_18001_b200 as P  # noqa: E402
from paper_2504_18001_b200.harness import OrbitTrajectory  # noqa: E402
from paper_2504_18001_b200.macrocell import MacroCellGrid, layout  # noqa: E402
from paper_2504_18001_b200.session import RenderSession, SessionConfig  # noqa: E402

res = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spp = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cached = (sys.argv[3] != "uncached") if len(sys.argv) > 3 else True
vol = 512
fld = bench.make_model(vol).as_field()
vmin, vmax, _ = bench.load_macro(vol)
grid, _, _ = layout((vol,) * 3, 16)
mg = MacroCellGrid(16, (vol,) * 3, grid, vmin, vmax, np.ones_like(vmin))
cfg = SessionConfig(cached=cached, mode="pathtrace", samples_per_pixel=spp, loader="inline",
                    cache=P.CacheConfig(brick_size=16, pool_dims=(32, 32, 32)),
                    scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20),
                    settings=P.RenderSettings(), seed=0)
traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=res, height=res)
sess = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
sess.impl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
for f in range(40):
    sess.set_camera(traj.camera_at(f))
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sess.stream)
    sess.render_frame_device()
    e1.record(sess.stream)
    rec = sess.collect_record(t0)
    torch.cuda.synchronize()
    if f % 5 == 4 or f < 3:
        print(f"frame {f}: {e0.elapsed_time(e1):.2f} ms samples {rec.samples} miss {rec.true_misses} "
              f"fb {rec.fallback_hits} iters {sess.last_frame_stats['iterations']} rays {sess.last_frame_stats['rays']}",
              flush=True)
