import sys, time, gc
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2504_18001_b200 as P
from paper_2504_18001_b200 import parallel
from paper_2504_18001_b200.harness import OrbitTrajectory
from paper_2504_18001_b200.macrocell import MacroCellGrid, layout
from paper_2504_18001_b200.session import SessionConfig
ctx = parallel.init_from_env()
model = bench.make_model(512); fld = model.as_field()
vmin, vmax, _ = bench.load_macro(512)
grid, _, _ = layout((512,) * 3, 16)
mg = MacroCellGrid(16, (512,) * 3, grid, vmin, vmax, np.ones_like(vmin))
cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(32, 32, 32)),
                    scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20), settings=P.RenderSettings(), seed=0)
traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
sess = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for f in range(5):
    sess.set_camera(traj.camera_at(f)); sess.render_frame_device(); sess.collect_record(time.perf_counter())
out = []
for f in range(5, 25):
    flush.zero_(); torch.cuda.synchronize()
    sess.set_camera(traj.camera_at(f))
    t0 = time.perf_counter()
    img_h, rec = sess.render_frame()
    out.append(round((time.perf_counter() - t0) * 1e3, 2))
print("walls", out, "pool", len(sess._pin_free))
