import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2504_18001_b200 as P
from paper_2504_18001_b200 import parallel
from paper_2504_18001_b200.harness import OrbitTrajectory
from paper_2504_18001_b200.macrocell import MacroCellGrid, layout
from paper_2504_18001_b200.session import SessionConfig
ctx = parallel.init_from_env()
dev = torch.device("cuda", 0)
model = bench.make_model(512)
fld = model.as_field()
vmin, vmax, _ = bench.load_macro(512)
grid, _, _ = layout((512,) * 3, 16)
mg = MacroCellGrid(16, (512,) * 3, grid, vmin, vmax, np.ones_like(vmin))
cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(32, 32, 32)),
                    scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20), settings=P.RenderSettings(), seed=0)
traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
sess = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
for f in range(10):
    sess.set_camera(traj.camera_at(f)); sess.render_frame()
for f in range(10, 40):
    torch.cuda.synchronize(); t0 = time.perf_counter(); sess.set_camera(traj.camera_at(f)); im, r = sess.render_frame()
    print(f"render_frame {1e3*(time.perf_counter()-t0):.2f} ms")
for f in range(40, 42):
    torch.cuda.synchronize()
    sess.set_camera(traj.camera_at(f))
    t0 = time.perf_counter()
    img = sess.render_frame_device()
    t1 = time.perf_counter()
    host = torch.empty(img.shape, dtype=torch.float32, pin_memory=True)
    t2 = time.perf_counter()
    with torch.cuda.stream(sess.stream):
        host.copy_(img, non_blocking=True)
    t3 = time.perf_counter()
    rec = sess.collect_record(t0)
    t4 = time.perf_counter()
    print(f"launch {1e3*(t1-t0):.2f} pin {1e3*(t2-t1):.2f} copyq {1e3*(t3-t2):.2f} sync+rec {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms")
