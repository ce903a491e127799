"""Per-iteration trace of a no-cache frame (every sample through the in-kernel INR)."""
import json, sys, time
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
cfg = SessionConfig(cached=False, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(32, 32, 32)),
                    scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20), settings=P.RenderSettings(), seed=0)
traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
sess = parallel.make_session(ctx, fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
for f in range(3):
    sess.set_camera(traj.camera_at(10 + f)); sess.render_frame_device(); sess.collect_record(time.perf_counter())
sess.timing = True
sess.trace = True
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(sess.stream)
sess.set_camera(traj.camera_at(13)); sess.render_frame_device()
e1.record(sess.stream)
rec = sess.collect_record(time.perf_counter())
torch.cuda.synchronize()
print("frame ms", e0.elapsed_time(e1), "samples", rec.samples, "misses", rec.true_misses, "iters", sess.last_frame_stats.get("iterations"))
json.dump(sess.frame_trace(), open("gpurun_out/trace_uncached.json", "w"))
