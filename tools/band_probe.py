"""Per-GPU frame time of sort-first bands (what one rank of an N-GPU run renders):
band (0, N) of the config-2 frame on one GPU, device-timed, L2 flushed."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2504_18001_b200 as P
from paper_2504_18001_b200 import parallel
from paper_2504_18001_b200.harness import OrbitTrajectory
from paper_2504_18001_b200.macrocell import MacroCellGrid, layout
from paper_2504_18001_b200.session import RenderSession, SessionConfig
fld = bench.make_model(512).as_field()
vmin, vmax, _ = bench.load_macro(512)
grid, _, _ = layout((512,) * 3, 16)
mg = MacroCellGrid(16, (512,) * 3, grid, vmin, vmax, np.ones_like(vmin))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for N in (1, 2, 4, 8):
    cfg = SessionConfig(cached=True, loader="inline", cache=P.CacheConfig(brick_size=16, pool_dims=(32, 32, 32)),
                        scheduler=P.SchedulerConfig(max_requests=40), policy=P.LodPolicy(1.2, 20), settings=P.RenderSettings(), seed=0)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
    s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg)
    s.set_band(0, N)
    for f in range(10):
        s.set_camera(traj.camera_at(f)); s.render_frame_device(); s.collect_record(time.perf_counter())
    ts = []
    for f in range(10, 30):
        flush.zero_(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream); s.set_camera(traj.camera_at(f)); s.render_frame_device(); e1.record(s.stream)
        s.collect_record(time.perf_counter()); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = sum(ts) / len(ts)
    print(f"N={N}: band frame {ms:.3f} ms -> whole-job {1000.0 / ms:.1f} fps (ideal {N * 1000.0 / ms if N == 1 else 0:.0f})")
    del s
