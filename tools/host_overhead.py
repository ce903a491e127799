"""Host-side cost of one frame submission (config 2): _frame_params, the march call,
the maintenance call, and render_frame_device as a whole (no synchronisation)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402


def main():
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    fld = bench.make_model(512).as_field()
    mg = macrocell.build(fld, (512,) * 3, 16)
    cfg = bench.session_config(P, SessionConfig)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
    s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, march="throughput")
    for f in range(30):
        s.set_camera(traj.camera_at(f))
        s.render_frame()
    img = torch.empty((1024, 1024, 4), device="cuda")
    torch.cuda.synchronize()
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        s._frame_params(img)
    t_params = (time.perf_counter() - t0) / n
    ts = []
    for f in range(30, 30 + n):
        s.set_camera(traj.camera_at(f))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.render_frame_device()
        t1 = time.perf_counter()
        s.collect_record(t0)
        ts.append(t1 - t0)
    print(f"_frame_params {t_params * 1e6:.0f} us, render_frame_device (submit only) {sorted(ts)[n // 2] * 1e6:.0f} us")


if __name__ == "__main__":
    main()
