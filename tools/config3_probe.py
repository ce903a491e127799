"""Config 3 (4096^3 virtual INR, 1024^2) frames for profiling: python tools/config3_probe.py [frames] [march]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402


def main(frames=40, march="throughput", impl=None):
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    dims = (4096,) * 3
    fld = bench.make_model(4096).as_field()
    mg = macrocell.build(fld, dims, 16)
    cfg = bench.session_config(P, SessionConfig, pool=64)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
    s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, march=march)
    if impl is not None:
        s.impl = impl
    for f in range(frames):
        s.set_camera(traj.camera_at(f))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rec = s.render_frame()
        if f >= frames - 5:
            print(f, round((time.perf_counter() - t0) * 1e3, 2), "ms", rec.samples, rec.true_misses, s.last_frame_stats.get("iterations"))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 40, sys.argv[2] if len(sys.argv) > 2 else "throughput",
         int(sys.argv[3]) if len(sys.argv) > 3 else None)
