"""End-to-end frame (render_frame(): pixels written into mapped pinned host memory)
against the device-resident frame: wall time, frame-kernel time (session events) and
the rest, medians over 50 steady config-2 frames."""
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402


def main(preroll=60, n=50):
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    fld = bench.make_model(512).as_field()
    mg = macrocell.build(fld, (512,) * 3, 16)
    cfg = bench.session_config(P, SessionConfig)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
    s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, march="throughput")
    s.reserve_host_frames(2)
    for f in range(preroll):
        s.set_camera(traj.camera_at(f))
        s.render_frame()
    s.timing = True
    med = statistics.median
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if "--flush" in sys.argv else None
    for mode in ("device", "host", "device", "host"):
        wall, mar = [], []
        for f in range(preroll, preroll + n):
            c = traj.camera_at(f)
            if flush is not None:
                flush.zero_()
            torch.cuda.synchronize()
            h0 = time.perf_counter()
            s.set_camera(c)
            if mode == "host":
                img, rec = s.render_frame()
                del img
            else:
                s.render_frame_device()
                s.collect_record(h0)
            wall.append((time.perf_counter() - h0) * 1e6)
            mar.append(s._ev_t0.elapsed_time(s._ev_t1) * 1e3)
        print(f"{'flush ' if flush is not None else ''}{mode:6s}: wall {med(wall):.1f} us, frame kernels {med(mar):.1f} us, rest {med(wall) - med(mar):.1f} us")


if __name__ == "__main__":
    main()
