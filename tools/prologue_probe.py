"""Where a device-timed config-2 step goes: host prologue as the GPU sees it (step
event -> the event before the frame kernels), frame kernels, and maintenance + record
copies (after the frame kernels -> step end event).  Medians over 50 steady frames."""
import statistics
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402


def main(preroll=60, n=50, graph=False):
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import macrocell
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import RenderSession, SessionConfig

    fld = bench.make_model(512).as_field()
    mg = macrocell.build(fld, (512,) * 3, 16)
    cfg = bench.session_config(P, SessionConfig)
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 2.2, 120, width=1024, height=1024)
    s = RenderSession(fld, P.warm_body(0.5, 0.9), traj.camera_at(0), cfg, macro=mg, march="throughput")
    s.maint_graph = graph
    for f in range(preroll):
        s.set_camera(traj.camera_at(f))
        s.render_frame_device()
        s.collect_record(time.perf_counter())
    s.timing = True
    pro, mar, post, host = [], [], [], []
    for f in range(preroll, preroll + n):
        c = traj.camera_at(f)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s.stream)
        h0 = time.perf_counter()
        s.set_camera(c)
        s.render_frame_device()
        h1 = time.perf_counter()
        e1.record(s.stream)
        s.collect_record(h0)
        torch.cuda.synchronize()
        pro.append(e0.elapsed_time(s._ev_t0) * 1e3)
        mar.append(s._ev_t0.elapsed_time(s._ev_t1) * 1e3)
        post.append(s._ev_t1.elapsed_time(e1) * 1e3)
        host.append((h1 - h0) * 1e6)
    med = statistics.median
    print(f"maint_graph={graph}: prologue {med(pro):.1f} us, frame kernels {med(mar):.1f} us, after {med(post):.1f} us, "
          f"host submit {med(host):.1f} us")


if __name__ == "__main__":
    for g in (False, True, False, True):
        main(graph=g)
