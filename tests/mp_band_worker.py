"""torchrun worker for tests/test_gpu_multirank.py: each rank renders its sort-first
film-row band of a throughput-schedule frame with a private cache, FrameGather
assembles the RGBA8 frame on rank 0, which also renders the whole frame in one
session and writes both to the output file."""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main(out_path):
    import paper_2504_18001_b200 as P
    from gpu_runner import product_field, product_tf
    from paper_2504_18001_b200 import parallel
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from paper_2504_18001_b200.session import SessionConfig
    from scene_specs import SESSION_SPECS

    ctx = parallel.init_from_env()
    torch.cuda.set_device(ctx.local_rank)
    spec = SESSION_SPECS["pressure"]
    fld = product_field(spec)
    W, H = 96, 80
    traj = OrbitTrajectory((0.5, 0.5, 0.5), 1.7, 120, width=W, height=H)

    def cfg():
        return SessionConfig(cached=True, loader="thread", cache=P.CacheConfig(brick_size=8, pool_dims=(12, 12, 12)),
                             scheduler=P.SchedulerConfig(max_requests=2000), policy=P.LodPolicy(1.5, 0, "corrected"),
                             seed=3)

    sess = parallel.make_session(ctx, fld, product_tf(spec["tf"]), traj.camera_at(0), cfg(), bands=True)
    sess.march = "throughput"
    gat = parallel.FrameGather(ctx, sess, H, W)
    for _ in range(14):
        img = sess.render_frame_device()
        gat.submit(img)
        rec = sess.collect_record(0.0)
    assert rec.true_misses == 0 and rec.fallback_hits == 0
    if ctx.rank == 0:
        frame = gat.host_frame()
        from paper_2504_18001_b200.session import RenderSession

        one = RenderSession(fld, product_tf(spec["tf"]), traj.camera_at(0), cfg(), march="throughput")
        for _ in range(14):
            img1, _ = one.render_frame()
        ref = np.clip(img1.astype(np.float64), 0.0, 1.0)
        ref8 = (ref * 255.0 + 0.5).astype(np.uint8)
        np.savez(out_path, frame=frame, ref=ref8, world=ctx.world, backend=ctx.backend)
    gat.close()
    parallel.shutdown(ctx)


if __name__ == "__main__":
    main(sys.argv[1])
