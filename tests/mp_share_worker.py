"""torchrun worker for tests/test_gpu_share.py: each rank renders its sort-first band
of an orbit twice — decoding its brick batches alone, and sharing the decodes with
the other ranks (parallel.BrickShare) — and records per frame the FrameRecord, the
cache state and the image of both runs, plus the bricks it decoded when sharing."""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main(out_dir, spec_name, frames):
    import paper_2504_18001_b200 as P
    from gpu_runner import product_config, product_field, product_tf
    from paper_2504_18001_b200 import parallel
    from paper_2504_18001_b200.harness import OrbitTrajectory
    from scene_specs import SESSION_SPECS

    ctx = parallel.init_from_env()
    torch.cuda.set_device(ctx.local_rank)
    spec = SESSION_SPECS[spec_name]
    fld = product_field(spec)
    W, H = spec["res"]
    traj = OrbitTrajectory((0.5, 0.5, 0.5), spec.get("radius", 2.2), 120, width=W, height=H)
    out = {}
    for shared in (False, True):
        sess = parallel.make_session(ctx, fld, product_tf(spec["tf"]), traj.camera_at(0), product_config(spec),
                                     bands=True)
        if shared:
            sess.share_decode(ctx)
        own = 0
        for f in range(frames):
            sess.set_camera(traj.camera_at(f * spec.get("cam_step", 1)))
            img, rec = sess.render_frame()
            st = sess.debug_state()
            tag = f"{'s' if shared else 'a'}{f}"
            out[tag + "_img"] = img
            out[tag + "_rec"] = np.array([rec.samples, rec.true_misses, rec.fallback_hits, rec.exact_hits,
                                          rec.bricks_loaded, rec.bricks_loaded_total, rec.requests_inflight])
            for k in ("tables", "owner", "last_used", "entries", "batch"):
                out[f"{tag}_{k}"] = st[k]
            if shared:
                own += int(sess._share.counts[0].item())
        if shared:
            out["owned_total"] = np.array(own)
    out["world"] = np.array(ctx.world)
    np.savez(Path(out_dir) / f"rank{ctx.rank}.npz", **out)
    parallel.shutdown(ctx)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]))
