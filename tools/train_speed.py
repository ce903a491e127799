"""GPU INR training throughput at the reference's default batch (65536)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2504_18001_b200 as P  # noqa: E402
from paper_2504_18001_b200.train import psnr_on_lattice, train  # noqa: E402
from scene_specs import smoothed_random_lattice  # noqa: E402

dims = (64, 64, 64)
field = P.RawLatticeField(smoothed_random_lattice(dims, 9), P.FieldDomain(dims))
model = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain(dims), seed=0)
train(model, field, steps=5, seed=1)  # warm-up
for steps in (200, 1000):
    model = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain(dims), seed=0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    res = train(model, field, steps=steps, seed=2)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"{steps} steps x 65536: {e0.elapsed_time(e1) / steps:.3f} ms/step device, {wall / steps * 1e3:.3f} ms/step wall, "
          f"loss {res.loss_trace[0]:.5f} -> {res.final_loss:.5f}, psnr {psnr_on_lattice(res.model, field):.2f} dB")
