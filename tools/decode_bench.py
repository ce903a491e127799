"""Isolated INR decode throughput (the BASELINE metric's second half): 2^24 uniform
positions through the CUDA-core and the tcgen05 decoders, CUDA-event timed."""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def run(n=1 << 24, reps=5):
    import paper_2504_18001_b200 as P
    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200.device import device_field, ptr

    m = P.InrModel(P.HashGridConfig(), P.MLPConfig(), P.FieldDomain((512,) * 3), seed=0)
    r = np.random.default_rng(42)
    m.set_parameters([r.uniform(-0.7, 0.7, size=p.shape).astype(np.float32) for p in m.parameters()])
    df = device_field(m.as_field())
    pos = torch.rand((n, 3), dtype=torch.float64, device="cuda")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    out2 = torch.empty(n, dtype=torch.float32, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = {}
    for name, fn, o in (("cuda_core", "vcb_field_points", out), ("tcgen05", "vcb_inr_points_tc", out2)):
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(2):
            N.call(fn, C.byref(df.desc), n, ptr(pos), ptr(o), ptr(flag), s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            N.call(fn, C.byref(df.desc), n, ptr(pos), ptr(o), ptr(flag), s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name] = {"samples_per_s": n / (ms / 1e3), "ms": ms,
                     "mlp_tflops": n * 3136 / (ms / 1e3) / 1e12}
    res["max_abs_diff_tc_vs_cc"] = float((out - out2).abs().max().item())
    res["n"] = n
    return res


if __name__ == "__main__":
    print(json.dumps(run()))
