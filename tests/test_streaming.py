"""Frame streaming: CFRM messages byte-identical to the reference's encode_frame
(CPU), and the device RGBA8 quantisation equal to image_io.to_rgba8 (GPU)."""

import numpy as np
import pytest

from conftest import GOLDEN


def test_frame_message_bytes_match_reference():
    from paper_2504_18001_b200.streaming import FORMAT_RGBA8, encode_frame

    g = np.load(GOLDEN / "stream_frame.npz")
    msg = encode_frame(42, 5, 7, FORMAT_RGBA8, g["rgba"].tobytes())
    assert msg == g["message"].tobytes()


@pytest.mark.gpu
def test_device_rgba8_matches_reference_to_rgba8():
    import torch

    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200.device import ptr

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    g = np.load(GOLDEN / "stream_frame.npz")
    img = torch.from_numpy(g["image"]).cuda()
    out = torch.empty(img.shape, dtype=torch.uint8, device="cuda")
    N.call("vcb_frame_rgba8", ptr(img), img.numel() // 4, ptr(out), 0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), g["rgba"])
    # and on a large random frame against the restated rule
    x = np.random.default_rng(1).uniform(-0.5, 1.5, size=(256, 512, 4)).astype(np.float32)
    want = (np.clip(x.astype(np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    t = torch.from_numpy(x).cuda()
    o = torch.empty(x.shape, dtype=torch.uint8, device="cuda")
    N.call("vcb_frame_rgba8", ptr(t), t.numel() // 4, ptr(o), 0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(o.cpu().numpy(), want)
