"""Golden frame-streaming bytes from the REFERENCE (service/protocol.py encode_frame,
render/image_io.py to_rgba8) for tests/test_streaming.py.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_stream.py
"""
from pathlib import Path

import numpy as np
from voxcache.render.image_io import to_rgba8
from voxcache.service.protocol import FORMAT_RGBA8, encode_frame

out = Path(__file__).resolve().parent
r = np.random.default_rng(9)
img = r.uniform(-0.2, 1.2, size=(7, 5, 4)).astype(np.float32)
img[0, 0] = [0.0, 1.0, 0.5, 0.49803922]       # x*255+0.5 on exact halves
img[0, 1] = [1.0 / 255.0, 254.5 / 255.0, 0.5 / 255.0, 2.0]
rgba = to_rgba8(img)
msg = encode_frame(42, 5, 7, FORMAT_RGBA8, rgba.tobytes())
np.savez(out / "stream_frame.npz", image=img, rgba=rgba, message=np.frombuffer(msg, dtype=np.uint8))
print("wrote", out / "stream_frame.npz", len(msg))
