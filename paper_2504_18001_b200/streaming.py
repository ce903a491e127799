"""Frame streaming to the reference's viewer protocol (service/protocol.py:40-61):
a CFRM frame message around an RGBA8 frame quantised on the GPU
(RenderSession.render_frame_rgba8, image_io.py:14-21)."""

from __future__ import annotations

import struct

FRAME_MAGIC = b"CFRM"
FORMAT_RGBA8 = 0
FORMAT_PNG = 1
KIND_FRAME = 3  # protocol.py:36

_LEN = struct.Struct("<I")
_FRAME = struct.Struct("<4sIHHB")


def encode_message(kind: int, payload: bytes) -> bytes:
    """protocol.py:47-49: u32 length of (kind byte + payload), kind, payload."""
    return _LEN.pack(len(payload) + 1) + bytes([kind]) + payload


def encode_frame(frame_id: int, width: int, height: int, fmt: int, pixels: bytes) -> bytes:
    """protocol.py:56-58."""
    return encode_message(KIND_FRAME, _FRAME.pack(FRAME_MAGIC, frame_id, width, height, fmt) + bytes(pixels))


def frame_message(session) -> tuple[bytes, object]:
    """Render one frame and wrap it for the viewer: (CFRM message bytes, FrameRecord)."""
    rgba, rec = session.render_frame_rgba8()
    h, w = rgba.shape[:2]
    return encode_frame(rec.frame, w, h, FORMAT_RGBA8, rgba.tobytes()), rec
