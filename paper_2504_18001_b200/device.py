"""Device plumbing: torch tensors for memory/streams, ABI struct builders.

torch is used only to own device memory and streams; all compute goes through
libcinr_b200.so.  A CUDA device is required — there is no CPU path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError

PROC_IDS = {"sphere": 0, "shells": 1, "marschner_lobb_like": 2}


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise N.NativeUnavailable("a CUDA device (B200, sm_100a) is required; there is no CPU fallback")
    N.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ConfigError(f"device must be a CUDA device, got {dev}")
    return dev


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class DeviceField:
    """A field's parameters resident on one device + its VcbField descriptor."""

    def __init__(self, desc: N.VcbField, keep):
        self.desc = desc
        self._keep = keep  # tensors referenced by raw pointers in desc


def _inr_desc(model_like, device, clip):
    g = model_like.grid_config
    m = model_like.mlp_config
    if g.levels > N.MAX_LEVELS:
        raise ConfigError(f"at most {N.MAX_LEVELS} hash-grid levels on the GPU path")
    if g.levels * g.features_per_entry > 128 or m.hidden_width > 128 or m.hidden_layers + 1 > N.MAX_LAYERS:
        # the generic decoder keeps one activation row per thread (128 floats) and the
        # weights in shared memory (width 128: 74 KB)
        raise ConfigError("MLP wider than 128 / deeper than 7 hidden layers is not supported on the GPU path")
    tables = [np.asarray(t, dtype=np.float32) for t in model_like.tables]
    rows = [t.shape[0] for t in tables]
    tab = torch.from_numpy(np.ascontiguousarray(np.concatenate(tables, axis=0))).to(device)
    ws = [np.asarray(w, dtype=np.float32) for w in model_like.weights]
    bs = [np.asarray(b, dtype=np.float32) for b in model_like.biases]
    wt = torch.from_numpy(np.concatenate([w.ravel() for w in ws])).to(device)
    bt = torch.from_numpy(np.concatenate([b.ravel() for b in bs])).to(device)
    d = N.VcbField()
    d.kind = 0
    d.levels = g.levels
    d.feats = g.features_per_entry
    d.out_sigmoid = 1 if m.output_activation == "sigmoid" else 0
    d.n_layers = len(ws)
    d.table_size = g.table_size
    off = 0
    for l in range(g.levels):
        r = int(np.floor(g.base_resolution * g.growth_factor ** l))
        d.res[l] = r
        d.dense[l] = 1 if (r + 1) ** 3 <= g.table_size else 0
        d.tab_off[l] = off
        off += rows[l]
    d.widths[0] = ws[0].shape[1]
    wo = bo = 0
    for i, w in enumerate(ws):
        d.widths[i + 1] = w.shape[0]
        d.w_off[i] = wo
        d.b_off[i] = bo
        wo += w.size
        bo += bs[i].size
    d.tables = ptr(tab)
    d.weights = ptr(wt)
    d.biases = ptr(bt)
    d.clip01 = 1 if clip else 0
    return DeviceField(d, (tab, wt, bt))


def _param_fingerprint(model):
    """Content fingerprint of an INR's parameters (1.4 MB for the default model, a CRC
    in well under a millisecond): in-place edits (the reference's optimizers update
    arrays in place, users may write model.tables[i][:]) invalidate the cached copy."""
    import zlib

    crc = 0
    for a in getattr(model, "parameters", lambda: [])():
        a = np.ascontiguousarray(a)
        crc = zlib.crc32(a.view(np.uint8).reshape(-1), crc)
        crc = zlib.crc32(repr((a.shape, a.dtype.str)).encode(), crc)
    return ("inr", crc)


def _lattice_identity(field_src):
    """Lattices can be GBs: keyed on the array's identity and data address (a lattice
    edited in place needs a new field object)."""
    lat = getattr(field_src, "lattice", None)
    if lat is None:
        return ("other", id(field_src))
    return ("lattice", id(lat), lat.__array_interface__["data"][0], lat.shape)


def device_field(field_src, device=None, clip=True) -> DeviceField:
    """Descriptor for this package's fields or the reference's (duck typed)."""
    dev = require_cuda(device)
    model = getattr(field_src, "model", None)
    key = (str(dev), clip, _param_fingerprint(model) if model is not None else _lattice_identity(field_src))
    cache = getattr(field_src, "_cinr_dev", None)
    if cache is not None and cache[0] == key:
        return cache[1]
    if model is not None and hasattr(model, "tables") and hasattr(model, "grid_config"):
        df = _inr_desc(model, dev, clip)
    elif getattr(field_src, "lattice", None) is not None:
        lat = np.ascontiguousarray(field_src.lattice, dtype=np.float32)
        lt = torch.from_numpy(lat.copy()).to(dev)
        d = N.VcbField()
        d.kind = 1
        d.lattice = ptr(lt)
        d.lz, d.ly, d.lx = lat.shape
        df = DeviceField(d, (lt,))
    elif getattr(field_src, "kind", None) in PROC_IDS:
        d = N.VcbField()
        d.kind = 2
        d.proc = PROC_IDS[field_src.kind]
        df = DeviceField(d, ())
    else:
        raise ConfigError(
            f"field type {type(field_src).__name__} has no GPU decoder (supported: hash-grid INR, lattice, procedural)")
    try:
        field_src._cinr_dev = (key, df)
    except AttributeError:
        pass
    return df


def field_points(df: DeviceField, pos: np.ndarray, return_flag=False, stream=None):
    """Field.sample_batch through vcb_field_points (host in, host out)."""
    dev = require_cuda()
    n = pos.shape[0]
    p = torch.from_numpy(np.ascontiguousarray(pos, dtype=np.float64)).to(dev, non_blocking=False)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    N.call("vcb_field_points", C.byref(df.desc), n, ptr(p), ptr(out), ptr(flag), stream_ptr(stream))
    res = out.cpu().numpy()
    if return_flag:
        return res, bool(flag.item())
    return res
