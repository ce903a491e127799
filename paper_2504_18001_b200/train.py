"""INR training on the GPU (the reference's inr/train.py:1-143).

`train(model, field_src, steps, ...)` has the reference's signature and result:
MSE on uniformly random coordinate batches drawn from numpy's PCG64 stream
`default_rng(seed)` (the device reproduces the draws), Adam or SGD with optional
gradient-norm clipping, a per-step loss trace, and TrainingDivergedError at the
first non-finite loss with the last finite update kept.  The step runs in
`csrc/train.cu` (encode -> MLP -> MSE -> MLP backward -> hash-table scatter-add ->
optimizer), for the default 8x2 hash grid + 16-32-32-1 network.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import _inr_desc, device_field, ptr, require_cuda
from .errors import ConfigError, TrainingDivergedError
from .render import pcg64_seeded_state

DEFAULT_BATCH_SIZE = 65536
MASK64 = (1 << 64) - 1


@dataclass
class TrainResult:
    model: object
    loss_trace: np.ndarray

    @property
    def final_loss(self) -> float:
        return float(self.loss_trace[-1])


def train(model, field_src, steps: int, batch_size: int = DEFAULT_BATCH_SIZE, learning_rate: float = 1e-2,
          optimizer: str = "adam", seed: int = 0, clip_norm: float | None = None, device=None) -> TrainResult:
    """train.py:98-132 on the GPU."""
    if steps < 1:
        raise ValueError("steps must be >= 1")
    g, mc = model.grid_config, model.mlp_config
    if (g.levels, g.features_per_entry, mc.hidden_width, mc.hidden_layers) != (8, 2, 32, 2):
        raise ConfigError("the GPU trainer supports the default 8x2 hash grid + 16-32-32-1 MLP")
    if np.dtype(getattr(model, "dtype", np.float32)) != np.float32:
        # the reference updates parameters in the model's dtype; the device trainer is f32
        raise ConfigError(f"the GPU trainer needs a float32 model (got {np.dtype(model.dtype)})")
    dev = require_cuda(device)
    df = _inr_desc(model, dev, clip=False)
    tab, wt, bt = df._keep
    tgt = device_field(field_src, dev)
    B = int(batch_size)
    n_tab, n_w, n_b = tab.numel(), wt.numel(), bt.numel()
    n_p = n_tab + n_w + n_b
    f64 = dict(dtype=torch.float64, device=dev)
    grads, m, v = torch.zeros(n_p, **f64), torch.zeros(n_p, **f64), torch.zeros(n_p, **f64)
    pos = torch.empty(3 * B, **f64)
    targets = torch.empty(B, dtype=torch.float32, device=dev)
    loss = torch.zeros(int(steps), **f64)
    scratch = torch.zeros(8, **f64)
    nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
    jump = torch.empty(int(N.load().vcb_train_workspace_bytes(B)), dtype=torch.uint8, device=dev)
    st, inc = pcg64_seeded_state(seed)
    p = N.VcbTrainParams()
    p.model = df.desc
    p.target = tgt.desc
    p.batch, p.steps, p.step0 = B, int(steps), 0
    p.optimizer = 2 if learning_rate == 0.0 else (0 if optimizer == "adam" else 1)
    p.lr, p.beta1, p.beta2, p.eps = float(learning_rate), 0.9, 0.999, 1e-9
    p.clip_norm = float(clip_norm) if clip_norm is not None else 0.0
    p.flags = 4 if clip_norm is not None else 0
    p.pcg_state[0], p.pcg_state[1] = st & MASK64, st >> 64
    p.pcg_inc[0], p.pcg_inc[1] = inc & MASK64, inc >> 64
    p.draw0 = 0
    p.n_table_params, p.n_weights, p.n_params = n_tab, n_w, n_p
    p.grads, p.m, p.v = ptr(grads), ptr(m), ptr(v)
    p.pos, p.targets, p.loss, p.scratch, p.nonfinite, p.jump = (ptr(pos), ptr(targets), ptr(loss), ptr(scratch),
                                                                 ptr(nonfinite), ptr(jump))
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        N.call("vcb_train_steps", C.byref(p), C.c_void_p(stream.cuda_stream))
    stream.synchronize()
    trace = loss.cpu().numpy() / B
    # parameters back into the model (tables split per level, like model.parameters())
    rows = [t.shape[0] for t in model.tables]
    nf = model.grid_config.features_per_entry
    flat = tab.cpu().numpy().reshape(-1, nf)
    tables = np.split(flat, np.cumsum(rows)[:-1])
    wflat, bflat = wt.cpu().numpy(), bt.cpu().numpy()
    ws, bs, o, q = [], [], 0, 0
    for w, b in zip(model.weights, model.biases):
        ws.append(wflat[o:o + w.size].reshape(w.shape).copy())
        bs.append(bflat[q:q + b.size].reshape(b.shape).copy())
        o += w.size
        q += b.size
    model.set_parameters([*[t.copy() for t in tables], *ws, *bs])
    bad = np.flatnonzero(~np.isfinite(trace))
    if bad.size:
        k = int(bad[0])
        raise TrainingDivergedError(f"loss became non-finite at step {k}", last_finite_step=k - 1 if k > 0 else None,
                                    loss_trace=trace[:k].copy())
    if int(nonfinite.item()):
        raise TrainingDivergedError("target field produced non-finite values", last_finite_step=None,
                                    loss_trace=trace)
    return TrainResult(model, trace)


def loss_and_grads(model, positions, targets, device=None):
    """train.py:16-37 on the GPU: MSE loss and the gradient of every parameter, in
    model.parameters() order (tables, weights, biases) and the model's dtype."""
    g, mc = model.grid_config, model.mlp_config
    if (g.levels, g.features_per_entry, mc.hidden_width, mc.hidden_layers) != (8, 2, 32, 2):
        raise ConfigError("the GPU trainer supports the default 8x2 hash grid + 16-32-32-1 MLP")
    dev = require_cuda(device)
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    tg = np.ascontiguousarray(np.asarray(targets, dtype=np.float32).reshape(-1))
    B = pos.shape[0]
    if tg.shape[0] != B:
        raise ValueError("positions and targets differ in length")
    df = _inr_desc(model, dev, clip=False)
    tab, wt, bt = df._keep
    n_tab, n_w, n_b = tab.numel(), wt.numel(), bt.numel()
    n_p = n_tab + n_w + n_b
    f64 = dict(dtype=torch.float64, device=dev)
    grads = torch.zeros(n_p, **f64)
    dpos = torch.from_numpy(pos).to(dev)
    dtg = torch.from_numpy(tg).to(dev)
    loss = torch.zeros(1, **f64)
    scratch = torch.zeros(8, **f64)
    nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
    jump = torch.empty(int(N.load().vcb_train_workspace_bytes(B)), dtype=torch.uint8, device=dev)
    p = N.VcbTrainParams()
    p.model = df.desc
    p.batch, p.steps, p.step0 = B, 1, 0
    p.optimizer, p.flags = 2, 3
    p.n_table_params, p.n_weights, p.n_params = n_tab, n_w, n_p
    p.grads, p.m, p.v = ptr(grads), ptr(grads), ptr(grads)
    p.pos, p.targets, p.loss, p.scratch, p.nonfinite, p.jump = (ptr(dpos), ptr(dtg), ptr(loss), ptr(scratch),
                                                                 ptr(nonfinite), ptr(jump))
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        N.call("vcb_train_steps", C.byref(p), C.c_void_p(stream.cuda_stream))
    stream.synchronize()
    gh = grads.cpu().numpy().astype(model.dtype)
    out, o = [], 0
    for t in model.tables:
        out.append(gh[o:o + t.size].reshape(t.shape))
        o += t.size
    for w in model.weights:
        out.append(gh[o:o + w.size].reshape(w.shape))
        o += w.size
    for b in model.biases:
        out.append(gh[o:o + b.size].reshape(b.shape))
        o += b.size
    return float(loss.item()) / B, out


def psnr_on_lattice(model, field_src, dims=None) -> float:
    """train.py:135-143: reconstruction PSNR against the field's lattice, in dB."""
    dims = dims or field_src.domain.dims
    truth = field_src.sample_lattice(dims)
    approx = model.as_field().sample_lattice(dims)
    mse = float(np.mean((truth.astype(np.float64) - approx.astype(np.float64)) ** 2))
    if mse == 0.0:
        return float("inf")
    return 10.0 * np.log10(1.0 / mse)
