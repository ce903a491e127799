"""ctypes binding of the C ABI in include/cinr_b200.h (libcinr_b200.so).

There is no fallback: if the library cannot be loaded, every GPU entry point
raises NativeUnavailable.  Struct layouts mirror the header field for field.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import VoxcacheError

MAX_LOD = 32
MAX_LEVELS = 16
MAX_LAYERS = 8

_LIB = None
_SO = Path(__file__).resolve().parent / "_lib" / "libcinr_b200.so"
if os.environ.get("CINR_LIB"):  # tools: an alternative build of the same library (A/B measurements)
    _SO = Path(os.environ["CINR_LIB"]).resolve()
elif os.environ.get("CINR_STATS"):  # diagnostics build (tools only), built by `CINR_STATS=1 python -m ..._build`
    _SO = _SO.with_name("libcinr_b200_stats.so")


class NativeUnavailable(VoxcacheError):
    """The sm_100a library is missing or failed to load (no CPU fallback exists)."""


class NativeError(VoxcacheError):
    """A C-ABI call returned a non-zero status."""


i64 = C.c_int64
i32 = C.c_int32
f64 = C.c_double
vp = C.c_void_p


class VcbCamera(C.Structure):
    _fields_ = [("origin", f64 * 3), ("rot", f64 * 9), ("tan_h", f64), ("tan_v", f64), ("width", i32), ("height", i32),
                ("row0", i32), ("row_step", i32), ("rows", i32), ("pad_", i32)]


class VcbMarchStatic(C.Structure):
    _fields_ = [("adaptive", i32), ("skip_empty", i32), ("dt_base", f64), ("mu_floor", f64),
                ("gx", i64), ("gy", i64), ("gz", i64), ("cwx", f64), ("cwy", f64), ("cwz", f64)]


class VcbProbeStatic(C.Structure):
    _fields_ = [("vx", f64), ("vy", f64), ("vz", f64), ("lod_scale", f64), ("mode", i32), ("max_lod", i32),
                ("b", i64), ("b_pow2", i32), ("pad_", i32), ("grid", (i64 * 3) * MAX_LOD), ("offset", i64 * MAX_LOD)]


class VcbField(C.Structure):
    _fields_ = [("kind", i32), ("levels", i32), ("feats", i32), ("out_sigmoid", i32), ("n_layers", i32),
                ("table_size", i64), ("res", i32 * MAX_LEVELS), ("dense", i32 * MAX_LEVELS),
                ("tab_off", i64 * MAX_LEVELS), ("widths", i32 * (MAX_LAYERS + 1)),
                ("w_off", i64 * MAX_LAYERS), ("b_off", i64 * MAX_LAYERS),
                ("tables", vp), ("weights", vp), ("biases", vp),
                ("lattice", vp), ("lx", i64), ("ly", i64), ("lz", i64), ("proc", i32), ("clip01", i32)]


class VcbBrickGeom(C.Structure):
    _fields_ = [("dims", i64 * 3), ("b", i64), ("n_lod", i32), ("pad_", i32), ("grid", (i64 * 3) * MAX_LOD),
                ("offset", i64 * MAX_LOD)]


class VcbFrameStats(C.Structure):
    _fields_ = [("requests", i64), ("exact", i64), ("fallback", i64), ("miss", i64), ("iterations", i64),
                ("rays", i64), ("misses_resolved", i64), ("nonfinite", i64), ("deferred_misses", i64),
                ("pad_", i64 * 7)]


class VcbCacheState(C.Structure):
    _fields_ = [("next_free", i64), ("loaded_total", i64), ("n_staged", i64), ("staged_frame", i64),
                ("decode_error", i64), ("bricks_loaded", i64), ("deferred", i64), ("inserted", i64),
                ("n_inflight", i64), ("n_reports", i64), ("n_pending", i64), ("n_batch", i64), ("pad_", i64 * 4)]


class VcbFrameParams(C.Structure):
    _fields_ = [("cam", VcbCamera), ("adv", VcbMarchStatic), ("probe", VcbProbeStatic), ("cached", i32),
                ("paged_dist", i32), ("cache_frame", i64), ("rng_base", C.c_uint64), ("term", f64), ("bg", f64 * 3),
                ("lut_size", i32), ("max_iterations", i32), ("epoch", C.c_uint32), ("timing", i32),
                ("mu", vp), ("lut", vp), ("table", vp), ("pool", vp), ("last_used", vp), ("miss_count", vp),
                ("field", VcbField), ("image", vp), ("stats", vp), ("workspace", vp), ("workspace_bytes", i64),
                ("impl", i32), ("image_global", i32), ("miss_budget", i64)]


class VcbMaintParams(C.Structure):
    _fields_ = [("geom", VcbBrickGeom), ("total", i64), ("slots", i64), ("session_frame", i64),
                ("max_requests", i32), ("ranking", i32), ("rank_clamp", i64), ("lin_bits", i32), ("lod_bits", i32),
                ("table", vp), ("pool", vp), ("owner", vp), ("last_used", vp), ("miss_count", vp),
                ("req_base", vp), ("req_hits", vp), ("state", vp), ("staging", vp), ("staged_keys", vp),
                ("workspace", vp), ("workspace_bytes", i64), ("dbg_reports", vp), ("field", VcbField),
                ("frame_stats", vp), ("decode_budget", i64), ("defer_decode", i32), ("pad2_", i32),
                ("pending_list", vp), ("list_counts", vp)]


class VcbPtParams(C.Structure):
    _fields_ = [("spp", i32), ("max_walk", i32), ("density", f64), ("ambient", f64), ("light", f64 * 3),
                ("n_tf", i32), ("pad_", i32), ("tf", vp), ("pcg_state", C.c_uint64 * 2), ("pcg_inc", C.c_uint64 * 2),
                ("lane_seed", C.c_uint64), ("lane_frame", i64), ("workspace", vp), ("workspace_bytes", i64)]


class VcbTrainParams(C.Structure):
    _fields_ = [("model", VcbField), ("target", VcbField), ("batch", i64), ("steps", i64), ("step0", i64),
                ("optimizer", i32), ("flags", i32), ("lr", f64), ("beta1", f64), ("beta2", f64), ("eps", f64),
                ("clip_norm", f64), ("pcg_state", C.c_uint64 * 2), ("pcg_inc", C.c_uint64 * 2),
                ("draw0", C.c_uint64), ("n_table_params", i64), ("n_weights", i64), ("n_params", i64),
                ("grads", vp), ("m", vp), ("v", vp), ("pos", vp), ("targets", vp), ("loss", vp), ("scratch", vp),
                ("nonfinite", vp), ("jump", vp)]


_PROTOS = {
    "vcb_last_error": (C.c_char_p, []),
    "vcb_abi_version": (i32, []),
    "vcb_device_sm_count": (i32, []),
    "vcb_struct_sizes": (i32, [vp, i32]),
    "vcb_raygen_pass": (i32, [i64, vp, vp, vp, f64, f64, vp, vp, vp, vp, vp]),
    "vcb_advance_pass": (i32, [i64, vp, vp, vp, vp, vp, vp, vp, C.POINTER(VcbMarchStatic), vp, vp, vp, vp, vp, vp, vp]),
    "vcb_probe_pass": (i32, [i64, vp, vp, vp, C.POINTER(VcbProbeStatic), vp, vp, vp, i64, vp, vp, vp, vp, vp]),
    "vcb_shade_pass": (i32, [i64, vp, vp, vp, vp, i64, i32, f64, f64, vp, vp, vp, vp]),
    "vcb_debug_pow": (i32, [i64, vp, vp, vp, vp]),
    "vcb_debug_pow_accurate": (i32, [i64, vp, vp, vp, vp]),
    "vcb_field_points": (i32, [C.POINTER(VcbField), i64, vp, vp, vp, vp]),
    "vcb_field_bricks": (i32, [C.POINTER(VcbField), C.POINTER(VcbBrickGeom), i64, vp, vp, vp, vp]),
    "vcb_inr_points_tc": (i32, [C.POINTER(VcbField), i64, vp, vp, vp, vp]),
    "vcb_inr_bricks_tc": (i32, [C.POINTER(VcbField), C.POINTER(VcbBrickGeom), i64, vp, vp, vp, vp]),
    "vcb_macro_minmax": (i32, [C.POINTER(VcbField), vp, i64, vp, vp, vp]),
    "vcb_update_majorants": (i32, [vp, vp, i64, vp, i32, vp, vp]),
    "vcb_frame_rgba8": (i32, [vp, i64, vp, vp]),
    "vcb_frame_workspace_bytes": (i64, [i64, i32]),
    "vcb_march_frame": (i32, [C.POINTER(VcbFrameParams), vp]),
    "vcb_pt_workspace_bytes": (i64, [i64]),
    "vcb_pathtrace_frame": (i32, [C.POINTER(VcbFrameParams), C.POINTER(VcbPtParams), vp]),
    "vcb_debug_pt_math": (i32, [i64, vp, vp, vp, vp, vp, vp]),
    "vcb_train_workspace_bytes": (i64, [i64]),
    "vcb_train_steps": (i32, [C.POINTER(VcbTrainParams), vp]),
    "vcb_trace_free_flight": (i32, [C.POINTER(VcbFrameParams), C.POINTER(VcbPtParams), i64, vp, vp, vp, vp, vp, vp,
                                    vp, vp]),
    "vcb_march_timing": (i32, [i32, vp, vp]),
    "vcb_last_launch_count": (i64, []),
    "vcb_frame_trace": (i32, [vp, i64, i32, i32, vp, vp]),
    "vcb_frame_counters": (i32, [vp, i64, i32, vp]),
    "vcb_maint_workspace_bytes": (i64, [i64, i64, i32]),
    "vcb_maintenance": (i32, [C.POINTER(VcbMaintParams), vp]),
    "vcb_maint_decode": (i32, [C.POINTER(VcbMaintParams), vp]),
    "vcb_share_keys": (i32, [C.POINTER(VcbMaintParams), vp, vp]),
    "vcb_share_plan": (i32, [vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "vcb_share_decode": (i32, [C.POINTER(VcbMaintParams), vp, vp, i32, vp, vp, vp]),
    "vcb_share_scatter": (i32, [C.POINTER(VcbMaintParams), vp, vp, i32, vp, vp, vp, vp, vp, vp]),
    "vcb_maint_graph_create": (i32, [C.POINTER(VcbMaintParams), C.POINTER(vp)]),
    "vcb_maint_graph_launch": (i32, [vp, C.POINTER(VcbMaintParams), vp]),
    "vcb_maint_graph_destroy": (None, [vp]),
}

EXPORTS = tuple(_PROTOS)


def library_path() -> Path:
    return _SO


def load():
    """Load (building in-tree first when sources are newer) the sm_100a library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    try:
        import fcntl

        from . import _build

        if _build.needs_build():
            # one builder at a time (torchrun ranks share the tree); the others wait and
            # then find the library current
            _build.OUT_DIR.mkdir(exist_ok=True)
            with open(_build.OUT_DIR / ".build.lock", "w") as lk:
                fcntl.flock(lk, fcntl.LOCK_EX)
                try:
                    if _build.needs_build():
                        _build.build()
                finally:
                    fcntl.flock(lk, fcntl.LOCK_UN)
    except Exception as exc:
        if not _SO.exists():
            raise NativeUnavailable(f"cannot build {_SO.name}: {exc}") from exc
        # a prebuilt library without a toolchain is fine; a failed rebuild of changed
        # sources is not (the stale library would not match them)
        if "nvcc not found" not in str(exc):
            raise NativeUnavailable(f"rebuild of {_SO.name} failed: {exc}") from exc
    if not _SO.exists():
        raise NativeUnavailable(f"{_SO} not built (run __graft_entry__.build())")
    try:
        lib = C.CDLL(str(_SO))
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {_SO}: {exc}") from exc
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _check_abi(lib)
    _LIB = lib
    return lib


def _check_abi(lib):
    """ctypes mirrors vs the library's struct sizes, on every load."""
    import numpy as np

    out = np.zeros(16, dtype=np.int64)
    n = lib.vcb_struct_sizes(out.ctypes.data, 16)
    bad = [(s.__name__, C.sizeof(s), int(out[i])) for i, s in enumerate(STRUCTS[:n]) if C.sizeof(s) != int(out[i])]
    if bad:
        raise NativeUnavailable(f"{_SO.name} ABI mismatch (python, C sizeof): {bad}")


STRUCTS = (VcbCamera, VcbMarchStatic, VcbProbeStatic, VcbField, VcbBrickGeom, VcbFrameStats, VcbCacheState,
           VcbFrameParams, VcbMaintParams, VcbPtParams, VcbTrainParams)


def struct_sizes():
    """(python sizeof, C sizeof) per ABI struct; host-only call, no GPU needed."""
    import numpy as np

    out = np.zeros(16, dtype=np.int64)
    n = load().vcb_struct_sizes(out.ctypes.data, 16)
    return [(s.__name__, C.sizeof(s), int(out[i])) for i, s in enumerate(STRUCTS[:n])]


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = load().vcb_last_error().decode(errors="replace")
        raise NativeError(f"{what}: {msg}" if what else msg)


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc
