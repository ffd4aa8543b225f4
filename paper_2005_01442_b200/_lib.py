"""ctypes binding of include/voxelray_b200.h (the C-ABI boundary).

The shared library is built in-tree by ``_build.py`` (``__graft_entry__.build()``).
There is no fallback: if the library is missing or no CUDA device is present,
every entry point that needs the GPU raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "libvoxelray_b200.so"
if os.environ.get("VR_LIB"):  # development: load an alternative build of the same ABI
    LIB_PATH = Path(os.environ["VR_LIB"]).resolve()

VR_OK, VR_EINVALID, VR_EBLOCKSPEC, VR_EISO, VR_ECUDA, VR_ENOMEM = range(6)
MODE_DVR, MODE_ISO = 0, 1
CLS_POST, CLS_PRE, CLS_PREINT = 0, 1, 2
PINHOLE, ORTHOGRAPHIC = 0, 1
PHANTOM_KINDS = {"sphere": 0, "shell": 1, "torso": 2}
SAMPLE_FORMATS = {"u8": 0, "i16": 1, "u16": 2, "i32": 3}

# every symbol include/voxelray_b200.h declares
EXPORTS = (
    "vr_last_error", "vr_abi_version", "vr_volume_create", "vr_volume_ingest", "vr_phantom_create",
    "vr_volume_destroy", "vr_volume_culling_tables", "vr_volume_info", "vr_volume_data", "vr_volume_download",
    "vr_grid_create", "vr_grid_destroy", "vr_grid_shape", "vr_grid_minmax",
    "vr_grid_visibility", "vr_render", "vr_render_views", "vr_render_to_host", "vr_preclassify",
    "vr_sample_points", "vr_gradient_points", "vr_threshold_count", "vr_threshold_measure",
    "vr_ball_measure",
    "vr_event_create", "vr_event_destroy", "vr_event_elapsed_ms", "vr_interleave_size",
    "vr_image_sse", "vr_image_ssim", "vr_enable_peer_access",
)


class Camera(ctypes.Structure):
    _fields_ = [
        ("projection", ctypes.c_int32), ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("tile_x", ctypes.c_int32), ("tile_y", ctypes.c_int32), ("tile_w", ctypes.c_int32),
        ("tile_h", ctypes.c_int32), ("interleave_n", ctypes.c_int32),
        ("interleave_k", ctypes.c_int32), ("interleave_frame", ctypes.c_int32),
        ("position", ctypes.c_double * 3), ("fwd", ctypes.c_double * 3),
        ("right", ctypes.c_double * 3), ("up", ctypes.c_double * 3),
        ("half_w", ctypes.c_double), ("half_h", ctypes.c_double),
    ]


class RenderParams(ctypes.Structure):
    _fields_ = [
        ("step", ctypes.c_double), ("ref_step", ctypes.c_double),
        ("mode", ctypes.c_int32), ("cubic", ctypes.c_int32), ("lighting", ctypes.c_int32),
        ("classify", ctypes.c_int32),
        ("isovalue", ctypes.c_double), ("term_alpha", ctypes.c_double),
        ("ka", ctypes.c_double), ("kd", ctypes.c_double), ("ks", ctypes.c_double),
        ("shininess", ctypes.c_double), ("bg", ctypes.c_double * 4),
        ("lut_lo", ctypes.c_double), ("lut_hi", ctypes.c_double),
        ("nlut", ctypes.c_int32), ("ntbl", ctypes.c_int32), ("margin", ctypes.c_double),
    ]


class RenderOutputs(ctypes.Structure):
    _fields_ = [
        ("pixels", ctypes.c_void_p), ("premult", ctypes.c_void_p), ("depth", ctypes.c_void_p),
        ("taken", ctypes.c_void_p), ("skipped", ctypes.c_void_p), ("blocks_hit", ctypes.c_void_p),
        ("totals", ctypes.c_void_p), ("work", ctypes.c_void_p),
        ("ev_start", ctypes.c_void_p), ("ev_stop", ctypes.c_void_p),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load the extension; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH.name} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
            "There is no CPU fallback."
        )
    L = ctypes.CDLL(str(LIB_PATH))
    P, i64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    VP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "vr_last_error": ([], ctypes.c_char_p),
        "vr_abi_version": ([], ctypes.c_int),
        "vr_volume_create": ([ctypes.c_int, i64, i64, i64, f64, f64, f64, P, ctypes.c_int, P, VP], ctypes.c_int),
        "vr_volume_ingest": ([ctypes.c_int, ctypes.c_int, i64, i64, i64, f64, f64, f64, P, ctypes.c_int, P, P, VP, P],
                             ctypes.c_int),
        "vr_phantom_create": ([ctypes.c_int, ctypes.c_int, i64, i64, i64, f64, f64, f64, P, VP], ctypes.c_int),
        "vr_volume_destroy": ([P], ctypes.c_int),
        "vr_volume_culling_tables": ([P, P, P], ctypes.c_int),
        "vr_volume_info": ([P, P, P, P, P], ctypes.c_int),
        "vr_volume_data": ([P], P),
        "vr_volume_download": ([P, P, P], ctypes.c_int),
        "vr_grid_create": ([P, i64, i64, P, VP], ctypes.c_int),
        "vr_grid_destroy": ([P], ctypes.c_int),
        "vr_grid_shape": ([P, P], ctypes.c_int),
        "vr_grid_minmax": ([P, P, P, P], ctypes.c_int),
        "vr_grid_visibility": ([P, P, i32, f64, f64, P, P, P, P], ctypes.c_int),
        "vr_render": ([P, P, ctypes.POINTER(Camera), ctypes.POINTER(RenderParams), P, P, P,
                       ctypes.POINTER(RenderOutputs), P], ctypes.c_int),
        "vr_render_views": ([P, P, ctypes.POINTER(Camera), P, i32, ctypes.POINTER(RenderParams), P, P, P,
                             ctypes.POINTER(RenderOutputs), P], ctypes.c_int),
        "vr_render_to_host": ([P, P, ctypes.POINTER(Camera), ctypes.POINTER(RenderParams), P, P,
                               P, P, P, P, P], ctypes.c_int),
        "vr_preclassify": ([P, P, i32, f64, f64, P, P], ctypes.c_int),
        "vr_sample_points": ([P, P, i64, ctypes.c_int, P, P], ctypes.c_int),
        "vr_gradient_points": ([P, P, i64, ctypes.c_int, P, P], ctypes.c_int),
        "vr_threshold_count": ([P, i32, P, P], ctypes.c_int),
        "vr_threshold_measure": ([P, i32, P, P], ctypes.c_int),
        "vr_ball_measure": ([P, i32, P, P, i64, P, P, P], ctypes.c_int),
        "vr_event_create": ([VP], ctypes.c_int),
        "vr_event_destroy": ([P], ctypes.c_int),
        "vr_event_elapsed_ms": ([P, P, ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
        "vr_interleave_size": ([ctypes.POINTER(Camera), P, P], ctypes.c_int),
        "vr_image_sse": ([P, P, i64, i64, ctypes.c_int, ctypes.c_int, P, P], ctypes.c_int),
        "vr_enable_peer_access": ([ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "vr_image_ssim": ([P, P, i64, i64, ctypes.c_int, ctypes.c_int, P, P, P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(status: int) -> None:
    """Map a C-ABI status to the reference's exception classes (errors.py)."""
    if status == VR_OK:
        return
    msg = (load().vr_last_error() or b"").decode(errors="replace")
    if status == VR_EINVALID:
        if msg.startswith("EmptyBlock"):
            raise errors.EmptyBlock(msg)
        raise errors.InvalidSettings(msg)
    if status == VR_EBLOCKSPEC:
        raise errors.InvalidBlockSpec(msg)
    if status == VR_EISO:
        raise errors.IsovalueOutOfRange(msg)
    raise errors.DeviceError(f"status {status}: {msg}")


def ptr(obj) -> ctypes.c_void_p:
    """Device/host address of a torch tensor or numpy array."""
    if obj is None:
        return ctypes.c_void_p(0)
    if hasattr(obj, "data_ptr"):
        return ctypes.c_void_p(obj.data_ptr())
    return obj.ctypes.data_as(ctypes.c_void_p)


def ptr_stream(stream) -> ctypes.c_void_p:
    """cudaStream_t of a torch.cuda.Stream (or a raw handle); None = legacy default."""
    if stream is None:
        return ctypes.c_void_p(0)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))
