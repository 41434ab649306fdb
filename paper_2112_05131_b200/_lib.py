"""ctypes binding of libplx.so (the C ABI declared in include/plx.h).

The shared library is built in-tree (paper_2112_05131_b200/libplx.so, see
csrc/Makefile and __graft_entry__.build()).  There is no fallback: if the
library is missing or the device is not an sm_100-class GPU, every entry
point raises -- the product path never degrades to CPU code.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PLX_LIB: development override (A/B of kernel variants built elsewhere in-tree)
LIB_PATH = os.environ.get("PLX_LIB") or os.path.join(_HERE, "libplx.so")

PLX_OK, PLX_EINVAL, PLX_ECUDA = 0, 1, 2
ROW = 28
STRIDE = 32   # row pitch of table / grad / v in floats (128-byte rows, plx.h)


class PlxError(RuntimeError):
    pass


class PlxGrid(ctypes.Structure):
    _fields_ = [("links", ctypes.c_void_p), ("table", ctypes.c_void_p),
                ("density", ctypes.c_void_p), ("dims", ctypes.c_int64 * 3), ("rows", ctypes.c_int64),
                ("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
                ("scale", ctypes.c_double * 3), ("dmax", ctypes.c_double * 3),
                ("cell_occ", ctypes.c_void_p), ("sigma_lat", ctypes.c_void_p),
                ("row_cell", ctypes.c_void_p), ("brick_dead", ctypes.c_void_p)]


class PlxGrad(ctypes.Structure):
    _fields_ = [("grad", ctypes.c_void_p), ("tmask", ctypes.c_void_p),
                ("tids", ctypes.c_void_p), ("tcnt", ctypes.c_void_p)]


MAX_PEERS = 8


class PlxDpPeers(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("rank", ctypes.c_int32), ("rows", ctypes.c_int64),
                ("grad", ctypes.c_void_p * MAX_PEERS), ("tmask", ctypes.c_void_p * MAX_PEERS),
                ("table", ctypes.c_void_p * MAX_PEERS), ("density", ctypes.c_void_p * MAX_PEERS),
                ("sigma_lat", ctypes.c_void_p * MAX_PEERS)]


class PlxRenderOpts(ctypes.Structure):
    _fields_ = [("step", ctypes.c_double), ("stop_thresh", ctypes.c_double),
                ("bg", ctypes.c_double * 3), ("nearest", ctypes.c_int32),
                ("absolute", ctypes.c_int32), ("stats", ctypes.c_void_p)]


CAM = 16   # doubles per camera record (PLX_CAM)


class PlxCameras(ctypes.Structure):
    _fields_ = [("cams", ctypes.c_void_p), ("rgb", ctypes.c_void_p), ("pixel", ctypes.c_void_p),
                ("n_views", ctypes.c_int64), ("width", ctypes.c_int64),
                ("height", ctypes.c_int64), ("ndc", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("scale", ctypes.c_double)]


class PlxRays(ctypes.Structure):
    _fields_ = [("origins", ctypes.c_void_p), ("dirs", ctypes.c_void_p),
                ("viewdirs", ctypes.c_void_p), ("target", ctypes.c_void_p),
                ("jitter", ctypes.c_void_p), ("idx", ctypes.c_void_p),
                ("n", ctypes.c_int64), ("cams", ctypes.POINTER(PlxCameras))]


class PlxStepArgs(ctypes.Structure):
    _fields_ = [("rays", PlxRays), ("opts", PlxRenderOpts), ("up_scale", ctypes.c_double),
                ("lam_cauchy", ctypes.c_double), ("scratch", ctypes.c_void_p),
                ("scratch_bytes", ctypes.c_int64), ("tv_start", ctypes.c_int64),
                ("tv_count", ctypes.c_int64), ("tv_fac", ctypes.c_double * 3),
                ("tv_eps", ctypes.c_double), ("tv_f_sigma", ctypes.c_double),
                ("tv_f_sh", ctypes.c_double), ("update", ctypes.c_int32),
                ("rmsprop", ctypes.c_int32), ("v", ctypes.c_void_p),
                ("lr_sigma", ctypes.c_double), ("lr_sh", ctypes.c_double),
                ("beta", ctypes.c_double), ("eps", ctypes.c_double),
                ("sums", ctypes.c_void_p), ("count", ctypes.c_void_p),
                ("events", ctypes.c_void_p * 4), ("dev_tv_start", ctypes.c_void_p),
                ("dev_lr", ctypes.c_void_p), ("dev_idx_off", ctypes.c_void_p),
                ("host_params", ctypes.c_void_p), ("dev_params", ctypes.c_void_p),
                ("host_sums", ctypes.c_void_p)]


class PlxMsi(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("radii", ctypes.c_void_p), ("L", ctypes.c_int64),
                ("H", ctypes.c_int64), ("W", ctypes.c_int64)]


class PlxMsiGrad(ctypes.Structure):
    _fields_ = [("grad", ctypes.c_void_p), ("tmask", ctypes.c_void_p), ("tids", ctypes.c_void_p),
                ("tcnt", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

# name -> argtypes (restype int unless listed in _RESTYPE)
_SIGS = {
    "plx_render_fwd": [ctypes.POINTER(PlxGrid), ctypes.POINTER(PlxRays),
                       ctypes.POINTER(PlxRenderOpts), _P, _P, _P, _P],
    "plx_render_scratch_bytes": [ctypes.POINTER(PlxGrid), ctypes.POINTER(PlxRenderOpts), _I64],
    "plx_render_fused_bwd": [ctypes.POINTER(PlxGrid), ctypes.POINTER(PlxRays),
                             ctypes.POINTER(PlxRenderOpts), _I32, _D, _D,
                             ctypes.POINTER(PlxGrad), _P, _P, _P, _I64, _P],
    "plx_max_weight": [ctypes.POINTER(PlxGrid), ctypes.POINTER(PlxRays),
                       ctypes.POINTER(PlxRenderOpts), _P, _P],
    "plx_tv": [ctypes.POINTER(PlxGrid), _P, _I64, _I64, _D, _D, _D, _D, _D, _D,
               _I32, _I32, _I32, _I32, ctypes.POINTER(PlxGrad), _P, _P],
    "plx_opt_step": [ctypes.POINTER(PlxGrid), _P, ctypes.POINTER(PlxGrad), _D, _D, _D,
                     _D, _I32, _I32, _P, _P, _P],
    "plx_clear_grad": [ctypes.POINTER(PlxGrad), _I64, _P, _P],
    "plx_count_touched": [_P, _I64, _P, _P],
    "plx_touched_list": [_P, _I64, _P, _P, _P, _P],
    "plx_pack_rows": [_P, _P, _P, _I64, _P, _P],
    "plx_opt_step_list": [ctypes.POINTER(PlxGrid), _P, ctypes.POINTER(PlxGrad), _P, _P, _P, _D,
                          _D, _D, _D, _I32, _I32, _P, _P, _P],
    "plx_dp_owner_update": [ctypes.POINTER(PlxDpPeers), _P, _P, _D, _D, _D, _D, _I32, _P, _P,
                            _P],
    "plx_ipc_export": [_P, ctypes.c_char_p, ctypes.POINTER(_I64)],
    "plx_ipc_import": [ctypes.c_char_p, _I64, ctypes.POINTER(_P), ctypes.POINTER(_P)],
    "plx_ipc_close": [_P],
    "plx_prune_mark": [ctypes.POINTER(PlxGrid), _P, _D, _P, _P, _P],
    "plx_prune_apply": [ctypes.POINTER(PlxGrid), _P, _P, _P, _P, _P],
    "plx_upsample_mark": [ctypes.POINTER(PlxGrid), ctypes.POINTER(_I64), _P, _P],
    "plx_upsample_apply": [ctypes.POINTER(PlxGrid), ctypes.POINTER(_I64), _P, _P, _P, _P],
    "plx_scan_scratch_bytes": [_I64],
    "plx_scan_ids": [_P, _I64, _P, _P, _P, _P],
    "plx_cell_occ_words": [ctypes.POINTER(_I64)],
    "plx_build_cell_occ": [ctypes.POINTER(PlxGrid), _P, _P],
    "plx_build_sigma_lat": [ctypes.POINTER(PlxGrid), _P, _P],
    "plx_build_row_cell": [ctypes.POINTER(PlxGrid), _P, _P],
    "plx_brick_words": [ctypes.POINTER(_I64)],
    "plx_build_brick_dead": [ctypes.POINTER(PlxGrid), _P, _P],
    "plx_grid_sample": [ctypes.POINTER(PlxGrid), _P, _I64, _I32, _P, _P],
    "plx_grid_sample_backward": [ctypes.POINTER(PlxGrid), _P, _P, _I64, _I32,
                                 ctypes.POINTER(PlxGrad), _P],
    "plx_train_step": [ctypes.POINTER(PlxGrid), ctypes.POINTER(PlxGrad),
                       ctypes.POINTER(PlxStepArgs), _P],
    "plx_msi_scratch_bytes": [ctypes.POINTER(PlxGrid), ctypes.POINTER(PlxMsi),
                              ctypes.POINTER(PlxRenderOpts), _I64],
    "plx_msi_render": [ctypes.POINTER(PlxGrid), ctypes.POINTER(PlxMsi), ctypes.POINTER(PlxRays),
                       ctypes.POINTER(PlxRenderOpts), _I32, _D, _D, _D, _D,
                       ctypes.POINTER(PlxGrad), ctypes.POINTER(PlxMsiGrad), _P, _P, _P, _P, _P,
                       _I64, _P],
    "plx_msi_tv": [ctypes.POINTER(PlxMsi), _P, _I64, _I64, _D, _D, _D,
                   ctypes.POINTER(PlxMsiGrad), _P, _P],
    "plx_msi_opt_step": [_P, _P, ctypes.POINTER(PlxMsiGrad), _I64, _D, _D, _D, _D, _I32, _I32,
                         _P, _P],
    "plx_generate_rays": [ctypes.POINTER(PlxCameras), _P, _I64, _P, _P, _P, _P, _P],
    "plx_to_ndc": [_P, _P, _P, _P, _I64, _P],
    "plx_image_metrics_scratch_bytes": [_I64, _I64, _I64],
    "plx_image_metrics": [_P, _P, _I64, _I64, _I64, _P, _D, _D, _P, _P, _I64, _P],
    "plx_release_streams": [],
    "plx_version": [],
    "plx_device_check": [],
}
_RESTYPE = {"plx_scan_scratch_bytes": _I64, "plx_render_scratch_bytes": _I64, "plx_cell_occ_words": _I64,
            "plx_brick_words": _I64,
            "plx_msi_scratch_bytes": _I64, "plx_image_metrics_scratch_bytes": _I64,
            "plx_version": ctypes.c_char_p}

EXPORTS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load libplx.so (no device needed).  Raises PlxError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise PlxError(
            f"{path} not found: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); "
            "there is no CPU fallback")
    lib = ctypes.CDLL(path)
    for name, argtypes in _SIGS.items():
        if os.environ.get("PLX_LIB") and not hasattr(lib, name):
            continue   # an older variant build (A/B) may lack newer entry points
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
    _lib = lib
    return lib


_device_ok = None


def lib():
    """The loaded library, after checking that a B200-class device exists."""
    global _device_ok
    L = load()
    if _device_ok is None:
        import torch
        if not torch.cuda.is_available():
            raise PlxError("no CUDA device: the plx path runs only on sm_100 GPUs "
                           "(no CPU fallback)")
        torch.cuda.init()
        _device_ok = L.plx_device_check() == 0
    if not _device_ok:
        raise PlxError("libplx.so needs a compute-capability 10.x (B200) device")
    return L


def check(status: int, what: str) -> None:
    if status == PLX_OK:
        return
    if status == PLX_EINVAL:
        raise ValueError(f"{what}: invalid argument")
    raise PlxError(f"{what}: CUDA error (status {status})")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


_scratch_cache: dict = {}


def render_scratch(c_grid, c_opts, n_rays: int, device):
    """Device workspace for plx_render_fused_bwd (cached per device, grown on
    demand).  Returns (ptr, nbytes, tensor)."""
    import torch
    need = int(lib().plx_render_scratch_bytes(ctypes.byref(c_grid), ctypes.byref(c_opts),
                                              int(n_rays)))
    if need < 0:
        raise ValueError("render_scratch: invalid grid / options")
    key = str(device)
    buf = _scratch_cache.get(key)
    if buf is None or buf.numel() < need:
        _scratch_cache.pop(key, None)
        buf = torch.empty(max(need, 1 << 20), dtype=torch.uint8, device=device)
        _scratch_cache[key] = buf
    return buf.data_ptr(), buf.numel(), buf


def dims_array(dims) -> ctypes.Array:
    return (ctypes.c_int64 * 3)(*[int(d) for d in dims])


def make_opts(step: float, stop: float, bg, nearest: bool, absolute: bool) -> PlxRenderOpts:
    o = PlxRenderOpts()
    o.step = float(step)
    o.stop_thresh = float(stop)
    o.bg = (ctypes.c_double * 3)(*[float(x) for x in np.asarray(bg, np.float64).reshape(3)])
    o.nearest = int(bool(nearest))
    o.absolute = int(bool(absolute))
    return o
