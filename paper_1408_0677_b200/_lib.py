"""ctypes binding of libmdc.so (the C-ABI declared in include/mdc.h).

There is no CPU fallback: importing the package works without a GPU (so the
host-side logic can be unit-tested), but every compute entry point calls
``require_cuda()`` and raises if the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MDC_LIB_PATH") or os.path.join(HERE, "libmdc.so")  # override: A/B experiments only

MDC_MEAN, MDC_AFFINE, MDC_RIGID = 1, 2, 3
MDC_F32, MDC_F64 = 0, 1
MDC_FLAG_NO_TC = 1
MDC_FLAG_TC_ONEPASS = 2  # A/B only: the experimental one-pass tensor-core kernel
VARIANT_CODE = {"mean": MDC_MEAN, "affine": MDC_AFFINE, "rigid": MDC_RIGID}

_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_c_d = ctypes.c_double
_vp = ctypes.c_void_p


class MdcMlsArgs(ctypes.Structure):
    _fields_ = [
        ("variant", _c_i32), ("dtype", _c_i32),
        ("width", _c_i32), ("height", _c_i32), ("row0", _c_i32), ("row1", _c_i32),
        ("n", _c_i64),
        ("d", _c_i32), ("ldq", _c_i32),
        ("x0", _c_d), ("y1", _c_d), ("sx", _c_d), ("sy", _c_d),
        ("pmx", _c_d), ("pmy", _c_d),
        ("alpha", _c_d), ("reg_eps", _c_d),
        ("pc", _vp), ("q", _vp), ("qm", _vp), ("axis", _vp),
        ("out", _vp),
        ("out_cs", _c_i64), ("out_rs", _c_i64), ("out_ps", _c_i64),
        ("bands", _vp),
        ("band_cs", _c_i64), ("band_rs", _c_i64),
        ("spacing", _vp),
        ("nonfinite", _vp),
        ("flags", _c_i32),
        ("workspace", _vp),
        ("workspace_bytes", ctypes.c_size_t),
        ("rgba", _vp), ("palette", _vp), ("palette_n", _c_i32),
        ("pm", _vp),
    ]


class MdcLayoutArgs(ctypes.Structure):
    _fields_ = [
        ("n", _c_i64), ("ntri", _c_i64),
        ("leaf", _c_i32),
        ("c", _c_d), ("spring", _c_d), ("dlen", _c_d), ("eta", _c_d), ("theta", _c_d),
        ("csr_off", _vp), ("csr_tgt", _vp), ("tris", _vp), ("inc_off", _vp), ("inc", _vp),
        ("pos", _vp),
        ("workspace", _vp),
        ("workspace_bytes", ctypes.c_size_t),
        ("dbg_bh", _vp), ("dbg_force", _vp), ("dbg_scale", _vp),
        ("part_rank", _c_i32), ("part_world", _c_i32),
    ]


class MdcLinearArgs(ctypes.Structure):
    _fields_ = [
        ("width", _c_i32), ("height", _c_i32), ("row0", _c_i32), ("row1", _c_i32),
        ("x0", _c_d), ("y1", _c_d), ("sx", _c_d), ("sy", _c_d),
        ("n", _c_i64), ("ntri", _c_i64),
        ("nch", _c_i32), ("dtype", _c_i32),
        ("pos", _vp), ("tvals", _vp),
        ("tris", _vp), ("hull", _vp),
        ("nhull", _c_i32),
        ("out", _vp),
        ("out_cs", _c_i64), ("out_rs", _c_i64), ("out_ps", _c_i64),
        ("workspace", _vp),
    ]


class MdcRenderArgs(ctypes.Structure):
    _fields_ = [
        ("mode", _c_i32), ("dtype", _c_i32), ("width", _c_i32), ("height", _c_i32),
        ("nimg", _c_i32), ("channels", _c_i32),
        ("values", _vp),
        ("img_stride", _c_i64), ("cs", _c_i64), ("rs", _c_i64), ("ps", _c_i64),
        ("spacing", _vp),
        ("line_width_px", _c_d),
        ("line_color", _c_i32 * 4), ("background", _c_i32 * 4),
        ("colormap", _vp),
        ("ncolors", _c_i32),
        ("out", _vp),
        ("coverage", _vp),
        ("gradient_corners", _c_i32 * 16),
        ("adaptive_target_px", _c_d),
        ("texture", _vp),
        ("tex_w", _c_i32), ("tex_h", _c_i32),
    ]


# Every symbol include/mdc.h declares, with its ctypes signature.
SIGNATURES = {
    "mdc_last_error": (ctypes.c_char_p, []),
    "mdc_version": (ctypes.c_int, []),
    "mdc_num_sms": (ctypes.c_int, []),
    "mdc_mls_field": (ctypes.c_int, [ctypes.POINTER(MdcMlsArgs), _vp]),
    "mdc_mls_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(MdcMlsArgs)]),
    "mdc_snap_workspace_bytes": (ctypes.c_size_t, [_c_i32, _c_i32]),
    "mdc_mls_snap": (ctypes.c_int, [ctypes.POINTER(MdcMlsArgs), _vp, _vp, _c_d, _vp, _vp]),
    "mdc_layout_workspace_bytes": (ctypes.c_size_t, [_c_i64, _c_i32]),
    "mdc_layout_plan_create": (ctypes.c_int, [ctypes.POINTER(MdcLayoutArgs), ctypes.POINTER(_vp), _vp]),
    "mdc_layout_plan_destroy": (ctypes.c_int, [_vp]),
    "mdc_layout_steps": (ctypes.c_int, [_vp, _c_i32, _vp, _c_i32, _vp]),
    "mdc_mls_prepare_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32]),
    "mdc_mls_prepare": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, _vp, _vp, ctypes.c_int32, ctypes.c_int32,
                                       _vp, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "mdc_copy_2d_async": (ctypes.c_int, [_vp, ctypes.c_size_t, _vp, ctypes.c_size_t, ctypes.c_size_t,
                                         ctypes.c_size_t, _vp]),
    "mdc_layout_set_peers": (ctypes.c_int, [_vp, ctypes.c_int32, _vp, _vp]),
    "mdc_layout_step_parity": (ctypes.c_int, [_vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp]),
    "mdc_layout_reset_counter": (ctypes.c_int, [_vp, _vp]),
    "mdc_layout_set_gather": (ctypes.c_int, [_vp, _vp]),
    "mdc_layout_scatter": (ctypes.c_int, [_vp, _vp, _c_i64, _vp]),
    "mdc_ipc_alloc": (ctypes.c_int, [ctypes.c_size_t, _vp, _vp]),
    "mdc_ipc_open": (ctypes.c_int, [_vp, _vp]),
    "mdc_ipc_close": (ctypes.c_int, [_vp]),
    "mdc_ipc_free": (ctypes.c_int, [_vp]),
    "mdc_layout_clamp_factors": (ctypes.c_int, [ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, ctypes.c_double, _vp,
                                                _vp]),
    "mdc_layout_profile": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "mdc_layout_repulsion": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "mdc_layout_node_count": (_c_i64, [_vp]),
    "mdc_layout_kdtree": (ctypes.c_int, [_vp, _vp] + [_vp] * 10 + [_vp]),
    "mdc_pca_workspace_bytes": (ctypes.c_size_t, [_c_i64, _c_i32]),
    "mdc_pca": (ctypes.c_int, [_c_i64, _c_i32] + [_vp] * 7 + [_vp]),
    "mdc_render": (ctypes.c_int, [ctypes.POINTER(MdcRenderArgs), _vp]),
    "mdc_linear_workspace_bytes": (ctypes.c_size_t, [_c_i32, _c_i32]),
    "mdc_overlay_workspace_bytes": (ctypes.c_size_t, [_c_i64, _c_d]),
    "mdc_overlay_points": (ctypes.c_int, [_vp, _c_i32, _c_i32, _c_i64, _vp, _c_d, _vp, _vp, ctypes.c_size_t, _vp]),
    "mdc_linear_field": (ctypes.c_int, [ctypes.POINTER(MdcLinearArgs), _vp]),
    "mdc_mean_field": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp, _c_d, _vp, _vp]),
    "mdc_affine_field": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp, _c_d, _c_d, _vp, _vp]),
    "mdc_rigid_field": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp, _c_d, _vp, _vp]),
    "mdc_rigid_field_norm": (ctypes.c_int, [_c_i64, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp, _c_d, _vp, _vp, _vp]),
    "mdc_bh_forces": (ctypes.c_int, [_c_i64] + [_vp] * 11 + [_c_d, _c_d, _c_d, _vp, _vp]),
    "mdc_peak_ffma": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp]),
    "mdc_peak_dfma": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp]),
}

_LIB = None


class MdcError(RuntimeError):
    """A libmdc call returned a negative status."""


def load() -> ctypes.CDLL:
    """Load libmdc.so (built by ``__graft_entry__.build()`` / ``make``)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                "there is no CPU fallback"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def require_cuda() -> ctypes.CDLL:
    lib = load()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1408_0677_b200 needs a CUDA device (no CPU fallback)")
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().mdc_last_error().decode(errors="replace")
        raise MdcError(f"{what} failed ({rc}): {msg}")


def stream_ptr(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


class nvtx:
    """NVTX range around a host-side stage (SURVEY.md §5 tracing): shows up
    in nsys / ncu --nvtx timelines; a no-op where NVTX is unavailable."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        try:
            import torch

            torch.cuda.nvtx.range_push(self.name)
            self.pushed = True
        except Exception:
            self.pushed = False
        return self

    def __exit__(self, *exc):
        if self.pushed:
            import torch

            torch.cuda.nvtx.range_pop()
        return False
