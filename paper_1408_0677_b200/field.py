"""Per-pixel moving-least-squares field on the GPU.

Drop-in mirror of the reference's ``field`` module
(/root/reference/pkg/src/mdcontour/field.py): same dataclasses, defaults,
validation and exceptions; ``compute_field`` keeps its signature and numpy
return type (fp64 by default, matching the reference's arithmetic to the
1e-10 normwise contract).  ``compute_fields`` is the fused entry the
north-star metric is measured on: d target channels in one launch, fp32 or
fp64, optional row band (multi-GPU sharding) and fused band epilogue, torch
CUDA tensors in and out.

All arithmetic runs in libmdc (``mdc_mls_field`` + ``mdc_mls_snap``); only
the O(N) centring / viewport set-up stays on the host, computed with the same
numpy expressions as field.py:596-613 so the pixel grid is bit-identical.
"""

from __future__ import annotations

import ctypes
import struct
import threading
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from .dataset import Dataset
from .projection import expand_bounds

VARIANTS = ("linear", "mean", "affine", "rigid")
DEFAULT_ALPHA = {"linear": 1.0, "mean": 1.0, "affine": 1.5, "rigid": 1.0}
ALPHA_RANGE = (0.25, 3.0)


class FieldError(Exception):
    pass


class DegenerateRotation(FieldError):
    """Rigid solve collapsed (zero rotation estimate) at the sample point."""


@dataclass(frozen=True)
class MlsParams:
    """field.py:52-72."""

    variant: str = "affine"
    alpha: float | None = None
    epsilon_dist: float | None = None
    reg_eps: float = 1e-12

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}, got {self.variant!r}")
        a = self.resolved_alpha
        if not 0.1 < a <= 4.0:
            raise ValueError(f"alpha must be in (0.1, 4.0], got {a}")
        if self.reg_eps <= 0:
            raise ValueError("reg_eps must be positive")
        if self.epsilon_dist is not None and self.epsilon_dist <= 0:
            raise ValueError("epsilon_dist must be positive")

    @property
    def resolved_alpha(self) -> float:
        return DEFAULT_ALPHA[self.variant] if self.alpha is None else self.alpha


@dataclass(frozen=True)
class TargetAssignment:
    """field.py:75-89."""

    targets: np.ndarray
    mode: str
    dims: tuple[str, ...] = ()

    def __post_init__(self):
        if not np.all(np.isfinite(self.targets)):
            raise FieldError("target coordinates must be finite")

    @property
    def active_channels(self) -> int:
        return 1 if self.mode == "dims" and len(self.dims) == 1 else 2


def projection_targets(mesh) -> TargetAssignment:
    return TargetAssignment(targets=mesh.original_pos.copy(), mode="projection")


def dimension_targets(ds: Dataset, dim_a: str, dim_b: str | None = None) -> TargetAssignment:
    """field.py:96-105."""
    a = ds.raw_column(dim_a)
    if dim_b is None:
        return TargetAssignment(targets=np.column_stack([a, np.zeros_like(a)]), mode="dims", dims=(dim_a,))
    b = ds.raw_column(dim_b)
    return TargetAssignment(targets=np.column_stack([a, b]), mode="dims", dims=(dim_a, dim_b))


@dataclass(frozen=True)
class ViewportTransform:
    """field.py:108-142."""

    x0: float
    y0: float
    x1: float
    y1: float
    width: int
    height: int

    @property
    def units_per_px(self) -> tuple[float, float]:
        return ((self.x1 - self.x0) / self.width, (self.y1 - self.y0) / self.height)

    def pixel_center_grids(self) -> tuple[np.ndarray, np.ndarray]:
        sx, sy = self.units_per_px
        xs = self.x0 + (np.arange(self.width) + 0.5) * sx
        ys = self.y1 - (np.arange(self.height) + 0.5) * sy
        return np.meshgrid(xs, ys)

    def to_pixels(self, points: np.ndarray) -> np.ndarray:
        sx, sy = self.units_per_px
        px = (points[:, 0] - self.x0) / sx - 0.5
        py = (self.y1 - points[:, 1]) / sy - 0.5
        return np.column_stack([px, py])

    @classmethod
    def fit(cls, points: np.ndarray, width: int, height: int) -> "ViewportTransform":
        x0, y0, x1, y1 = expand_bounds(points)
        return cls(x0, y0, x1, y1, width, height)


@dataclass
class CoordinateField:
    """field.py:145-161."""

    width: int
    height: int
    coords: np.ndarray
    source_positions: np.ndarray
    transform: ViewportTransform
    active_channels: int = 2
    # GPU-resident copy of ``coords`` ((H, W, 2) fp64 CUDA tensor, same
    # values) kept by compute_field so render / service caches skip the
    # re-upload; not part of the reference's dataclass identity.
    device_coords: object = dc_field(default=None, repr=False, compare=False)

    def jacobian(self) -> np.ndarray:
        dy, dx = np.gradient(self.coords, axis=(0, 1))
        out = np.empty(self.coords.shape[:2] + (2, 2))
        out[..., 0] = dx
        out[..., 1] = dy
        return out


def field_gradient(fld: CoordinateField, x: int, y: int) -> np.ndarray:
    """field.py:164-185."""
    c = fld.coords

    def diff(axis: int, idx: int, limit: int):
        if 0 < idx < limit - 1:
            lo, hi, scale = idx - 1, idx + 1, 0.5
        else:
            lo, hi, scale = max(idx - 1, 0), min(idx + 1, limit - 1), 1.0
        if axis == 0:
            return scale * (c[y, hi] - c[y, lo])
        return scale * (c[hi, x] - c[lo, x])

    out = np.empty((2, 2))
    out[:, 0] = diff(0, x, fld.width)
    out[:, 1] = diff(1, y, fld.height)
    return out


# ---------------------------------------------------------------------------
# GPU evaluation


# Sentinel-filled scratch, one per (device, stream): the last kernel of a
# call restores the sentinel, so calls on one stream can share it as long as
# their launch sequences do not interleave -- each call enqueues under the
# scratch's lock (several Python threads may share a stream; ctypes releases
# the GIL during the launches).  Calls on different streams use different
# scratch and never race.
_SNAP_WS: dict[tuple[int, int], torch.Tensor] = {}
_LIN_WS: dict[tuple[int, int], torch.Tensor] = {}
_WS_LOCKS: dict[tuple[str, int, int], threading.Lock] = {}
_WS_LOCKS_GUARD = threading.Lock()


def _ws_key(device: torch.device) -> tuple[int, int]:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    return idx, int(torch.cuda.current_stream(idx).cuda_stream)


def _ws_lock(kind: str, device: torch.device) -> threading.Lock:
    key = (kind, *_ws_key(device))
    with _WS_LOCKS_GUARD:
        lk = _WS_LOCKS.get(key)
        if lk is None:
            lk = _WS_LOCKS[key] = threading.Lock()
    return lk


class AtControlPoint:
    """field.py:42-49: sentinel for samples inside a control's snap radius."""

    def __repr__(self):
        return "AtControlPoint"


AT_CONTROL_POINT = AtControlPoint()


def mls_weight(v, pi, alpha: float, epsilon_dist: float = 1e-18):
    """field.py:188-194: |pi - v|^(-2 alpha), or the sentinel inside the snap radius."""
    d = np.asarray(pi, dtype=float) - np.asarray(v, dtype=float)
    d2 = float(d @ d)
    return AT_CONTROL_POINT if d2 < epsilon_dist else d2 ** (-alpha)


def _point_mls(kind: str, v, controls_p, controls_q, params: MlsParams) -> np.ndarray:
    """Single-point MLS (field.py:208-269) evaluated by the GPU seam kernel
    (mdc_{mean,affine,rigid}_field on one sample); the snap rule first."""
    lib = _lib.require_cuda()
    v = np.asarray(v, dtype=np.float64).reshape(2)
    p = np.asarray(controls_p, dtype=np.float64).reshape(-1, 2)
    q = np.asarray(controls_q, dtype=np.float64).reshape(-1, 2)
    eps = params.epsilon_dist if params.epsilon_dist is not None else 1e-18
    d2 = ((p - v) ** 2).sum(axis=1)
    hit = int(np.argmin(d2))
    if d2[hit] < eps:
        return q[hit].copy()
    dev = torch.device("cuda", torch.cuda.current_device())
    qq = q - p if kind == "mean" else q  # the mean kernel takes dq = q - p (_kernels.py:52-67)
    t = [torch.as_tensor(np.ascontiguousarray(a)).to(dev)
         for a in (v[:1], v[1:], p[:, 0], p[:, 1], qq[:, 0], qq[:, 1])]
    out = torch.empty((1, 2), dtype=torch.float64, device=dev)
    args = [1, *(_lib.ptr(x) for x in t[:2]), len(p), *(_lib.ptr(x) for x in t[2:]), params.resolved_alpha]
    if kind == "affine":
        args.append(params.reg_eps)
    if kind == "rigid":
        norm = torch.empty(1, dtype=torch.float64, device=dev)
        _lib.check(lib.mdc_rigid_field_norm(*args, _lib.ptr(out), _lib.ptr(norm), _lib.stream_ptr()),
                   "mdc_rigid_field_norm")
        if float(norm[0]) < 1e-12:  # field.py:263-265
            raise DegenerateRotation("rigid MLS rotation estimate vanished")
        return out[0].cpu().numpy()
    fn = {"mean": lib.mdc_mean_field, "affine": lib.mdc_affine_field}[kind]
    _lib.check(fn(*args, _lib.ptr(out), _lib.stream_ptr()), f"mdc_{kind}_field")
    return out[0].cpu().numpy()


def mean_mls(v, controls_p, controls_q, params: MlsParams) -> np.ndarray:
    """field.py:208-218: v + weighted mean of (q - p), on the GPU."""
    return _point_mls("mean", v, controls_p, controls_q, params)


def affine_mls(v, controls_p, controls_q, params: MlsParams) -> np.ndarray:
    """field.py:221-240: the weighted affine map through the controls at v, on the GPU."""
    return _point_mls("affine", v, controls_p, controls_q, params)


def rigid_mls(v, controls_p, controls_q, params: MlsParams) -> np.ndarray:
    """field.py:243-269: the weighted rigid map at v, on the GPU.  Where the
    rotation estimate vanishes (|f| < 1e-12) it raises DegenerateRotation
    like the reference's scalar evaluator (field.py:263-265); only the
    per-pixel field path takes _kernels.rigid_field's mean fallback."""
    return _point_mls("rigid", v, controls_p, controls_q, params)


def triangle_neighbors(tris: np.ndarray) -> np.ndarray:
    """field.py:415-428: neighbour triangle across the edge opposite each
    vertex (-1 on the hull)."""
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    t = len(tris)
    edges = np.stack([tris[:, [1, 2]], tris[:, [2, 0]], tris[:, [0, 1]]], axis=1).reshape(-1, 2)
    edges.sort(axis=1)
    slot = np.arange(3 * t)
    order = np.lexsort((slot, edges[:, 1], edges[:, 0]))
    e = edges[order]
    same = np.all(e[1:] == e[:-1], axis=1)
    nbrs = np.full(3 * t, -1, dtype=np.int64)
    a, b = order[:-1][same], order[1:][same]
    nbrs[a] = b // 3
    nbrs[b] = a // 3
    return nbrs.reshape(t, 3)


def hull_edges(tris: np.ndarray) -> np.ndarray:
    """field.py:440-447 `_hull_edges`, vectorised: (u, v, triangle) per
    boundary edge, u < v, in first-appearance order over triangles' edges
    (a, b), (b, c), (c, a)."""
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    e = np.stack([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [2, 0]]], axis=1).reshape(-1, 2)
    key = np.sort(e, axis=1)
    uniq, first, counts = np.unique(key, axis=0, return_index=True, return_counts=True)
    keep = counts == 1
    order = np.argsort(first[keep], kind="stable")
    sel = uniq[keep][order]
    tri = first[keep][order] // 3
    return np.column_stack([sel, tri]).astype(np.int64)


def _linear_workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    key = _ws_key(device)
    ws = _LIN_WS.get(key)
    if ws is None or ws.numel() * 4 < nbytes:
        ws = torch.full((max(nbytes // 4, 1),), 2**31 - 1, dtype=torch.int32, device=device)
        _LIN_WS[key] = ws
    return ws


def linear_device(positions, tvals, triangles, width, height, row_range=None, dtype="f64", out=None,
                  strides=None):
    """The 'linear' variant (field.py:497-515) on the GPU (mdc_linear_field).
    Returns the output tensor ((nch, rows, W) unless ``out``/``strides``)."""
    lib = _lib.require_cuda()
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    tv = np.ascontiguousarray(tvals, dtype=np.float64)
    if tv.ndim == 1:
        tv = tv[:, None]
    tris = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
    hull = hull_edges(tris)
    tr = ViewportTransform.fit(pos, width, height)
    sx, sy = tr.units_per_px
    r0, r1 = (0, height) if row_range is None else (int(row_range[0]), int(row_range[1]))
    dev = torch.device("cuda", torch.cuda.current_device())
    dcode = _resolve_dtype(dtype)
    nch = tv.shape[1]
    if out is None:
        out = torch.empty((nch, r1 - r0, width), dtype=torch.float32 if dcode == _lib.MDC_F32 else torch.float64,
                          device=dev)
        strides = ((r1 - r0) * width, width, 1)
    t_pos, t_tv = _h2d(pos, dev), _h2d(tv, dev)
    t_tris, t_hull = _h2d(tris.astype(np.int32), dev), _h2d(hull.astype(np.int32), dev)
    a = _lib.MdcLinearArgs()
    a.width, a.height, a.row0, a.row1 = width, height, r0, r1
    a.x0, a.y1, a.sx, a.sy = tr.x0, tr.y1, sx, sy
    a.n, a.ntri, a.nch, a.dtype = len(pos), len(tris), nch, dcode
    a.pos, a.tvals, a.tris, a.hull = _lib.ptr(t_pos), _lib.ptr(t_tv), _lib.ptr(t_tris), _lib.ptr(t_hull)
    a.nhull = len(hull)
    a.out = _lib.ptr(out)
    a.out_cs, a.out_rs, a.out_ps = (int(v) for v in strides)
    with _ws_lock("linear", dev):
        ws = _linear_workspace(int(lib.mdc_linear_workspace_bytes(width, r1 - r0)), dev)
        a.workspace = _lib.ptr(ws)
        _lib.check(lib.mdc_linear_field(ctypes.byref(a), _lib.stream_ptr()), "mdc_linear_field")
    return out, tr


def _snap_workspace(nbytes: int, device: torch.device) -> torch.Tensor:
    """Per-(device, stream) scratch for mdc_mls_snap, kept all-0xFF between calls."""
    key = _ws_key(device)
    ws = _SNAP_WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.full((max(nbytes, 1),), 255, dtype=torch.uint8, device=device)
        _SNAP_WS[key] = ws
    return ws


def _ldq(d: int, dtype: int, variant: int) -> int:
    """Padded target row stride libmdc's stager needs (mirrors mls.cu)."""
    es = 4 if dtype == _lib.MDC_F32 else 8
    if variant == _lib.MDC_RIGID:
        chunk = 2
    else:
        cap = 32 if dtype == _lib.MDC_F32 else 16
        chunk = 1
        while chunk < d and chunk < cap:
            chunk *= 2
    ld = -(-d // chunk) * chunk
    vec = 16 // es
    return -(-ld // vec) * vec


@dataclass
class FieldBlock:
    """Result of ``compute_fields``: device tensors for rows [row0, row1)."""

    values: torch.Tensor            # (d, rows, W) float32/float64
    bands: torch.Tensor | None      # (d, rows, W) int32
    transform: ViewportTransform
    row0: int
    row1: int
    nonfinite: torch.Tensor         # () int32 device counter
    h2d_bytes: int = 0              # host->device bytes this call uploaded
    rgba: torch.Tensor | None = None  # (d, rows, W, 4) uint8: discrete band shading per channel

    def check_finite(self) -> None:
        if int(self.nonfinite.item()) != 0:
            raise FieldError("field evaluation produced non-finite coordinates")


def _to_device(t: torch.Tensor, device: torch.device) -> torch.Tensor:
    """CPU tensor -> device (async when the caller's tensor is pinned)."""
    if t.is_cuda:
        return t.to(device)
    return t.to(device, non_blocking=t.is_pinned())


def _h2d(arr: np.ndarray, device: torch.device) -> torch.Tensor:
    """Host -> device through a pinned staging buffer (async on the current stream)."""
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.pin_memory().to(device, non_blocking=True)


def _resolve_dtype(dtype) -> int:
    if dtype in ("f32", "float32", torch.float32, np.float32):
        return _lib.MDC_F32
    if dtype in ("f64", "float64", torch.float64, np.float64):
        return _lib.MDC_F64
    raise ValueError(f"dtype must be f32 or f64, got {dtype!r}")


class MlsProblem:
    """Host-side set-up of one MLS evaluation (field.py:596-613), reusable
    across row bands / repeated frames.  Controls live on the device."""

    def __init__(self, positions, targets, variant: str, width: int, height: int,
                 alpha=None, reg_eps=1e-12, epsilon_dist=None, dtype="f32", axis=None,
                 device=None, tensor_cores: bool = True):
        lib = _lib.require_cuda()
        self.lib = lib
        if variant not in ("mean", "affine", "rigid"):
            raise ValueError(f"GPU MLS variant must be mean, affine or rigid, got {variant!r}")
        # inputs may be numpy arrays or (ideally pinned) CPU torch tensors
        pos_t0 = positions if torch.is_tensor(positions) else torch.from_numpy(
            np.ascontiguousarray(positions, dtype=np.float64))
        tv_t0 = targets if torch.is_tensor(targets) else torch.from_numpy(
            np.ascontiguousarray(targets, dtype=np.float64))
        pos_t0 = pos_t0.to(torch.float64).contiguous()
        tv_t0 = tv_t0.to(torch.float64).contiguous()
        if tv_t0.ndim == 1:
            tv_t0 = tv_t0[:, None]
        n, d = tv_t0.shape
        if n == 0 or d == 0:
            raise FieldError("MLS needs at least one control point and one target channel")
        if pos_t0.ndim != 2 or pos_t0.shape[1] != 2:
            raise ValueError(f"positions must be (n, 2), got {tuple(pos_t0.shape)}")
        if pos_t0.shape[0] != n:
            raise ValueError("positions and targets disagree on the control count")
        if variant == "rigid" and d != 2:
            raise FieldError("rigid MLS needs exactly two target channels")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.variant = variant
        self.vcode = _lib.VARIANT_CODE[variant]
        self.dcode = _resolve_dtype(dtype)
        self.tdtype = torch.float32 if self.dcode == _lib.MDC_F32 else torch.float64
        self.width, self.height, self.n, self.d = int(width), int(height), n, d
        self.alpha = DEFAULT_ALPHA[variant] if alpha is None else float(alpha)
        self.reg_eps = float(reg_eps)
        pos_np = pos_t0.numpy() if not pos_t0.is_cuda else pos_t0.cpu().numpy()
        self.transform = ViewportTransform.fit(pos_np, width, height)
        sx, sy = self.transform.units_per_px
        self.eps = epsilon_dist if epsilon_dist is not None else (0.25 * max(sx, sy)) ** 2
        dev = self.device
        # raw inputs to the device once; centring + dtype/padding on the device
        # (mdc_mls_prepare: field.py:607-613, deterministic means)
        self.pos_t = _to_device(pos_t0, dev)
        self.tvals_t = _to_device(tv_t0, dev)
        if variant == "mean":
            ax = np.zeros(d, dtype=np.int32) if axis is None else np.asarray(axis, dtype=np.int32)
        else:
            ax = np.zeros(d, dtype=np.int32)
        self.axis_t = _to_device(torch.from_numpy(np.ascontiguousarray(ax)), dev)
        ldq = _ldq(d, self.dcode, self.vcode)
        self.pc_t = torch.empty((n, 2), dtype=torch.float64, device=dev)
        self.q_t = torch.empty((n, ldq), dtype=self.tdtype, device=dev)
        pm_t = torch.empty(2, dtype=torch.float64, device=dev)
        self.qm_t = torch.empty(d, dtype=torch.float64, device=dev)
        wsb = int(lib.mdc_mls_prepare_workspace_bytes(d))
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        with _lib.nvtx("mls.prepare"):
            _lib.check(lib.mdc_mls_prepare(n, d, _lib.ptr(self.pos_t), _lib.ptr(self.tvals_t), self.vcode,
                                           self.dcode, _lib.ptr(self.axis_t), ldq, _lib.ptr(self.pc_t),
                                           _lib.ptr(self.q_t), _lib.ptr(pm_t), _lib.ptr(self.qm_t), _lib.ptr(ws), wsb,
                                           _lib.stream_ptr()), "mdc_mls_prepare")
        self.pm_t = pm_t  # the kernels read the frame centre on the device (no host round trip)
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in (self.pos_t, self.tvals_t, self.axis_t))
        self.ldq = ldq
        self.flags = 0 if tensor_cores else _lib.MDC_FLAG_NO_TC
        self._ws = None

    def args(self, out, out_strides, row0, row1, bands=None, band_strides=(0, 0), spacing=None,
             nonfinite=None, rgba=None, palette=None) -> _lib.MdcMlsArgs:
        t = self.transform
        sx, sy = t.units_per_px
        a = _lib.MdcMlsArgs()
        a.variant, a.dtype = self.vcode, self.dcode
        a.width, a.height, a.row0, a.row1 = self.width, self.height, int(row0), int(row1)
        a.n, a.d, a.ldq = self.n, self.d, self.ldq
        a.x0, a.y1, a.sx, a.sy = t.x0, t.y1, sx, sy
        a.pmx = a.pmy = 0.0
        a.pm = _lib.ptr(self.pm_t)
        a.alpha, a.reg_eps = self.alpha, self.reg_eps
        a.pc, a.q, a.qm, a.axis = _lib.ptr(self.pc_t), _lib.ptr(self.q_t), _lib.ptr(self.qm_t), _lib.ptr(self.axis_t)
        a.out = _lib.ptr(out)
        a.out_cs, a.out_rs, a.out_ps = (int(s) for s in out_strides)
        a.bands = _lib.ptr(bands)
        a.band_cs, a.band_rs = (int(s) for s in band_strides)
        a.spacing = _lib.ptr(spacing)
        a.nonfinite = _lib.ptr(nonfinite)
        a.rgba = _lib.ptr(rgba)
        a.palette = _lib.ptr(palette)
        a.palette_n = 0 if palette is None else int(palette.numel())
        a.flags = self.flags
        need = int(self.lib.mdc_mls_workspace_bytes(ctypes.byref(a)))
        if need:
            if self._ws is None or self._ws.numel() < need:
                self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            a.workspace, a.workspace_bytes = _lib.ptr(self._ws), self._ws.numel()
        return a

    def run(self, a: _lib.MdcMlsArgs, snap: bool = True) -> None:
        stream = _lib.stream_ptr()
        with _lib.nvtx(f"mls.field rows {a.row0}-{a.row1}"):
            _lib.check(self.lib.mdc_mls_field(ctypes.byref(a), stream), "mdc_mls_field")
        if snap:
            rows = a.row1 - a.row0
            with _lib.nvtx("mls.snap"), _ws_lock("snap", self.device):
                ws = _snap_workspace(int(self.lib.mdc_snap_workspace_bytes(self.width, rows)), self.device)
                _lib.check(self.lib.mdc_mls_snap(ctypes.byref(a), _lib.ptr(self.pos_t), _lib.ptr(self.tvals_t),
                                                 ctypes.c_double(self.eps), _lib.ptr(ws), stream),
                           "mdc_mls_snap")


_PALETTES: dict = {}
_COPY_STREAMS: dict = {}
_CACHE_GUARD = threading.Lock()


def _palette_device(colormap, dev: torch.device) -> torch.Tensor:
    """The packed palette on ``dev``, uploaded once per (colormap, device)."""
    key = (tuple(tuple(c) for c in colormap), dev.index if dev.index is not None else torch.cuda.current_device())
    with _CACHE_GUARD:
        t = _PALETTES.get(key)
    if t is None:
        t = _h2d(palette_rgba8(colormap).view(np.int32), dev)
        with _CACHE_GUARD:
            t = _PALETTES.setdefault(key, t)
    return t


def _copy_stream(dev: torch.device) -> torch.cuda.Stream:
    """One side stream per (device, thread) for the band D2H copies (creating
    a stream per call costs tens of microseconds on small frames)."""
    key = (dev.index if dev.index is not None else torch.cuda.current_device(), threading.get_ident())
    with _CACHE_GUARD:
        st = _COPY_STREAMS.get(key)
        if st is None:
            st = _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
    return st


def palette_rgba8(colormap) -> np.ndarray:
    """render.py:142-148's colour table as packed RGBA8 words (the bytes
    render_discrete writes: clip(rint(255 * rgba)))."""
    from .render import _rgba

    tab = np.array([_rgba(c) for c in colormap], dtype=np.float64)
    px = np.clip(np.rint(tab * 255.0), 0, 255).astype(np.uint8)
    return px.reshape(-1, 4).copy().view(np.uint32).reshape(-1)


def compute_fields(positions, targets, params: MlsParams, width: int, height: int,
                   row_range=None, dtype="f32", band_spacing=None, axis=None,
                   problem: MlsProblem | None = None, tensor_cores: bool = True, colormap=None) -> FieldBlock:
    """Fused d-channel MLS: every column of ``targets`` (n, d) is one field.

    Channel k equals channel 0 of the reference's ``compute_field`` for the
    single-dimension target (targets[:, k], 0) -- exactly what the reference
    CLI renders once per dimension (cli.py:143-165) -- for mean and affine;
    rigid takes d == 2 and matches the reference's two channels.
    ``band_spacing`` (scalar or (d,)) fuses render._band_indices; with
    ``colormap`` (a list of colours, e.g. render.DEFAULT_COLORMAP) the same
    epilogue also writes each channel's discrete band shading as RGBA8
    (render.py:142-148 for that channel's single-dimension field).
    Returns a FieldBlock of device tensors (rows [row0, row1) only).
    """
    if params.variant == "linear":
        raise FieldError("compute_fields(variant='linear') needs the mesh: use linear_device")
    prob = problem or MlsProblem(positions, targets, params.variant, width, height,
                                 alpha=params.resolved_alpha, reg_eps=params.reg_eps,
                                 epsilon_dist=params.epsilon_dist, dtype=dtype, axis=axis,
                                 tensor_cores=tensor_cores)
    r0, r1 = (0, height) if row_range is None else (int(row_range[0]), int(row_range[1]))
    rows = r1 - r0
    dev = prob.device
    out = torch.empty((prob.d, rows, width), dtype=prob.tdtype, device=dev)
    bands = spacing_t = None
    if band_spacing is not None:
        sp = np.broadcast_to(np.asarray(band_spacing, dtype=np.float64), (prob.d,)).copy()
        spacing_t = _h2d(sp, dev)
        bands = torch.empty((prob.d, rows, width), dtype=torch.int32, device=dev)
    rgba = pal_t = None
    if colormap is not None:
        if spacing_t is None:
            raise ValueError("colormap shading needs band_spacing")
        pal_t = _palette_device(colormap, dev)
        rgba = torch.empty((prob.d, rows, width), dtype=torch.int32, device=dev)
    nonfinite = torch.zeros((), dtype=torch.int32, device=dev)
    a = prob.args(out, (rows * width, width, 1), r0, r1, bands, (rows * width, width), spacing_t, nonfinite,
                  rgba=rgba, palette=pal_t)
    prob.run(a)
    h2d = 0 if problem is not None else prob.h2d_bytes + (spacing_t.numel() * 8 if spacing_t is not None else 0)
    return FieldBlock(values=out, bands=bands, transform=prob.transform, row0=r0, row1=r1,
                      nonfinite=nonfinite, h2d_bytes=h2d,
                      rgba=None if rgba is None else rgba.view(torch.uint8).view(prob.d, rows, width, 4))


SMALL_FRAME_PIXELS = 1 << 20  # below this the band split's extra launches cost more than the copy it hides


def plan_row_bands(r0: int, r1: int, nbands: int = 4, width: int | None = None) -> list[tuple[int, int]]:
    """Row bands for ``compute_fields_to_host``: a large band, then a tail of
    ~rows / (2 nbands) rows whose compute hides the large band's device->host
    copy and whose own (exposed) copy is small.  Each band is one kernel
    launch with its own ramp-up/ramp-down (~1.2 ms at 4K, measured), so two
    bands beat many: 4K config 3 e2e 905 -> 893 ms/frame vs 7 whole-wave
    bands or 4 equal ones.  Frames under SMALL_FRAME_PIXELS (given ``width``)
    take one band: there the second band's launches cost more than the copy
    they would hide (config 1, 256x256)."""
    rows = r1 - r0
    if rows < 2 or (width is not None and rows * width < SMALL_FRAME_PIXELS):
        return [(r0, r1)]
    tail = max(1, rows // (2 * max(1, int(nbands))))
    return [(r0, r1 - tail), (r1 - tail, r1)]


def compute_fields_to_host(positions, targets, params: MlsParams, width: int, height: int,
                           out: torch.Tensor, bands_out: torch.Tensor | None = None, row_range=None,
                           dtype="f32", band_spacing=None, nbands: int = 4, tensor_cores: bool = True,
                           rgba_out: torch.Tensor | None = None, colormap=None) -> int:
    """``compute_fields`` with the result delivered into HOST memory: ``out``
    (d, rows, W) pinned float tensor (and optional int32 ``bands_out``, and
    with ``colormap`` the fused band shading into ``rgba_out``: (d, rows, W,
    4) uint8).

    The frame is evaluated in row bands (``plan_row_bands``); each band's
    device->host copy runs on a side stream while the next band computes (two
    device band buffers, event-ordered), so only the small last band's copy
    is exposed.  Bands
    are bit-identical to the whole-frame result (tile frames are global).
    Returns the host->device bytes uploaded.  Raises FieldError on
    non-finite output."""
    if params.variant == "linear":
        raise FieldError("compute_fields_to_host(variant='linear') is not supported; use linear_device")
    prob = MlsProblem(positions, targets, params.variant, width, height, alpha=params.resolved_alpha,
                      reg_eps=params.reg_eps, epsilon_dist=params.epsilon_dist, dtype=dtype,
                      tensor_cores=tensor_cores)
    r0, r1 = (0, height) if row_range is None else (int(row_range[0]), int(row_range[1]))
    rows = r1 - r0
    d = prob.d
    if tuple(out.shape) != (d, rows, width) or out.is_cuda or out.dtype != prob.tdtype or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous host {prob.tdtype} tensor of shape {(d, rows, width)}")
    if bands_out is not None and (tuple(bands_out.shape) != (d, rows, width) or bands_out.is_cuda
                                  or bands_out.dtype != torch.int32 or not bands_out.is_contiguous()):
        raise ValueError(f"bands_out must be a contiguous host int32 tensor of shape {(d, rows, width)}")
    if (rgba_out is None) != (colormap is None):
        raise ValueError("rgba_out and colormap go together")
    if rgba_out is not None and (tuple(rgba_out.shape) != (d, rows, width, 4) or rgba_out.is_cuda
                                 or rgba_out.dtype != torch.uint8 or not rgba_out.is_contiguous()):
        raise ValueError(f"rgba_out must be a contiguous host uint8 tensor of shape {(d, rows, width, 4)}")
    dev = prob.device
    plan = plan_row_bands(r0, r1, nbands, width)
    step = max(b1 - b0 for b0, b1 in plan)
    spacing_t = None
    if band_spacing is not None:
        sp = np.broadcast_to(np.asarray(band_spacing, dtype=np.float64), (d,)).copy()
        spacing_t = _h2d(sp, dev)
    if colormap is not None and spacing_t is None:
        raise ValueError("colormap shading needs band_spacing")
    pal_t = _palette_device(colormap, dev) if colormap is not None else None
    rgba_host = rgba_out.view(torch.int32).view(d, rows, width) if rgba_out is not None else None
    nonfinite = torch.zeros((), dtype=torch.int32, device=dev)
    vbuf = [torch.empty((d, step, width), dtype=prob.tdtype, device=dev) for _ in range(2)]
    bbuf = [torch.empty((d, step, width), dtype=torch.int32, device=dev) for _ in range(2)] \
        if bands_out is not None else [None, None]
    cbuf = [torch.empty((d, step, width), dtype=torch.int32, device=dev) for _ in range(2)] \
        if rgba_out is not None else [None, None]
    compute = torch.cuda.current_stream(dev)
    copy = _copy_stream(dev)
    done = [None, None]  # copy-finished events per buffer
    for i, (b0, b1) in enumerate(plan):
        n_rows = b1 - b0
        k = i & 1
        if done[k] is not None:
            compute.wait_event(done[k])
        v = vbuf[k][:, :n_rows]
        bt = bbuf[k][:, :n_rows] if bbuf[k] is not None else None
        ct = cbuf[k][:, :n_rows] if cbuf[k] is not None else None
        # the shading shares the band strides
        a = prob.args(v, (step * width, width, 1), b0, b1, bt, (step * width, width), spacing_t, nonfinite,
                      rgba=ct, palette=pal_t)
        prob.run(a)
        ready = torch.cuda.Event()
        ready.record(compute)
        copy.wait_event(ready)
        # one strided async copy per plane set: d rows of (n_rows x W) elements
        for src, dst in ((v, out), (bt, bands_out), (ct, rgba_host)):
            if src is None:
                continue
            es = src.element_size()
            _lib.check(prob.lib.mdc_copy_2d_async(
                ctypes.c_void_p(dst.data_ptr() + (b0 - r0) * width * es), rows * width * es,
                _lib.ptr(src), step * width * es, n_rows * width * es, d, ctypes.c_void_p(copy.cuda_stream)),
                "mdc_copy_2d_async")
        ev = torch.cuda.Event()
        ev.record(copy)
        done[k] = ev
        vbuf[k].record_stream(copy)
        for buf in (bbuf[k], cbuf[k]):
            if buf is not None:
                buf.record_stream(copy)
    copy.synchronize()
    if int(nonfinite.item()) != 0:
        raise FieldError("field evaluation produced non-finite coordinates")
    return prob.h2d_bytes + (spacing_t.numel() * 8 if spacing_t is not None else 0)


def compute_field(mesh, positions: np.ndarray, targets: TargetAssignment, params: MlsParams,
                  width: int, height: int, threads: int = 1, dtype="f64") -> CoordinateField:
    """field.py:582-659 on the GPU.  ``threads`` is accepted for signature
    compatibility (the GPU result does not depend on it); ``dtype`` selects
    the fp64 parity mode (default) or the fp32 throughput mode."""
    if params.variant == "rigid" and targets.active_channels == 1:
        raise FieldError("rigid MLS is degenerate for single-dimension targets; use mean or affine")
    positions = np.asarray(positions, dtype=np.float64)
    tvals = targets.targets.astype(float)
    if params.variant == "linear":
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        if dev is None:
            _lib.require_cuda()
        tdt = torch.float32 if _resolve_dtype(dtype) == _lib.MDC_F32 else torch.float64
        out = torch.empty((height, width, 2), dtype=tdt, device=dev)
        _, tr = linear_device(positions, tvals, mesh.triangles, width, height, dtype=dtype, out=out,
                              strides=(1, 2 * width, 2))
        dev64 = out if out.dtype == torch.float64 else out.double()
        coords = dev64.cpu().numpy()
        if not np.all(np.isfinite(coords)):
            raise FieldError("field evaluation produced non-finite coordinates")
        return CoordinateField(width=width, height=height, coords=coords,
                               source_positions=positions, transform=tr,
                               active_channels=targets.active_channels, device_coords=dev64)
    prob = MlsProblem(positions, tvals, params.variant, width, height, alpha=params.resolved_alpha,
                      reg_eps=params.reg_eps, epsilon_dist=params.epsilon_dist, dtype=dtype,
                      axis=[0, 1])
    out = torch.empty((height, width, 2), dtype=prob.tdtype, device=prob.device)
    nonfinite = torch.zeros((), dtype=torch.int32, device=prob.device)
    a = prob.args(out, (1, 2 * width, 2), 0, height, nonfinite=nonfinite)
    prob.run(a)
    dev64 = out if out.dtype == torch.float64 else out.double()
    coords = dev64.cpu().numpy()
    if int(nonfinite.item()) != 0 or not np.all(np.isfinite(coords)):
        raise FieldError("field evaluation produced non-finite coordinates")
    return CoordinateField(width=width, height=height, coords=coords,
                           source_positions=np.asarray(positions, dtype=float),
                           transform=prob.transform, active_channels=targets.active_channels,
                           device_coords=dev64)


MAGIC = b"MLSF"


def write_field(fld: CoordinateField, path) -> None:
    """field.py:665-670: magic, u32 width/height, row-major f64 (u, v) pairs."""
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<II", fld.width, fld.height))
        fh.write(fld.coords.astype("<f8").tobytes())


def read_field(path) -> tuple[int, int, np.ndarray]:
    """field.py:673-679."""
    with open(path, "rb") as fh:
        if fh.read(4) != MAGIC:
            raise FieldError(f"{path}: not a field raster")
        w, h = struct.unpack("<II", fh.read(8))
        data = np.frombuffer(fh.read(), dtype="<f8").reshape(h, w, 2)
    return w, h, data
