"""Field-to-pixels mappings (contour lines, discrete bands, point overlay).

Mirror of the reference's ``render`` module (render.py:21-283) for the modes
on the hot path: ``contour``, ``discrete``,
``discrete+contour`` render on the GPU (``mdc_render``: np.gradient
gradients, line coverage, band shading, fp64 compositing, RGBA8), both for
drop-in ``CoordinateField`` callers and for whole ``compute_fields`` blocks
(``render_fields``).  Band indices also come fused out of the MLS epilogue.
The adaptive / gradient / texture modes and the legend are SURVEY.md §8f
row 2 (next).
"""

from __future__ import annotations

import ctypes
import io
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .field import CoordinateField

MODES = ("contour", "discrete", "discrete+contour", "adaptive", "gradient", "texture")
GPU_MODES = ("contour", "discrete", "discrete+contour")

DEFAULT_COLORMAP = [
    (255, 255, 217), (237, 248, 177), (199, 233, 180), (127, 205, 187),
    (65, 182, 196), (29, 145, 192), (34, 94, 168), (37, 52, 148),
    (8, 29, 88), (5, 15, 60), (2, 8, 40),
]
GRADIENT_CORNERS = [(56, 80, 200), (228, 110, 200), (90, 200, 225), (245, 245, 245)]


class RenderError(Exception):
    pass


def auto_spacing(values) -> float:
    """cli.py:24-42: contour interval from the 1/2/5 ladder giving 8-15
    levels over the value range (host helper feeding the band epilogue)."""
    values = np.asarray(values, dtype=float)
    lo, hi = float(values.min()), float(values.max())
    rng = hi - lo
    if rng <= 0:
        return 1.0
    k = int(np.ceil(np.log10(rng)))
    ladder = [m * 10.0**e for e in range(k, k - 6, -1) for m in (5.0, 2.0, 1.0)]
    best, best_dist = ladder[0], np.inf
    for s in ladder:
        count = int(rng / s)
        if 8 <= count <= 15:
            return s
        dist = (8 - count) if count < 8 else (count - 15)
        if dist < best_dist:
            best, best_dist = s, dist
    return best


@dataclass(frozen=True)
class RenderSpec:
    """render.py:37-59."""

    mode: str = "contour"
    spacing: float = 1.0
    line_width_px: float = 1.5
    colormap: list = field(default_factory=lambda: list(DEFAULT_COLORMAP))
    gradient_corners: list = field(default_factory=lambda: list(GRADIENT_CORNERS))
    texture: np.ndarray | None = None
    line_color: tuple = (40, 40, 40, 255)
    background: tuple = (255, 255, 255, 255)
    point_radius: float = 2.5
    point_color: tuple = (20, 20, 20, 255)
    adaptive_target_px: float = 24.0

    def __post_init__(self):
        if self.mode not in MODES:
            raise RenderError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.spacing <= 0:
            raise RenderError("spacing must be positive")
        if self.line_width_px <= 0:
            raise RenderError("line_width_px must be positive")
        if self.mode == "texture" and self.texture is None:
            raise RenderError("texture mode requires a texture image")


@dataclass
class RenderedImage:
    width: int
    height: int
    pixels: np.ndarray  # (h, w, 4) uint8

    def to_png_bytes(self) -> bytes:
        from PIL import Image

        buf = io.BytesIO()
        Image.fromarray(self.pixels, "RGBA").save(buf, format="PNG")
        return buf.getvalue()

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.to_png_bytes())


def _rgba(color) -> np.ndarray:
    c = list(color)
    if len(c) == 3:
        c.append(255)
    return np.array(c, dtype=float) / 255.0


def _flat(shape, color) -> np.ndarray:
    img = np.empty(shape + (4,), dtype=float)
    img[:] = _rgba(color)
    return img


def _over(base: np.ndarray, color, alpha: np.ndarray) -> np.ndarray:
    """render.py:91-97 source-over composite."""
    src = _rgba(color)
    a = np.clip(alpha, 0.0, 1.0)[..., None] * src[3]
    base[..., :3] = base[..., :3] * (1.0 - a) + src[:3] * a
    base[..., 3:] = base[..., 3:] * (1.0 - a) + a
    return base


def _to_image(img: np.ndarray) -> RenderedImage:
    px = np.clip(np.rint(img * 255.0), 0, 255).astype(np.uint8)
    return RenderedImage(width=px.shape[1], height=px.shape[0], pixels=px)


_MODE_CODE = {"contour": 0, "discrete": 1, "discrete+contour": 2}


def _cmap_tensor(colormap, device) -> torch.Tensor:
    return torch.as_tensor(np.array([_rgba(c) for c in colormap], dtype=np.float64)).to(device)


def render_planes(values: torch.Tensor, strides, nimg: int, channels: int, width: int, height: int,
                  spacing, spec: RenderSpec, want_coverage: bool = False):
    """GPU render of ``nimg`` images (mdc_render): RGBA8 (nimg, H, W, 4) and
    optionally the float coverage (nimg, H, W).  ``strides`` =
    (img_stride, channel_stride, row_stride, pixel_stride) in elements."""
    lib = _lib.require_cuda()
    if spec.mode not in _MODE_CODE:
        raise RenderError(f"mode {spec.mode!r} is not implemented on the GPU yet (SURVEY.md §8f); use {GPU_MODES}")
    dev = values.device
    sp = torch.as_tensor(np.broadcast_to(np.asarray(spacing, dtype=np.float64), (nimg,)).copy()).to(dev)
    out = torch.empty((nimg, height, width, 4), dtype=torch.uint8, device=dev)
    cov = torch.empty((nimg, height, width), dtype=torch.float32, device=dev) if want_coverage else None
    cmap = _cmap_tensor(spec.colormap, dev)
    a = _lib.MdcRenderArgs()
    a.mode = _MODE_CODE[spec.mode]
    a.dtype = _lib.MDC_F32 if values.dtype == torch.float32 else _lib.MDC_F64
    a.width, a.height, a.nimg, a.channels = width, height, nimg, channels
    a.values = _lib.ptr(values)
    a.img_stride, a.cs, a.rs, a.ps = (int(v) for v in strides)
    a.spacing = _lib.ptr(sp)
    a.line_width_px = float(spec.line_width_px)
    lc = list(spec.line_color) + [255] * (4 - len(spec.line_color))
    bg = list(spec.background) + [255] * (4 - len(spec.background))
    for k in range(4):
        a.line_color[k] = int(lc[k])
        a.background[k] = int(bg[k])
    a.colormap, a.ncolors = _lib.ptr(cmap), len(spec.colormap)
    a.out = _lib.ptr(out)
    a.coverage = _lib.ptr(cov)
    _lib.check(lib.mdc_render(ctypes.byref(a), _lib.stream_ptr()), "mdc_render")
    return out, cov


def _field_planes(fld: CoordinateField):
    coords = torch.as_tensor(np.ascontiguousarray(fld.coords, dtype=np.float64)).cuda()
    w, h = fld.width, fld.height
    return coords, (0, 1, 2 * w, 2)


def render_fields(block, spacing, spec: RenderSpec):
    """Per-channel isocontour images of a ``compute_fields`` FieldBlock that
    covers the full frame: (d, H, W, 4) uint8 CUDA tensor."""
    vals = block.values
    d, rows, w = vals.shape
    if block.row0 != 0 or rows != block.transform.height:
        raise RenderError("render_fields needs a full-frame FieldBlock (np.gradient spans rows)")
    out, _ = render_planes(vals, (rows * w, 0, w, 1), d, 1, w, rows, spacing, spec)
    return out


def _gradient_magnitudes(fld: CoordinateField) -> np.ndarray:
    jac = fld.jacobian()
    return np.hypot(jac[..., 0], jac[..., 1])


def line_coverage(fld: CoordinateField, spacing: float, line_width_px: float) -> np.ndarray:
    """render.py:116-126, on the GPU (float32 coverage, fp64 arithmetic)."""
    coords, strides = _field_planes(fld)
    spec = RenderSpec(mode="contour", spacing=spacing, line_width_px=line_width_px)
    _, cov = render_planes(coords, strides, 1, fld.active_channels, fld.width, fld.height, spacing, spec,
                           want_coverage=True)
    return cov[0].double().cpu().numpy()


def band_indices(fld: CoordinateField, spacing: float) -> np.ndarray:
    """render.py:135-139 `_band_indices`."""
    bands = np.floor(fld.coords[..., 0] / spacing).astype(np.int64)
    if fld.active_channels == 2:
        bands = bands + np.floor(fld.coords[..., 1] / spacing).astype(np.int64)
    return bands


_band_indices = band_indices


def _render_gpu(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    coords, strides = _field_planes(fld)
    out, _ = render_planes(coords, strides, 1, fld.active_channels, fld.width, fld.height, spec.spacing, spec)
    px = out[0].cpu().numpy()
    return RenderedImage(width=px.shape[1], height=px.shape[0], pixels=px)


def render_contours(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:129-132 on the GPU."""
    return _render_gpu(fld, RenderSpec(**{**spec.__dict__, "mode": "contour"}))


def render_discrete(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:142-148 on the GPU."""
    mode = spec.mode if spec.mode in ("discrete", "discrete+contour") else "discrete"
    return _render_gpu(fld, RenderSpec(**{**spec.__dict__, "mode": mode}))


def render(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:272-283 for the GPU modes."""
    if spec.mode in _MODE_CODE:
        return _render_gpu(fld, spec)
    raise RenderError(f"mode {spec.mode!r} is not implemented yet (SURVEY.md §8f); use {GPU_MODES}")


def overlay_points(img: RenderedImage, positions, transform, spec: RenderSpec) -> RenderedImage:
    """render.py:237-257 anti-aliased discs at the projected points."""
    base = img.pixels.astype(float) / 255.0
    h, w = base.shape[:2]
    r = spec.point_radius
    pix = transform.to_pixels(np.asarray(positions, dtype=float).reshape(-1, 2))
    for px, py in pix:
        if not (-r - 1 <= px <= w + r and -r - 1 <= py <= h + r):
            continue
        c0 = max(0, int(np.floor(px - r - 1)))
        c1 = min(w - 1, int(np.ceil(px + r + 1)))
        r0 = max(0, int(np.floor(py - r - 1)))
        r1 = min(h - 1, int(np.ceil(py + r + 1)))
        if c0 > c1 or r0 > r1:
            continue
        yy, xx = np.mgrid[r0: r1 + 1, c0: c1 + 1]
        cov = np.clip(r + 0.5 - np.hypot(xx - px, yy - py), 0.0, 1.0)
        _over(base[r0: r1 + 1, c0: c1 + 1], spec.point_color, cov)
    return _to_image(base)
