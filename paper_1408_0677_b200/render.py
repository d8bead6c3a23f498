"""Field-to-pixels mappings (contour lines, discrete bands, point overlay).

Mirror of the reference's ``render`` module (render.py:21-283) for the modes
on the hot path: ``contour``, ``discrete``,
``discrete+contour``.  Band indices for fields produced by
``compute_fields(..., band_spacing=...)`` come fused out of the MLS kernel's
epilogue; this module computes them (and the anti-aliased contour coverage)
from a ``CoordinateField`` for drop-in callers.  The adaptive / gradient /
texture modes and the legend are SURVEY.md §8f row 2 (next).
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field

import numpy as np

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


def _gradient_magnitudes(fld: CoordinateField) -> np.ndarray:
    jac = fld.jacobian()
    return np.hypot(jac[..., 0], jac[..., 1])


def line_coverage(fld: CoordinateField, spacing: float, line_width_px: float) -> np.ndarray:
    """render.py:116-126."""
    grads = _gradient_magnitudes(fld)
    cov = np.zeros(fld.coords.shape[:2])
    for ch in range(fld.active_channels):
        vals = fld.coords[..., ch]
        dist = np.abs(vals - spacing * np.round(vals / spacing))
        g = grads[..., ch]
        px = np.where(g > 1e-30, dist / np.where(g > 1e-30, g, 1.0), np.inf)
        cov = np.maximum(cov, np.clip(0.5 * line_width_px + 0.5 - px, 0.0, 1.0))
    return cov


def band_indices(fld: CoordinateField, spacing: float) -> np.ndarray:
    """render.py:135-139 `_band_indices`."""
    bands = np.floor(fld.coords[..., 0] / spacing).astype(np.int64)
    if fld.active_channels == 2:
        bands = bands + np.floor(fld.coords[..., 1] / spacing).astype(np.int64)
    return bands


_band_indices = band_indices


def render_contours(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    img = _flat(fld.coords.shape[:2], spec.background)
    _over(img, spec.line_color, line_coverage(fld, spec.spacing, spec.line_width_px))
    return _to_image(img)


def render_discrete(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    table = np.array([_rgba(c) for c in spec.colormap])
    img = table[np.mod(band_indices(fld, spec.spacing), len(table))]
    if spec.mode == "discrete+contour":
        _over(img, spec.line_color, line_coverage(fld, spec.spacing, spec.line_width_px))
    return _to_image(img)


def render(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    if spec.mode == "contour":
        return render_contours(fld, spec)
    if spec.mode in ("discrete", "discrete+contour"):
        return render_discrete(fld, spec)
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
