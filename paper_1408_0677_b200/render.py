"""Field-to-pixels mappings (contour lines, discrete bands, point overlay).

Mirror of the reference's ``render`` module (render.py:21-318).  Every
render mode -- contour, discrete, discrete+contour,
adaptive, gradient, texture (§8f row 2) -- runs on the GPU (``mdc_render``:
np.gradient gradients, line coverage, band shading, fp64 compositing,
RGBA8), for drop-in ``CoordinateField`` callers and whole ``compute_fields``
blocks (``render_fields``); the point overlay too (``mdc_overlay_points``).
Band indices also come fused out of the MLS epilogue.  The legend strip
(text via PIL) stays on the host.
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
GPU_MODES = MODES

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


_MODE_CODE = {"contour": 0, "discrete": 1, "discrete+contour": 2, "adaptive": 3, "gradient": 4, "texture": 5}


def _texture_rgba(tex) -> np.ndarray:
    """render.py:224-229 texture normalisation to RGBA8."""
    tex = np.asarray(tex)
    if tex.ndim == 2:
        tex = np.stack([tex] * 3, axis=-1)
    if tex.shape[2] == 3:
        tex = np.concatenate([tex, np.full(tex.shape[:2] + (1,), 255, tex.dtype)], axis=2)
    return np.ascontiguousarray(tex.astype(np.uint8))


def _cmap_tensor(colormap, device) -> torch.Tensor:
    return torch.as_tensor(np.array([_rgba(c) for c in colormap], dtype=np.float64)).to(device)


def render_planes(values: torch.Tensor, strides, nimg: int, channels: int, width: int, height: int,
                  spacing, spec: RenderSpec, want_coverage: bool = False):
    """GPU render of ``nimg`` images (mdc_render): RGBA8 (nimg, H, W, 4) and
    optionally the float coverage (nimg, H, W).  ``strides`` =
    (img_stride, channel_stride, row_stride, pixel_stride) in elements."""
    lib = _lib.require_cuda()
    if spec.mode not in _MODE_CODE:
        raise RenderError(f"unknown mode {spec.mode!r}")
    if spec.mode in ("gradient", "texture") and channels != 2:
        raise RenderError(f"{spec.mode} mode requires a two-dimensional target")
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
    for i, c in enumerate(spec.gradient_corners):
        cc = list(c) + [255] * (4 - len(c))
        for k in range(4):
            a.gradient_corners[4 * i + k] = int(cc[k])
    a.adaptive_target_px = float(spec.adaptive_target_px)
    tex_t = None
    if spec.mode == "texture":
        tex = _texture_rgba(spec.texture)
        tex_t = torch.as_tensor(tex).to(dev)
        a.texture, a.tex_h, a.tex_w = _lib.ptr(tex_t), tex.shape[0], tex.shape[1]
    _lib.check(lib.mdc_render(ctypes.byref(a), _lib.stream_ptr()), "mdc_render")
    if tex_t is not None:
        torch.cuda.current_stream().synchronize()
    return out, cov


def _field_planes(fld: CoordinateField):
    dev = getattr(fld, "device_coords", None)
    if isinstance(dev, torch.Tensor) and dev.is_cuda and dev.dtype == torch.float64 and dev.is_contiguous():
        coords = dev  # compute_field kept the GPU copy (same values as fld.coords)
    else:
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


def render_device(fld: CoordinateField, spec: RenderSpec) -> torch.Tensor:
    """``render`` without the host round trip: (H, W, 4) uint8 CUDA tensor
    (the service composes the overlay on it and downloads once)."""
    mode = spec.mode
    if mode not in MODES:
        raise RenderError(f"unknown mode {mode!r}")
    coords, strides = _field_planes(fld)
    out, _ = render_planes(coords, strides, 1, fld.active_channels, fld.width, fld.height, spec.spacing, spec)
    return out[0]


def point_mask(img_shape, positions, transform, spec: RenderSpec) -> np.ndarray:
    """render.py:260-269: boolean mask of pixels the point overlay covers
    (a host helper for comparisons, not a render path)."""
    h, w = img_shape
    mask = np.zeros((h, w), dtype=bool)
    r = spec.point_radius
    pix = transform.to_pixels(np.asarray(positions, dtype=float).reshape(-1, 2))
    yy, xx = np.mgrid[0:h, 0:w]
    for px, py in pix:
        mask |= np.hypot(xx - px, yy - py) <= r + 0.5
    return mask


def render_contours(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:129-132 on the GPU."""
    return _render_gpu(fld, RenderSpec(**{**spec.__dict__, "mode": "contour"}))


def render_discrete(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:142-148 on the GPU."""
    mode = spec.mode if spec.mode in ("discrete", "discrete+contour") else "discrete"
    return _render_gpu(fld, RenderSpec(**{**spec.__dict__, "mode": mode}))


def render_adaptive(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:169-178 on the GPU."""
    return _render_gpu(fld, RenderSpec(**{**spec.__dict__, "mode": "adaptive"}))


def render_gradient(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:194-201 on the GPU."""
    if fld.active_channels != 2:
        raise RenderError("gradient mode requires a two-dimensional target")
    return _render_gpu(fld, RenderSpec(**{**spec.__dict__, "mode": "gradient"}))


def render_texture(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:224-234 on the GPU."""
    return _render_gpu(fld, RenderSpec(**{**spec.__dict__, "mode": "texture"}))


def render(fld: CoordinateField, spec: RenderSpec) -> RenderedImage:
    """render.py:272-283: every mode renders on the GPU (mdc_render)."""
    if spec.mode in _MODE_CODE:
        if spec.mode == "gradient" and fld.active_channels != 2:
            raise RenderError("gradient mode requires a two-dimensional target")
        return _render_gpu(fld, spec)
    raise RenderError(f"unknown mode {spec.mode!r}")


def overlay_points_device(pixels: torch.Tensor, positions, transform, spec: RenderSpec) -> torch.Tensor:
    """render.py:237-257 on the GPU (mdc_overlay_points): discs composited in
    point order onto an (H, W, 4) uint8 CUDA tensor, in place."""
    lib = _lib.require_cuda()
    h, w = pixels.shape[:2]
    pix = np.ascontiguousarray(transform.to_pixels(np.asarray(positions, dtype=float).reshape(-1, 2)))
    n = len(pix)
    if n == 0:
        return pixels
    dev = pixels.device
    pix_t = torch.as_tensor(pix).to(dev)
    col = list(spec.point_color) + [255] * (4 - len(spec.point_color))
    r = float(spec.point_radius)
    nbytes = int(lib.mdc_overlay_workspace_bytes(n, r))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    col_arr = (ctypes.c_int32 * 4)(*[int(c) for c in col])
    _lib.check(lib.mdc_overlay_points(_lib.ptr(pixels), w, h, n, _lib.ptr(pix_t), r,
                                      ctypes.cast(col_arr, ctypes.c_void_p), _lib.ptr(ws), nbytes,
                                      _lib.stream_ptr()), "mdc_overlay_points")
    return pixels


def overlay_points(img: RenderedImage, positions, transform, spec: RenderSpec) -> RenderedImage:
    """render.py:237-257 anti-aliased discs at the projected points (GPU)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
    if dev is None:
        _lib.require_cuda()
    px = torch.as_tensor(np.ascontiguousarray(img.pixels)).to(dev)
    overlay_points_device(px, positions, transform, spec)
    out = px.cpu().numpy()
    return RenderedImage(width=out.shape[1], height=out.shape[0], pixels=out)


def render_legend(fld: CoordinateField, spec: RenderSpec, width: int = 72) -> RenderedImage:
    """render.py:286-308: value-to-colour strip for channel 0 with PIL text
    labels (a UI helper; host-side, SURVEY.md §2 'legend' is out of the GPU
    hot path)."""
    from PIL import Image, ImageDraw

    h = fld.height
    vals = np.linspace(fld.coords[..., 0].max(), fld.coords[..., 0].min(), h)[:, None].repeat(width, axis=1)
    if spec.mode in ("discrete", "discrete+contour"):
        table = np.array([_rgba(c) for c in spec.colormap])
        img = table[np.mod(np.floor(vals / spec.spacing).astype(np.int64), len(table))]
    elif spec.mode == "gradient":
        c00, c10, c01, c11 = (_rgba(c) for c in spec.gradient_corners)
        fu = np.mod(vals / spec.spacing, 1.0)[..., None]
        img = (1 - fu) * c00 + fu * c10
    else:
        img = _flat(vals.shape, spec.background)
    on_line = np.abs(vals - spec.spacing * np.round(vals / spec.spacing))
    step = abs(vals[0, 0] - vals[-1, 0]) / max(h - 1, 1)
    _over(img, spec.line_color, np.clip(1.0 - on_line / max(step, 1e-30), 0.0, 1.0))
    pil = Image.fromarray(np.clip(np.rint(img * 255), 0, 255).astype(np.uint8), "RGBA")
    draw = ImageDraw.Draw(pil)
    draw.text((3, 2), f"{vals[0, 0]:.3g}", fill=(0, 0, 0, 255))
    draw.text((3, h - 12), f"{vals[-1, 0]:.3g}", fill=(0, 0, 0, 255))
    draw.text((3, h // 2), f"step {spec.spacing:.3g}", fill=(0, 0, 0, 255))
    return RenderedImage(width=width, height=h, pixels=np.array(pil))


def attach_legend(img: RenderedImage, legend: RenderedImage) -> RenderedImage:
    """render.py:311-318."""
    if legend.height != img.height:
        raise RenderError("legend height must match the image")
    return RenderedImage(width=img.width + legend.width, height=img.height,
                         pixels=np.concatenate([img.pixels, legend.pixels], axis=1))
