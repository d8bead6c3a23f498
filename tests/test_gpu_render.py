"""GPU rendering (mdc_render) against the reference's line coverage (golden)
and the oracle's restatement of render.py's compositing."""
import numpy as np
import pytest

import oracle as O

from paper_1408_0677_b200 import field as F
from paper_1408_0677_b200 import render as R

pytestmark = pytest.mark.gpu


def _fld(c1, name):
    W, H = (int(v) for v in c1["field_wh"])
    ch = int(c1[f"channels_{name}"])
    tr = F.ViewportTransform.fit(c1["field_positions"], W, H)
    return F.CoordinateField(W, H, np.ascontiguousarray(c1[f"field_{name}"]), c1["field_positions"], tr, ch)


def test_line_coverage_matches_reference(c1):
    for k in range(4):
        name = f"affine_dim{k}"
        fld = _fld(c1, name)
        cov = R.line_coverage(fld, float(c1[f"spacing_{name}"]), 1.5)
        assert np.abs(cov - c1[f"coverage_{name}"]).max() <= 1e-6, k


@pytest.mark.parametrize("mode", ["contour", "discrete", "discrete+contour"])
def test_render_rgba_matches_restated_reference(c1, mode):
    for name in ("affine_dim0", "affine_dim2", "rigid_dims01", "affine_proj"):
        fld = _fld(c1, name)
        sp = float(c1[f"spacing_{name}"]) if f"spacing_{name}" in c1.files else 0.5
        img = R.render(fld, R.RenderSpec(mode=mode, spacing=sp))
        ref = O.render_rgba(fld.coords, fld.active_channels, sp, mode)
        diff = np.abs(img.pixels.astype(int) - ref.astype(int))
        assert diff.max() <= 1, (name, mode)
        assert (diff > 0).mean() <= 1e-3, (name, mode)


def test_render_fields_per_channel(c1):
    pos = c1["field_positions"]
    W, H = (int(v) for v in c1["field_wh"])
    raw = c1["raw"]
    sp = np.array([float(c1[f"spacing_affine_dim{k}"]) for k in range(4)])
    blk = F.compute_fields(pos, raw, F.MlsParams("affine"), W, H, dtype="f64")
    imgs = R.render_fields(blk, sp, R.RenderSpec(mode="discrete+contour", spacing=1.0)).cpu().numpy()
    for k in range(4):
        ref = O.render_rgba(np.stack([c1[f"field_affine_dim{k}"][..., 0]] * 2, axis=-1), 1, sp[k],
                            "discrete+contour")
        diff = np.abs(imgs[k].astype(int) - ref.astype(int))
        assert (diff > 1).mean() <= 2e-3, k   # fp64 field vs reference field: ~1e-12 apart


@pytest.mark.parametrize("mode", ["adaptive", "gradient", "texture"])
def test_render_remaining_modes(c1, mode):
    rng = np.random.default_rng(4)
    tex = rng.integers(0, 256, (13, 17, 3)).astype(np.uint8)
    names = ("affine_dims23", "rigid_dims01", "affine_proj") if mode != "adaptive" else ("affine_dim1", "affine_proj")
    for name in names:
        fld = _fld(c1, name)
        sp = float(c1[f"spacing_{name}"]) if f"spacing_{name}" in c1.files else 0.5
        spec = R.RenderSpec(mode=mode, spacing=sp, texture=tex if mode == "texture" else None)
        img = R.render(fld, spec)
        ref = O.render_rgba(fld.coords, fld.active_channels, sp, mode, texture=tex)
        diff = np.abs(img.pixels.astype(int) - ref.astype(int))
        assert diff.max() <= 1, (name, mode)
        assert (diff > 0).mean() <= 1e-3, (name, mode)


def test_gradient_mode_needs_two_channels(c1):
    with pytest.raises(R.RenderError):
        R.render(_fld(c1, "affine_dim0"), R.RenderSpec(mode="gradient", spacing=1.0))


def test_overlay_points_matches_reference_order(c1):
    fld = _fld(c1, "affine_dim0")
    base = R.render(fld, R.RenderSpec(mode="discrete", spacing=float(c1["spacing_affine_dim0"])))
    pos = np.concatenate([c1["field_positions"], c1["field_positions"][:20] + 1e-3])  # overlapping discs
    spec = R.RenderSpec(point_radius=2.5)
    got = R.overlay_points(base, pos, fld.transform, spec).pixels
    ref = O.overlay_points(base.pixels, fld.transform.to_pixels(pos), 2.5)
    diff = np.abs(got.astype(int) - ref.astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() <= 1e-3


@pytest.mark.parametrize("dtype,eps", [("f64", 1e-9), ("f32", 1e-4)])
def test_fused_band_shading_matches_reference_render_discrete(c1, dtype, eps):
    """North-star (3): band shading fused into the MLS epilogue.  Each
    channel's RGBA8 from compute_fields(..., colormap=...) equals the
    reference's render_discrete of that single-dimension field
    (render.py:142-148: table[mod(floor(u / s), 11)] -> clip(rint(255 x))),
    built here from the reference's own golden band indices; exact except
    within eps of a band boundary (the snap pass restamps snapped pixels)."""
    pos = c1["field_positions"]
    W, H = (int(v) for v in c1["field_wh"])
    names = [f"affine_dim{k}" for k in range(4)]
    tv = np.column_stack([c1[f"targets_{nm}"][:, 0] for nm in names])
    sp = np.array([float(c1[f"spacing_{nm}"]) for nm in names])
    blk = F.compute_fields(pos, tv, F.MlsParams("affine"), W, H, dtype=dtype, band_spacing=sp,
                           colormap=R.DEFAULT_COLORMAP)
    got = blk.rgba.cpu().numpy()
    table = F.palette_rgba8(R.DEFAULT_COLORMAP).view(np.uint8).reshape(-1, 4)
    for k, nm in enumerate(names):
        ref_bands = c1[f"bands_{nm}"]
        want = table[np.mod(ref_bands, len(table))]
        u = c1[f"field_{nm}"][..., 0] / sp[k]
        ok = np.abs(u - np.rint(u)) >= eps
        assert np.array_equal(got[k][ok], want[ok]), nm
        # and the fused bands agree with the fused colours everywhere
        assert np.array_equal(got[k], table[np.mod(blk.bands[k].cpu().numpy(), len(table))])
