"""GPU rendering (mdc_render) against the reference's line coverage (golden)
and the oracle's restatement of render.py's compositing."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import golden_mesh

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
