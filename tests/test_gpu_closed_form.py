"""Closed-form MLS properties through the GPU path (fp64 and fp32), ported
from the reference's test_field.py:191-262 field-level tests, plus the edge
cases of the fused entry (one control, one channel, one-pixel rasters,
degenerate control sets)."""
import numpy as np
import pytest

from conftest import normwise
from paper_1408_0677_b200 import field as F
from paper_1408_0677_b200 import mesh as M

pytestmark = pytest.mark.gpu


def _off_snap(fld, pts):
    xs, ys = fld.transform.pixel_center_grids()
    centers = np.stack([xs, ys], axis=-1)
    eps = (0.25 * max(fld.transform.units_per_px)) ** 2
    d2 = ((centers[:, :, None, :] - pts[None, None, :, :]) ** 2).sum(-1).min(-1)
    return centers, d2 >= eps


@pytest.mark.parametrize("variant", ["mean", "affine", "rigid"])
def test_identity_targets_identity_field(variant):
    """test_field.py:191-207."""
    rng = np.random.default_rng(14)
    pts = rng.uniform(0.0, 4.0, (30, 2))
    mesh = M.delaunay(pts, seed=0)
    fld = F.compute_field(mesh, mesh.original_pos, F.projection_targets(mesh), F.MlsParams(variant=variant), 80, 80)
    centers, off = _off_snap(fld, pts)
    assert np.abs(fld.coords - centers)[off].max() <= 1e-9
    assert np.all(np.isfinite(fld.coords))


def test_single_control_uniform_shift_field():
    """test_field.py:210-219 (mean: the field is v + (q - p) everywhere)."""
    mesh = M.delaunay(np.array([[0.0, 0.0], [4.0, 0.0], [0.0, 4.0]]))
    targets = F.TargetAssignment(targets=np.array([[1.0, 2.0], [5.0, 2.0], [1.0, 6.0]]), mode="projection")
    fld = F.compute_field(mesh, mesh.original_pos, targets, F.MlsParams(variant="mean"), 50, 50)
    xs, ys = fld.transform.pixel_center_grids()
    np.testing.assert_allclose(fld.coords[..., 0], xs + 1.0, atol=1e-9)
    np.testing.assert_allclose(fld.coords[..., 1], ys + 2.0, atol=1e-9)


def test_control_pixels_near_targets():
    """test_field.py:222-240 (discrete point identity, affine)."""
    rng = np.random.default_rng(33)
    pts = rng.uniform(0.0, 6.0, (40, 2))
    mesh = M.delaunay(pts, seed=0)
    q = pts + rng.normal(0, 0.3, pts.shape)
    fld = F.compute_field(mesh, pts, F.TargetAssignment(targets=q, mode="projection"),
                          F.MlsParams(variant="affine"), 120, 120)
    jac = fld.jacobian()
    pix = fld.transform.to_pixels(pts)
    for i, (px, py) in enumerate(pix):
        x = int(np.clip(round(px), 0, fld.width - 1))
        y = int(np.clip(round(py), 0, fld.height - 1))
        err = np.hypot(*(fld.coords[y, x] - q[i]))
        local = np.linalg.norm(jac[max(0, y - 1):y + 2, max(0, x - 1):x + 2].reshape(-1, 4), axis=1).max()
        assert err <= local


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-9), ("f32", 1e-4)])
def test_affine_reproduces_global_affine_map(dtype, tol):
    """test_field.py:70-80 at field level: q = p A + b  =>  f(v) = v A + b."""
    rng = np.random.default_rng(5)
    a = np.array([[2.0, 0.5], [-0.3, 1.0]])
    b = np.array([1.0, -2.0])
    p = rng.uniform(-1, 1, (60, 2))
    q = p @ a + b
    mesh = M.delaunay(p, seed=0)
    fld = F.compute_field(mesh, p, F.TargetAssignment(targets=q, mode="projection"), F.MlsParams("affine"),
                          64, 48, dtype=dtype)
    centers, off = _off_snap(fld, p)
    expect = centers @ a + b
    assert normwise(fld.coords[off], expect[off]) <= tol


def test_rigid_reproduces_rot90_plus_translation():
    """test_field.py:83-93 at field level."""
    rng = np.random.default_rng(6)
    rot90 = np.array([[0.0, 1.0], [-1.0, 0.0]])
    t = np.array([1.0, 1.0])
    p = rng.uniform(-1, 1, (40, 2))
    q = p @ rot90 + t
    mesh = M.delaunay(p, seed=0)
    fld = F.compute_field(mesh, p, F.TargetAssignment(targets=q, mode="projection"), F.MlsParams("rigid"), 64, 64)
    centers, off = _off_snap(fld, p)
    assert np.abs(fld.coords - (centers @ rot90 + t))[off].max() <= 1e-8


def test_fused_single_channel_single_control_and_tiny_rasters():
    """Edge cases of the fused entry: d = 1, one control (mean: uniform shift),
    1 x 1 and 1 x H / W x 1 rasters, row bands of one row."""
    pos = np.array([[0.3, -0.2], [1.0, 2.0], [-1.5, 0.5]])
    q = np.array([[1.0], [2.0], [-3.0]])
    for W, H in ((1, 1), (1, 17), (23, 1), (5, 3)):
        for dt in ("f32", "f64"):
            blk = F.compute_fields(pos, q, F.MlsParams("affine"), W, H, dtype=dt)
            blk.check_finite()
            assert tuple(blk.values.shape) == (1, H, W)
            if H > 1:
                rows = [F.compute_fields(pos, q, F.MlsParams("affine"), W, H, dtype=dt,
                                         row_range=(r, r + 1)).values for r in range(H)]
                import torch
                assert torch.equal(torch.cat(rows, dim=1), blk.values)
    one = F.compute_fields(pos[:1], q[:1], F.MlsParams("mean"), 16, 9, dtype="f64")
    xs = one.transform.pixel_center_grids()[0]
    # mean with one control: f = v_axis + (q - p_axis) everywhere (axis 0)
    np.testing.assert_allclose(one.values[0].cpu().numpy(), xs + (q[0, 0] - pos[0, 0]), atol=1e-12)


def test_degenerate_affine_controls_raise_like_the_reference():
    """One control (or all coincident) leaves the affine moment matrix
    singular: the reference produces non-finite values and raises FieldError
    (field.py:650-651); so does the GPU path."""
    pos = np.array([[0.0, 0.0]])
    mesh = M.delaunay(np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]))
    with pytest.raises(F.FieldError):
        F.compute_field(mesh, pos, F.TargetAssignment(targets=np.array([[1.0, 0.0]]), mode="dims", dims=("a",)),
                        F.MlsParams("affine"), 8, 8)


def test_point_evaluators_closed_form():
    """test_field.py:52-93: the single-point MLS evaluators (GPU seam kernels)."""
    params = F.MlsParams(variant="mean")
    p, q = np.array([[0.5, 0.5]]), np.array([[3.5, -0.5]])
    for v in np.random.default_rng(1).uniform(-5, 5, (20, 2)):
        np.testing.assert_allclose(F.mean_mls(v, p, q, params), v + [3.0, -1.0], atol=1e-12)
    p2, q2 = np.array([[-1.0, 0.0], [1.0, 0.0]]), np.array([[-1.0, 0.0], [1.0, 2.0]])
    np.testing.assert_allclose(F.mean_mls((0.0, 0.0), p2, q2, F.MlsParams("mean", alpha=1.0)), [0.0, 1.0], atol=1e-12)
    rng = np.random.default_rng(5)
    a, b = np.array([[2.0, 0.0], [0.0, 1.0]]), np.array([1.0, 0.0])
    pa = rng.uniform(-1, 1, (5, 2))
    for v in rng.uniform(-2, 2, (50, 2)):
        np.testing.assert_allclose(F.affine_mls(v, pa, pa @ a + b, F.MlsParams("affine")), v @ a + b, atol=1e-6)
    rot90, t = np.array([[0.0, 1.0], [-1.0, 0.0]]), np.array([1.0, 1.0])
    pr = np.random.default_rng(6).uniform(-1, 1, (5, 2))
    for v in np.random.default_rng(7).uniform(-2, 2, (50, 2)):
        np.testing.assert_allclose(F.rigid_mls(v, pr, pr @ rot90 + t, F.MlsParams("rigid")), v @ rot90 + t, atol=1e-6)
    # inside the snap radius: the control's own target, exactly
    assert np.array_equal(F.affine_mls(pa[2], pa, pa @ a + b, F.MlsParams("affine")), (pa @ a + b)[2])
    assert F.mls_weight((0.0, 0.0), (0.0, 0.0), 1.5) is F.AT_CONTROL_POINT
    assert F.mls_weight((0.0, 0.0), (2.0, 0.0), 1.0) == 0.25


def test_empty_and_ragged_inputs_raise_cleanly():
    with pytest.raises(F.FieldError):
        F.compute_fields(np.zeros((0, 2)), np.zeros((0, 3)), F.MlsParams("affine"), 8, 8)
    with pytest.raises(F.FieldError):
        F.compute_fields(np.zeros((4, 2)), np.zeros((4, 0)), F.MlsParams("affine"), 8, 8)
    with pytest.raises(ValueError):
        F.compute_fields(np.zeros((4, 3)), np.zeros((4, 1)), F.MlsParams("affine"), 8, 8)
    with pytest.raises(ValueError):
        F.compute_fields(np.random.rand(4, 2), np.zeros((5, 1)), F.MlsParams("affine"), 8, 8)


def test_rigid_degenerate_raises():
    """Reference test_field.py:108-113: a symmetric pinch cancels the rotation
    estimate at the midpoint; the scalar rigid evaluator raises (field.py:263-265)
    while the field path keeps _kernels.rigid_field's per-pixel mean fallback."""
    p = np.array([[-1.0, 0.0], [1.0, 0.0]])
    q = np.array([[0.0, -1.0], [0.0, 1.0]])
    with pytest.raises(F.DegenerateRotation):
        F.rigid_mls(np.array([0.0, 0.0]), p, q, F.MlsParams(variant="rigid", alpha=1.0))
    # off the pinch the rotation is well defined
    out = F.rigid_mls(np.array([0.3, 0.2]), p, q, F.MlsParams(variant="rigid", alpha=1.0))
    assert np.isfinite(out).all()
