"""MLS parity at the configurations bench.py reports (SURVEY.md §8d configs
2, 3 and 5), against the CPU oracle (pinned bit-exact to the reference's own
fields, tests/test_oracle.py).  The small golden scenes pin every code path;
these tests pin the same kernels at the bench's sizes, where fp32 summation
over 100k controls and the multi-chunk tensor-core path are exercised.

Contracts (written here): fp32 <= 1e-4 and fp64 <= 1e-10
normwise per channel; band indices bit-exact except within eps of a band
boundary (1e-4 fp32); snapped pixels exactly the control's target.
Reference: field.py:582-659 (compute_field), render.py:135-139 (bands),
field.py:388-412 (snap)."""
import numpy as np
import pytest
import torch

import bench
import oracle as O
from conftest import normwise

from paper_1408_0677_b200 import dataset as D
from paper_1408_0677_b200 import field as F
from paper_1408_0677_b200 import layout as L
from paper_1408_0677_b200 import mesh as M
from paper_1408_0677_b200 import projection as P
from paper_1408_0677_b200.render import auto_spacing

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
FP64_TOL = 1e-10
BAND_EPS = 1e-4
REPORT = {}


def _scene(cfg_id, layout_iters=None):
    """bench.py's workload: GMM data -> PCA -> Delaunay -> layout on the GPU
    (CUDA-graph steps, as bench.py) -> positions; raw targets; auto spacing."""
    cfg = bench.CONFIGS[cfg_id]
    X = bench.gmm(cfg["n"], cfg["d"], cfg["seed"])
    ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(cfg["d"])], data=X))
    _, cloud = P.pca_project(ds)
    raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])
    pos = cloud.positions
    iters = cfg["iters"] if layout_iters is None else layout_iters
    if iters:
        mesh = M.delaunay(cloud, seed=0)
        params = L.LayoutParams.defaults_for(mesh, iterations=iters)
        eng = L.LayoutEngine(mesh, params)
        eng.set_positions(mesh.original_pos)
        eng.run(L.temperature_schedule(params.initial_temp, params.decay_lambda, iters))
        pos = eng.pos.cpu().numpy()
    return cfg, pos, raw


@pytest.fixture(scope="module")
def config3():
    return _scene(3)


def _rows_spread(H, k):
    return sorted({int(r) for r in np.linspace(0, H - 1, k)})


def _gpu_rows(pos, raw, W, H, rows, dtype, spacing=None):
    vals, bands = [], []
    for r in rows:
        blk = F.compute_fields(pos, raw, F.MlsParams("affine"), W, H, dtype=dtype, row_range=(r, r + 1),
                               band_spacing=spacing)
        vals.append(blk.values.double().cpu().numpy()[:, 0])
        if spacing is not None:
            bands.append(blk.bands.cpu().numpy()[:, 0])
    v = np.stack(vals, axis=1).transpose(1, 2, 0)  # (rows, W, d)
    b = np.stack(bands, axis=1).transpose(1, 2, 0) if spacing is not None else None
    return v, b


def _oracle_snapped(pos, raw, W, H, rows, cols=None):
    """Oracle field on the rows (and columns), then field.py:388-412's snap
    restricted to each row (the snap is per pixel, so a row is independent)."""
    ref = O.affine_fields(pos, raw, W, H, rows=rows, cols=cols)
    if cols is not None:
        return ref, np.zeros(ref.shape[:2], bool)
    vp = O.viewport(pos, W, H)
    x0, y0, x1, y1, sx, sy = vp
    eps = (0.25 * max(sx, sy)) ** 2
    snapped = np.zeros(ref.shape[:2], bool)
    for i, r in enumerate(rows):
        before = ref[i:i + 1].copy()
        row = np.ascontiguousarray(ref[i:i + 1])
        O.snap(row, pos, raw, (x0, y0, x1, y1 - r * sy, sx, sy), eps)
        ref[i] = row[0]
        snapped[i] = (row[0] != before[0]).any(axis=-1)
    return ref, snapped


def test_config3_all_channels_bands_and_snap(config3):
    """Config 3 (4K, N=100k laid out 500 iterations, d=32): all 32 channels on
    8 rows spread top to bottom; band indices bit-exact outside eps; snapped
    pixels exactly the control targets."""
    cfg, pos, raw = config3
    W, H, d = cfg["W"], cfg["H"], cfg["d"]
    rows = _rows_spread(H, 8)
    spacing = np.array([auto_spacing(raw[:, k]) for k in range(d)])
    got, gb = _gpu_rows(pos, raw, W, H, rows, "f32", spacing)
    ref, snapped = _oracle_snapped(pos, raw, W, H, rows)
    errs = [normwise(got[..., k], ref[..., k]) for k in range(d)]
    REPORT["config3_fp32_worst_channel"] = max(errs)
    assert max(errs) <= FP32_TOL, errs
    # snapped pixels: exactly the (fp32-rounded) target of the winning control
    assert snapped.any(), "the 8 rows should cross at least one snap disc at N=100k"
    assert np.array_equal(got[snapped], ref[snapped].astype(np.float32).astype(np.float64))
    REPORT["config3_snapped_pixels"] = int(snapped.sum())
    # bands: floor(u / s) (render.py:135-139), bit-exact away from a boundary
    u = ref / spacing
    ok = np.abs(u - np.rint(u)) >= BAND_EPS
    assert np.array_equal(gb[ok], np.floor(u[ok]).astype(np.int32))
    REPORT["config3_band_pixels_compared"] = int(ok.sum())
    REPORT["config3_band_pixels_within_eps"] = int((~ok).sum())


def test_config3_fp64_mode(config3):
    """fp64 parity mode at the bench scale (summation over 100k controls in
    fp64): 4 rows, all channels, <= 1e-10 normwise."""
    cfg, pos, raw = config3
    W, H, d = cfg["W"], cfg["H"], cfg["d"]
    rows = _rows_spread(H, 4)
    got, _ = _gpu_rows(pos, raw, W, H, rows, "f64")
    ref, _ = _oracle_snapped(pos, raw, W, H, rows)
    errs = [normwise(got[..., k], ref[..., k]) for k in range(d)]
    REPORT["config3_fp64_worst_channel"] = max(errs)
    assert max(errs) <= FP64_TOL, errs


def test_config2_32_rows_16_dims():
    """Config 2 (1080p, N=10k laid out 500 iterations, d=16): 32 rows x 16 dims."""
    cfg, pos, raw = _scene(2)
    W, H, d = cfg["W"], cfg["H"], cfg["d"]
    rows = _rows_spread(H, 32)
    spacing = np.array([auto_spacing(raw[:, k]) for k in range(d)])
    got, gb = _gpu_rows(pos, raw, W, H, rows, "f32", spacing)
    ref, snapped = _oracle_snapped(pos, raw, W, H, rows)
    errs = [normwise(got[..., k], ref[..., k]) for k in range(d)]
    REPORT["config2_fp32_worst_channel"] = max(errs)
    assert max(errs) <= FP32_TOL, errs
    assert np.array_equal(got[snapped], ref[snapped].astype(np.float32).astype(np.float64))
    u = ref / spacing
    ok = np.abs(u - np.rint(u)) >= BAND_EPS
    assert np.array_equal(gb[ok], np.floor(u[ok]).astype(np.int32))


@pytest.mark.parametrize("d,stride", [(64, 4), (128, 8), (256, 8)])
def test_config5_multichunk_tensor_core_path(d, stride):
    """Config 5 (4K, N=100k, d = 64 / 128 / 256: several 32-channel chunks of
    the tcgen05 kernel, each re-evaluating the weights): 4 rows spread top to
    bottom, every `stride`-th column (bounds the fp64 oracle's cost)."""
    cfg = bench.CONFIGS[3]
    X = bench.gmm(cfg["n"], 256, 3)  # tools/dsweep.py's config-5 data
    ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(256)], data=X))
    _, cloud = P.pca_project(ds)
    pos = cloud.positions
    raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])[:, :d]
    W, H = cfg["W"], cfg["H"]
    rows = _rows_spread(H, 4)
    cols = np.arange(0, W, stride)
    got, _ = _gpu_rows(pos, raw, W, H, rows, "f32")
    got = got[:, cols]
    ref = O.affine_fields(pos, raw, W, H, rows=rows, cols=cols)
    # compare away from snap discs (the oracle here is unsnapped)
    vp = O.viewport(pos, W, H)
    xs, ys = O.pixel_centers(vp, W, H)
    eps = (0.25 * max(vp[4], vp[5])) ** 2
    keep = np.ones(got.shape[:2], bool)
    from scipy.spatial import cKDTree

    dist, _ = cKDTree(pos).query(np.stack([xs[rows][:, cols], ys[rows][:, cols]], -1).reshape(-1, 2))
    keep = (dist.reshape(keep.shape) ** 2 >= eps)
    errs = [normwise(got[..., k][keep], ref[..., k][keep]) for k in range(d)]
    REPORT[f"config5_d{d}_fp32_worst_channel"] = max(errs)
    assert max(errs) <= FP32_TOL, errs


def test_zz_print_report():
    """Collected numbers for profiles/r02_parity_report.txt."""
    for k, v in sorted(REPORT.items()):
        print(f"{k}: {v}")
