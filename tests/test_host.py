"""Host-side logic and the C-ABI boundary, without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

from paper_1408_0677_b200 import _lib, field, layout, mesh
from paper_1408_0677_b200.field import MlsParams, _ldq


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "mdc.h")).read()
    return sorted(set(re.findall(r"MDC_API[^;]*?\b(mdc_[a-z0-9_]+)\s*\(", txt, flags=re.S)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, s
    assert lib.mdc_version() == 1


def test_ctypes_structs_match_header_field_order():
    txt = open(os.path.join(ROOT, "include", "mdc.h")).read()
    for cname, py in (("MdcMlsArgs", _lib.MdcMlsArgs), ("MdcLayoutArgs", _lib.MdcLayoutArgs),
                      ("MdcRenderArgs", _lib.MdcRenderArgs), ("MdcLinearArgs", _lib.MdcLinearArgs)):
        body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (cname, cname), txt, re.S).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        names = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            decl = re.sub(r"^(const\s+)?\w+\s*", "", decl)
            names += [re.sub(r"\[.*\]", "", n).strip().lstrip("*").strip() for n in decl.split(",")]
        assert names == [f[0] for f in py._fields_], cname


def test_workspace_size_queries_without_gpu():
    lib = _lib.load()
    assert lib.mdc_snap_workspace_bytes(3840, 2160) == 3840 * 2160 * 12
    assert lib.mdc_layout_workspace_bytes(10000, 32) > 10000 * 16
    assert lib.mdc_pca_workspace_bytes(1000, 16) > 16 * 16 * 8


def test_mlsparams_validation_mirrors_reference():
    with pytest.raises(ValueError):
        MlsParams(variant="mean", alpha=0.05)
    with pytest.raises(ValueError):
        MlsParams(variant="mean", alpha=4.5)
    with pytest.raises(ValueError):
        MlsParams(variant="bogus")
    with pytest.raises(ValueError):
        MlsParams(reg_eps=0.0)
    assert MlsParams(variant="affine").resolved_alpha == 1.5
    assert MlsParams(variant="rigid").resolved_alpha == 1.0


def test_ldq_padding_rules():
    F32, F64 = _lib.MDC_F32, _lib.MDC_F64
    assert _ldq(1, F32, _lib.MDC_AFFINE) == 4
    assert _ldq(2, F64, _lib.MDC_AFFINE) == 2
    assert _ldq(32, F32, _lib.MDC_AFFINE) == 32
    assert _ldq(33, F32, _lib.MDC_AFFINE) == 64
    assert _ldq(5, F32, _lib.MDC_MEAN) == 8
    assert _ldq(17, F64, _lib.MDC_AFFINE) == 32
    assert _ldq(2, F32, _lib.MDC_RIGID) == 4


def test_assemble_matches_reference_mesh(c1, g2k):
    for g in (c1, g2k):
        pts = g["original_pos"]
        m = mesh.delaunay(pts, seed=0)
        for k in ("triangles", "csr_offsets", "csr_targets", "fan_offsets", "fan_nodes"):
            assert np.array_equal(getattr(m, k), g[k]), k


def test_layout_topology_order(c1):
    from helpers import golden_mesh

    m = golden_mesh(c1)
    topo = mesh.layout_topology(m)
    tris = c1["triangles"]
    inc, off = topo["inc"], topo["inc_off"]
    assert off[-1] == 3 * len(tris)
    for v in range(m.node_count):
        ent = inc[off[v]:off[v + 1]]
        t, k = ent >> 2, ent & 3
        assert np.all(tris[t, k] == v)
        key = k.astype(np.int64) * len(tris) + t
        assert np.all(np.diff(key) > 0)  # sorted by (corner, triangle)
    assert topo["tris"].shape[1] == 4 and topo["tris"].dtype == np.int32


def test_temperature_schedule_is_sequential_product():
    t = layout.temperature_schedule(0.37, 0.99, 500)
    ref = 0.37
    for i in range(500):
        assert t[i] == ref
        ref = ref * 0.99


def test_layout_params_defaults(c1):
    from helpers import golden_mesh

    m = golden_mesh(c1)
    p = layout.LayoutParams.defaults_for(m, iterations=50)
    assert p.repulsion_c == float(c1["lp_repulsion_c"])
    assert p.softening_eta == float(c1["lp_softening_eta"])
    with pytest.raises(ValueError):
        layout.LayoutParams(1, 1, 1, 1, 1, 1.5)


def test_interpolate_layout_bounds(c1):
    from helpers import golden_mesh

    m = golden_mesh(c1)
    st = layout.LayoutState(mesh=m, iteration=1, temperature=1.0, relaxed_pos=c1["states"][5])
    assert np.array_equal(layout.interpolate_layout(st, 0.0), m.original_pos)
    assert np.array_equal(layout.interpolate_layout(st, 1.0), c1["states"][5])
    with pytest.raises(layout.TOutOfRange):
        layout.interpolate_layout(st, 1.5)


def test_field_raster_round_trip(tmp_path):
    tr = field.ViewportTransform(0.0, 0.0, 1.0, 1.0, 40, 30)
    xs, ys = tr.pixel_center_grids()
    fld = field.CoordinateField(40, 30, np.stack([xs, xs * ys], axis=-1), np.zeros((0, 2)), tr)
    path = tmp_path / "f.mlsf"
    field.write_field(fld, path)
    w, h, data = field.read_field(path)
    assert (w, h) == (40, 30) and np.array_equal(data, fld.coords)


def test_compute_paths_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        _lib.require_cuda()



def test_row_band_plan():
    """compute_fields_to_host band planning: contiguous cover of the rows, a
    small tail band last."""
    from paper_1408_0677_b200.field import plan_row_bands

    for r0, r1, nb in [(0, 2160, 4), (0, 1080, 4), (100, 2000, 3), (0, 37, 4), (0, 2, 8), (0, 1, 4), (5, 6, 4)]:
        plan = plan_row_bands(r0, r1, nb)
        assert plan[0][0] == r0 and plan[-1][1] == r1
        assert all(a[1] == b[0] for a, b in zip(plan, plan[1:])) and all(a < b for a, b in plan)
        if r1 - r0 >= 2:
            assert len(plan) == 2 and plan[1][1] - plan[1][0] <= plan[0][1] - plan[0][0]
    assert plan_row_bands(0, 2160, 4) == [(0, 1890), (1890, 2160)]
    assert plan_row_bands(0, 2160, 4, width=3840) == [(0, 1890), (1890, 2160)]
    assert plan_row_bands(0, 256, 4, width=256) == [(0, 256)]  # small frames: one band


def test_delaunay_degenerate_inputs():
    """Robust host preprocessing (reference mesh.py:419-467): exact
    collinearity test, every vertex triangulated, and exactly cocircular
    lattices flagged (the triangulation is not unique there; Qhull's tie-break
    may differ from the reference's Bowyer-Watson insertion order)."""
    import warnings

    with pytest.raises(mesh.DegenerateInput):
        mesh.delaunay(np.column_stack([np.arange(6.0), 3.0 * np.arange(6.0) + 1.0]))
    # nearly collinear but not exactly: triangulates, or fails as a MeshError (never a raw QhullError)
    pts = np.column_stack([np.arange(6.0), np.zeros(6)])
    pts[3, 1] = 1e-12
    m = mesh.delaunay(pts)
    assert len(np.unique(m.triangles)) == 6
    pts[3, 1] = 1e-300
    with pytest.raises(mesh.MeshError):
        mesh.delaunay(pts)
    xs, ys = np.meshgrid(np.arange(5.0), np.arange(4.0))
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        m = mesh.delaunay(np.column_stack([xs.ravel(), ys.ravel()]))
    assert any("cocircular" in str(x.message) for x in w)
    assert len(np.unique(m.triangles)) == 20 and (m.signed_areas() > 0).all()
    rng = np.random.default_rng(0)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        mesh.delaunay(rng.normal(size=(500, 2)))
