"""One consolidated, measured parity table over SURVEY.md §8(a)'s rows.

Each entry recomputes the GPU result and its reference (golden vectors the
reference produced, or the pinned oracle restatement), records the observed
error next to the contract, and asserts the contract.  Run with -s to see the
table (the round's copy is committed as profiles/r01_parity_report.txt)."""
import json

import numpy as np
import pytest

import oracle as O
from conftest import layout_params, normwise
from helpers import golden_mesh
from test_gpu_mls import _targets

from paper_1408_0677_b200 import bhtree, field as F, layout as L, projection as P, render as R
from paper_1408_0677_b200 import dataset as D

pytestmark = pytest.mark.gpu


def _lp(g, iterations):
    p = layout_params(g)
    return L.LayoutParams(iterations=iterations, **{k: p[k] for k in (
        "repulsion_c", "spring_scale", "desired_edge_d", "softening_eta", "initial_temp", "decay_lambda",
        "bh_theta")})


def test_parity_report(c1, g10k, cars):
    rows = []

    def add(row, what, observed, contract, ok=None):
        ok = (observed <= contract) if ok is None else ok
        rows.append({"row": row, "check": what, "observed": float(observed), "contract": contract, "ok": bool(ok)})

    # ---- M4-M8: fields vs the reference's own (golden) fields -------------
    m = golden_mesh(c1)
    pos = c1["field_positions"]
    W, H = (int(v) for v in c1["field_wh"])
    for dtype, tol in (("f64", 1e-10), ("f32", 1e-4)):
        worst = 0.0
        for name, var, a in zip(c1["field_cases"], c1["field_variants"], c1["field_alphas"]):
            if str(var) == "linear":
                continue
            params = F.MlsParams(variant=str(var), alpha=None if np.isnan(a) else float(a))
            fld = F.compute_field(m, pos, _targets(c1, name), params, W, H, dtype=dtype)
            ref = c1[f"field_{name}"]
            worst = max([worst] + [normwise(fld.coords[..., k], ref[..., k]) for k in range(2)
                                   if np.abs(ref[..., k]).max() > 0])
        add("M4-M8", f"compute_field mean/affine/rigid (+generic alpha) vs golden, {dtype}, max normwise", worst, tol)

    # ---- M6': fused fp32 (tcgen05) at the bench scale vs the oracle ---------
    import bench

    cfg = bench.CONFIGS[3]
    X = bench.gmm(cfg["n"], cfg["d"], cfg["seed"])
    ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(cfg["d"])], data=X))
    _, cloud = P.pca_project(ds)
    raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])
    Wb, Hb = cfg["W"], cfg["H"]
    worst = 0.0
    for r0, r1 in ((0, 2), (Hb // 2, Hb // 2 + 2), (Hb - 2, Hb)):
        v = F.compute_fields(cloud.positions, raw, F.MlsParams("affine"), Wb, Hb, dtype="f32",
                             row_range=(r0, r1)).values.double().cpu().numpy()
        ref = O.compute_field(cloud.positions, raw[:, [0, 31]], "affine", Wb, Hb, rows=(r0, r1))
        worst = max(worst, normwise(v[0], ref[..., 0]), normwise(v[31], ref[..., 1]))
    add("M6'", "fused fp32 tcgen05 field, config 3 (4K, N=100k, d=32), 3 row bands, max normwise", worst, 1e-4)

    # ---- M9 snap: exact; M11 bands: exact outside eps ------------------------
    tv = c1["targets_affine_proj"]
    eps = (2.0 * max(F.ViewportTransform.fit(pos, W, H).units_per_px)) ** 2
    fld = F.compute_field(m, pos, F.TargetAssignment(tv, "projection"),
                          F.MlsParams(variant="affine", epsilon_dist=eps), W, H)
    ref = O.compute_field(pos, tv, "affine", W, H, epsilon_dist=eps)
    snapped = np.zeros((H, W), bool)
    for q in tv:
        snapped |= np.all(ref == q, axis=-1)
    add("M9", f"snapped pixels differing from the reference ({int(snapped.sum())} snapped)",
        int((fld.coords[snapped] != ref[snapped]).any(-1).sum()), 0)
    spacing = np.array([float(c1[f"spacing_affine_dim{k}"]) for k in range(4)])
    for dtype, e in (("f64", 1e-9), ("f32", 1e-4)):
        blk = F.compute_fields(pos, c1["raw"], F.MlsParams("affine"), W, H, dtype=dtype, band_spacing=spacing)
        bands = blk.bands.cpu().numpy()
        bad = 0
        for k in range(4):
            r = c1[f"field_affine_dim{k}"][..., 0]
            ok = np.abs(r / spacing[k] - np.round(r / spacing[k])) > e
            bad += int((bands[k][ok] != c1[f"bands_affine_dim{k}"][ok]).sum())
        add("M11", f"band indices differing outside eps={e} ({dtype})", bad, 0)

    # ---- linear variant: bit-exact -----------------------------------------
    bad = 0
    for name in ("linear_dim0", "linear_proj", "linear_dims13"):
        f = F.compute_field(m, pos, _targets(c1, name), F.MlsParams("linear"), W, H)
        bad += int((f.coords != c1[f"field_{name}"]).sum())
    add("(f) linear", "linear-variant values differing from golden (bit-exact)", bad, 0)

    # ---- M10-M12 render: RGBA vs the restated reference ----------------------
    worst_d, frac = 0, 0.0
    for mode in ("contour", "discrete", "discrete+contour"):
        for name in ("affine_dim0", "rigid_dims01", "affine_proj"):
            f = F.compute_field(m, pos, _targets(c1, name), F.MlsParams(str(name.split("_")[0])), W, H)
            sp = float(c1[f"spacing_{name}"]) if f"spacing_{name}" in c1.files else 0.5
            diff = np.abs(R.render(f, R.RenderSpec(mode=mode, spacing=sp)).pixels.astype(int)
                          - O.render_rgba(f.coords, f.active_channels, sp, mode).astype(int))
            worst_d, frac = max(worst_d, int(diff.max())), max(frac, float((diff > 0).mean()))
    add("M10-M12", "RGBA8 render vs restated reference: max |diff| (8-bit levels)", worst_d, 1)
    add("M10-M12", "RGBA8 render vs restated reference: fraction of channels differing by 1", frac, 1e-3)

    # ---- L3-L10 layout --------------------------------------------------------
    p = _lp(c1, 50)
    st, T = c1["states"], c1["temps"]
    worst = 0.0
    for k in range(len(st) - 1):
        m.current_pos = st[k].copy()
        nxt = L.layout_step(L.LayoutState(m, k, float(T[k]), st[k]), p)
        worst = max(worst, normwise(nxt.relaxed_pos, st[k + 1]))
    add("L3-L10", f"teacher-forced step vs golden, N=150, all {len(st) - 1} steps, max normwise", worst, 1e-12)
    mg = golden_mesh(g10k)
    pg = _lp(g10k, 50)
    its = list(g10k["state_iters"])
    worst = 0.0
    for a in range(len(its) - 1):
        if its[a + 1] == its[a] + 1:
            mg.current_pos = g10k["states"][a].copy()
            nxt = L.layout_step(L.LayoutState(mg, its[a], float(g10k["temps"][a]), g10k["states"][a]), pg)
            worst = max(worst, normwise(nxt.relaxed_pos, g10k["states"][a + 1]))
    add("L3-L10", "teacher-forced step vs golden, N=10k, max normwise", worst, 1e-12)
    m5 = golden_mesh(c1)
    s5 = L.layout_run(m5, _lp(c1, 5))
    add("L3", "free-running 5 steps vs golden, N=150, normwise", normwise(s5.relaxed_pos, st[5]), 1e-9)
    pts = g10k["states"][0]
    gt, ot = bhtree.KdTree(pts, leaf_size=32), O.KdTree(pts, leaf_size=32)
    nn = ot.count
    differ = sum(set(gt.perm[gt.lo[i]:gt.hi[i]].tolist()) != set(ot.perm[ot.lo[i]:ot.hi[i]].tolist())
                 for i in range(nn))
    add("L4", f"kd-tree nodes whose membership differs from the oracle ({nn} nodes)", differ, 0)
    lp = layout_params(c1)
    bh = bhtree.repulsive_forces(st[0], lp["repulsion_c"], lp["softening_eta"], lp["bh_theta"])
    add("L5", "Barnes-Hut forces vs golden, normwise", normwise(bh, c1["bh_0"]), 1e-13)

    # ---- P1 PCA -----------------------------------------------------------------
    dsc = D.Dataset(names=[f"c{i}" for i in range(cars["ds_data"].shape[1])], data=cars["ds_data"])
    model, _ = P.pca_project(dsc)
    add("P1", "PCA eigenvalues vs golden, normwise", normwise(model.eigenvalues, cars["pca_eigenvalues"]), 1e-9)
    add("P1", "PCA axes vs golden, max abs", float(np.abs(model.axes - cars["pca_axes"]).max()), 1e-9)

    width = max(len(r["check"]) for r in rows)
    print()
    for r in rows:
        print(f"{r['row']:11s} {r['check']:{width}s} observed {r['observed']:.3e}  contract {r['contract']:.0e}  "
              f"{'ok' if r['ok'] else 'FAIL'}")
    print(json.dumps(rows))
    assert all(r["ok"] for r in rows), [r for r in rows if not r["ok"]]
