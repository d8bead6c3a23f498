"""The CPU oracle (oracle/) pinned against vectors produced by the reference
itself (tests/golden/make_golden.py).  No GPU needed."""
import numpy as np
import pytest

import oracle as O
from conftest import layout_params, normwise


def test_oracle_mls_fields_bit_exact(c1):
    pos = c1["field_positions"]
    W, H = (int(v) for v in c1["field_wh"])
    for name, var, a in zip(c1["field_cases"], c1["field_variants"], c1["field_alphas"]):
        got = O.compute_field(pos, c1[f"targets_{name}"], str(var), W, H,
                              alpha=None if np.isnan(a) else float(a), tris=c1["triangles"])
        # numba kernels and the C restatement perform the same IEEE sequence
        assert np.array_equal(got, c1[f"field_{name}"]), name


def test_oracle_linear_larger(g2k):
    got = O.compute_field(g2k["field_positions"], g2k["targets_affine_dim0"], "linear", 120, 90,
                          tris=g2k["triangles"])
    assert np.array_equal(got, g2k["field_linear_dim0"])


def test_oracle_bands_and_coverage(c1):
    for name in c1["field_cases"]:
        if f"bands_{name}" not in c1.files:
            continue
        coords = c1[f"field_{name}"]
        sp = float(c1[f"spacing_{name}"])
        assert O.auto_spacing(c1[f"targets_{name}"][:, 0]) == sp
        assert np.array_equal(O.band_indices(coords, sp, 1), c1[f"bands_{name}"])
        assert np.array_equal(O.line_coverage(coords, sp, 1.5, 1), c1[f"coverage_{name}"])


def test_oracle_layout_teacher_forced_all_steps(c1):
    p = layout_params(c1)
    st, T = c1["states"], c1["temps"]
    for k in range(len(st) - 1):
        nxt = O.layout_step(st[k], c1["csr_offsets"], c1["csr_targets"], c1["triangles"], p, T[k])
        assert normwise(nxt, st[k + 1]) <= 1e-13, k


def test_oracle_layout_free_running(c1):
    p = layout_params(c1)
    pos, t = O.layout_run(c1["states"][0], c1["csr_offsets"], c1["csr_targets"], c1["triangles"], p, 5)
    assert normwise(pos, c1["states"][5]) <= 1e-12
    assert t == pytest.approx(c1["temps"][5], rel=1e-15)


def test_oracle_force_components(c1):
    p = layout_params(c1)
    for k in (0, 25):
        pos = c1["states"][k]
        bh = O.repulsive_forces(pos, p["repulsion_c"], p["softening_eta"], p["bh_theta"])
        assert normwise(bh, c1[f"bh_{k}"]) <= 1e-14
        sp = O.spring_forces(pos, c1["csr_offsets"], c1["csr_targets"], p["spring_scale"],
                             p["softening_eta"], p["desired_edge_d"])
        assert normwise(sp, c1[f"spring_{k}"]) <= 1e-14
        ne = O.node_edge_forces(pos, c1["triangles"], p["repulsion_c"], p["softening_eta"])
        assert np.array_equal(ne, c1[f"nodeedge_{k}"])
        cf = O.clamp_factors(pos, c1[f"clampdisp_{k}"], c1["triangles"], p["softening_eta"])
        assert np.array_equal(cf, c1[f"clamp_{k}"])
    ex = O.repulsive_forces_exact(c1["states"][0], p["repulsion_c"], p["softening_eta"])
    assert normwise(ex, c1["bh_exact_0"]) <= 1e-13


@pytest.mark.parametrize("scene", ["g2k", "g10k"])
def test_oracle_layout_larger_scenes(scene, request):
    g = request.getfixturevalue(scene)
    p = layout_params(g)
    st, T = g["states"], g["temps"]
    its = list(g["state_iters"]) if "state_iters" in g.files else list(range(len(st)))
    checked = 0
    for a in range(len(its) - 1):
        if its[a + 1] != its[a] + 1:
            continue
        nxt = O.layout_step(st[a], g["csr_offsets"], g["csr_targets"], g["triangles"], p, T[a])
        assert normwise(nxt, st[a + 1]) <= 1e-13
        checked += 1
    assert checked >= 2


def test_oracle_pca(c1, cars):
    for g in (c1, cars):
        mean, axes, ev, pos = O.pca_project(g["ds_data"])
        assert normwise(ev, g["pca_eigenvalues"]) <= 1e-12
        assert np.abs(axes - g["pca_axes"]).max() <= 1e-12
        assert np.abs(pos - g["pca_positions"]).max() <= 1e-11


def test_oracle_bh_vs_exact_within_5_percent(g2k):
    p = layout_params(g2k)
    pts = g2k["states"][0]
    bh = O.repulsive_forces(pts, p["repulsion_c"], p["softening_eta"], p["bh_theta"])
    ex = g2k["bh_exact_0"]
    rel = np.linalg.norm(bh - ex, axis=1) / np.linalg.norm(ex, axis=1)
    assert rel.max() < 0.05


def test_oracle_pinned_to_500_step_reference_trajectory(g10k):
    """The oracle's step against the reference's own 500-step config-2
    trajectory (tests/golden/g10k_traj.npz) at an early, a middle and the last
    stored pair (the GPU test checks every stored pair)."""
    from conftest import load_golden

    t = load_golden("g10k_traj")
    p = layout_params(g10k)
    its = list(t["state_iters"])
    for k in (0, 249 if 249 in its else 199, 498):
        a, b = its.index(k), its.index(k + 1)
        nxt = O.layout_step(t["states"][a], g10k["csr_offsets"], g10k["csr_targets"], g10k["triangles"], p,
                            t["temps"][a])
        assert normwise(nxt, t["states"][b]) <= 1e-13, k
