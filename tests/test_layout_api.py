"""The rest of the reference's layout / mesh API surface (layout.py:87-116,
160-213, 259-263, 323-350; mesh.py:157-217): the scalar force laws, the
single-node clamp, the text dumps (CPU), and clamp_factors / total_forces on
the GPU against the oracle and the golden component forces.  Ported from the
reference's test_layout.py closed-form cases."""
import numpy as np
import pytest

import oracle as O
from conftest import layout_params, normwise
from helpers import golden_mesh

from paper_1408_0677_b200 import layout as L
from paper_1408_0677_b200 import mesh as M


def _params(**kw):
    base = dict(repulsion_c=1.0, spring_scale=1.0, desired_edge_d=1.0, softening_eta=1e-7, initial_temp=1.0,
                decay_lambda=0.99, bh_theta=0.5, iterations=10)
    base.update(kw)
    return L.LayoutParams(**base)


def test_repulsive_force_law():
    p = _params()
    f = L.repulsive_force((1.0, 0.0), (0.0, 0.0), p)
    assert f[0] == pytest.approx(1.0 / (1.0 + 1e-7)) and f[1] == 0.0
    f2 = L.repulsive_force((2.0, 0.0), (0.0, 0.0), p)
    assert f2[0] == pytest.approx(f[0] / 4.0, rel=1e-6)          # inverse square
    assert np.all(np.isfinite(L.repulsive_force((0.0, 0.0), (0.0, 0.0), p)))


def test_spring_force_law():
    p = _params(desired_edge_d=2.0, softening_eta=1e-12)
    assert np.allclose(L.spring_force((2.0, 0.0), (0.0, 0.0), p), 0.0)   # rest length
    assert L.spring_force((3.0, 0.0), (0.0, 0.0), p)[0] < 0.0             # stretched: attracts
    assert L.spring_force((1.0, 0.0), (0.0, 0.0), p)[0] > 0.0             # compressed: repels
    assert np.array_equal(L.spring_force((0.0, 0.0), (0.0, 0.0), p), np.zeros(2))


def test_node_edge_force_law():
    p = _params(softening_eta=1e-12)
    f1 = L.node_edge_force((0.0, 1.0), (-1.0, 0.0), (1.0, 0.0), p)
    f2 = L.node_edge_force((0.0, 2.0), (-1.0, 0.0), (1.0, 0.0), p)
    assert f1[1] > 0.0 and f1[0] == pytest.approx(0.0)                   # away from the edge
    assert f2[1] == pytest.approx(f1[1] / 4.0)                             # inverse square
    assert np.array_equal(L.node_edge_force((0.5, 0.0), (-1.0, 0.0), (1.0, 0.0), p), np.zeros(2))


def _one_triangle():
    pts = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    return M.assemble(pts, pts.copy(), np.array([[0, 1, 2]]))


def test_clamp_displacement_single_node():
    mesh = _one_triangle()
    p = _params(softening_eta=1e-12)
    assert np.array_equal(L.clamp_displacement(0, (0.0, 0.0), mesh, p), np.zeros(2))
    # moving vertex 0 toward (1, 1): the mid-line through (0.5, 0) and (0, 0.5)
    # is at distance sqrt(2)/4; a displacement of length sqrt(2)/2 is halved
    d = L.clamp_displacement(0, (0.5, 0.5), mesh, p)
    assert np.allclose(d, [0.25, 0.25])
    # moving away from every line is unchanged
    assert np.allclose(L.clamp_displacement(0, (-0.3, -0.2), mesh, p), [-0.3, -0.2])


def test_mesh_and_layout_text_round_trip(c1):
    m = golden_mesh(c1)
    m2 = M.parse_mesh_text(m.dump_text())
    for f in ("original_pos", "current_pos", "csr_offsets", "csr_targets", "fan_offsets", "fan_nodes", "triangles"):
        assert np.array_equal(getattr(m, f), getattr(m2, f)), f
    st = L.LayoutState(mesh=m, iteration=7, temperature=0.123456789, relaxed_pos=c1["states"][7])
    st2 = L.parse_layout_text(L.dump_layout_text(st))
    assert st2.iteration == 7 and st2.temperature == st.temperature
    assert np.array_equal(st2.relaxed_pos, st.relaxed_pos)
    def canon(t):
        k = int(np.argmin(t))
        return tuple(int(t[(k + j) % 3]) for j in range(3))

    assert sorted(m.node_triangles(0)) == sorted(canon(t) for t in m.triangles if 0 in t)
    with pytest.raises(M.MeshError):
        M.parse_mesh_text("grid 1 2\n")


@pytest.mark.gpu
def test_clamp_factors_matches_oracle(c1):
    m = golden_mesh(c1)
    lp = layout_params(c1)
    rng = np.random.default_rng(3)
    pos = c1["states"][10]
    disp = rng.normal(0, 2.0 * lp["desired_edge_d"], pos.shape)
    got = L.clamp_factors(pos, disp, m.triangles, lp["softening_eta"])
    ref = O.clamp_factors(pos, disp, m.triangles, lp["softening_eta"])
    # CUDA hypot may differ from glibc's in the last ulp (DESIGN.md "Known
    # deviations"): same clamped set, factors to ~1e-15
    assert np.array_equal(got < 1.0, ref < 1.0)
    assert np.abs(got - ref).max() <= 1e-13
    assert (got < 1.0).any()


@pytest.mark.gpu
def test_total_forces_matches_golden(c1):
    m = golden_mesh(c1)
    p = layout_params(c1)
    params = L.LayoutParams(iterations=1, **{k: p[k] for k in (
        "repulsion_c", "spring_scale", "desired_edge_d", "softening_eta", "initial_temp", "decay_lambda",
        "bh_theta")})
    for k in (0, 25):
        assert normwise(L.total_forces(c1["states"][k], m, params), c1[f"total_{k}"]) <= 1e-13


def test_triangle_neighbors_matches_brute_force(c1):
    from paper_1408_0677_b200 import field as F

    tris = golden_mesh(c1).triangles
    got = F.triangle_neighbors(tris)
    for t, (a, b, c) in enumerate(tris):
        for k, edge in enumerate(({b, c}, {c, a}, {a, b})):
            others = [u for u in range(len(tris)) if u != t and edge <= set(tris[u].tolist())]
            assert got[t, k] == (others[0] if others else -1)
