"""Layout parity on the GPU: teacher-forced steps against the
reference's own trajectory, free-running K <= 5, exact invariants."""
import numpy as np
import pytest
import torch

import oracle as O
from conftest import layout_params, normwise
from helpers import golden_mesh

from paper_1408_0677_b200 import bhtree, layout as L

pytestmark = pytest.mark.gpu

TF_TOL = 1e-12      # teacher-forced per step
FREE_TOL = 1e-9     # free-running, K = 5


def _params(g, iterations=50):
    p = layout_params(g)
    return L.LayoutParams(iterations=iterations, **{k: p[k] for k in (
        "repulsion_c", "spring_scale", "desired_edge_d", "softening_eta", "initial_temp",
        "decay_lambda", "bh_theta")})


def test_teacher_forced_every_step_c1(c1):
    m = golden_mesh(c1)
    p = _params(c1)
    st, T = c1["states"], c1["temps"]
    worst = 0.0
    for k in range(len(st) - 1):
        m.current_pos = st[k].copy()
        nxt = L.layout_step(L.LayoutState(m, k, float(T[k]), st[k]), p)
        worst = max(worst, normwise(nxt.relaxed_pos, st[k + 1]))
        assert nxt.temperature == T[k + 1]
    assert worst <= TF_TOL, worst


@pytest.mark.parametrize("scene", ["g2k", "g10k"])
def test_teacher_forced_larger(scene, request):
    g = request.getfixturevalue(scene)
    m = golden_mesh(g)
    p = _params(g)
    st, T = g["states"], g["temps"]
    its = list(g["state_iters"]) if "state_iters" in g.files else list(range(len(st)))
    for a in range(len(its) - 1):
        if its[a + 1] != its[a] + 1:
            continue
        m.current_pos = st[a].copy()
        nxt = L.layout_step(L.LayoutState(m, its[a], float(T[a]), st[a]), p)
        assert normwise(nxt.relaxed_pos, st[a + 1]) <= TF_TOL, (scene, its[a])


def test_free_running_5_steps(c1, g2k):
    for g in (c1, g2k):
        m = golden_mesh(g)
        p = _params(g, iterations=5)
        state = L.layout_run(m, p)
        assert normwise(state.relaxed_pos, g["states"][5]) <= FREE_TOL
        assert state.temperature == pytest.approx(g["temps"][5], rel=1e-15)


def test_components_teacher_forced(c1):
    m = golden_mesh(c1)
    p = _params(c1)
    for k in (0, 25):
        new, bh, force, s = L.layout_debug_step(m, c1["states"][k], p, float(c1["temps"][k]))
        assert normwise(bh, c1[f"bh_{k}"]) <= 1e-13
        assert normwise(force, c1[f"total_{k}"]) <= 1e-13
        assert normwise(new, c1["states"][k + 1]) <= TF_TOL


def test_bh_matches_reference_and_exact(g2k, g10k):
    p = layout_params(g2k)
    got = bhtree.repulsive_forces(g2k["states"][0], p["repulsion_c"], p["softening_eta"], p["bh_theta"])
    assert normwise(got, g2k["bh_0"]) <= 1e-13
    ex = g2k["bh_exact_0"]
    rel = np.linalg.norm(got - ex, axis=1) / np.linalg.norm(ex, axis=1)
    assert rel.max() < 0.05
    p = layout_params(g10k)
    got = bhtree.repulsive_forces(g10k["states"][3], p["repulsion_c"], p["softening_eta"], p["bh_theta"])
    assert normwise(got, g10k["bh_30"]) <= 1e-13


def test_kdtree_membership_matches_oracle(g2k):
    pts = g2k["states"][2]
    gt = bhtree.KdTree(pts, leaf_size=32)
    ot = O.KdTree(pts, leaf_size=32)
    nn = ot.count
    assert gt._count == nn
    for arr in ("lo", "hi", "left", "right"):
        assert np.array_equal(getattr(gt, arr)[:nn], getattr(ot, arr)[:nn]), arr
    for i in range(nn):
        a = set(gt.perm[gt.lo[i]:gt.hi[i]].tolist())
        b = set(ot.perm[ot.lo[i]:ot.hi[i]].tolist())
        assert a == b, i
    assert np.array_equal(gt.bmin, ot.bmin[:nn]) and np.array_equal(gt.bmax, ot.bmax[:nn])
    # CUDA hypot vs glibc hypot: within 1 ulp
    assert np.allclose(gt.size, ot.size[:nn], rtol=4e-16, atol=0)
    assert np.abs(gt.com - ot.com[:nn]).max() <= 1e-14 * np.abs(pts).max()


def test_barnes_hut_coincident_points_finite():
    pts = np.array([[0.0, 0.0], [0.0, 0.0], [1.0, 1.0]])
    f = bhtree.repulsive_forces(pts, c=1.0, eta=1e-6, theta=0.5)
    assert np.all(np.isfinite(f))


def test_planarity_and_temperature_full_run(c1):
    m = golden_mesh(c1)
    p = _params(c1, iterations=500)
    signs0 = np.sign(m.signed_areas(m.original_pos))
    state = L.layout_run(m, p)
    assert np.array_equal(np.sign(m.signed_areas(state.relaxed_pos)), signs0)
    t = p.initial_temp
    for _ in range(500):
        t = t * p.decay_lambda
    assert state.temperature == t


def test_planarity_under_stress_every_step():
    from paper_1408_0677_b200 import mesh as M

    rng = np.random.default_rng(123)
    pts = np.round(rng.uniform(0, 8, size=(120, 2)) * 2) / 2  # heavy overplot
    m = M.delaunay(pts, seed=3)
    p = L.LayoutParams.defaults_for(m, iterations=150)
    signs0 = np.sign(m.signed_areas(m.original_pos))
    state = L.initial_state(m, p)
    for _ in range(150):
        state = L.layout_step(state, p)
        assert np.all(np.sign(m.signed_areas()) == signs0)


def test_eta_clearance_after_own_move():
    """test_layout.py:170-187 restated against the GPU step."""
    from paper_1408_0677_b200 import mesh as M

    rng = np.random.default_rng(17)
    m = M.delaunay(rng.uniform(0, 5, (60, 2)), seed=0)
    p = L.LayoutParams.defaults_for(m, iterations=30)
    state = L.initial_state(m, p)
    tris = m.triangles
    for _ in range(30):
        before = m.current_pos.copy()
        state = L.layout_step(state, p)
        a, b, c = before[tris[:, 0]], before[tris[:, 1]], before[tris[:, 2]]
        mab, mbc, mca = 0.5 * (a + b), 0.5 * (b + c), 0.5 * (c + a)
        for pt, dr in ((mab, mca - mab), (mab, mbc - mab), (mbc, mca - mbc)):
            nrm = np.stack([-dr[:, 1], dr[:, 0]], axis=1)
            nrm /= np.hypot(nrm[:, 0], nrm[:, 1])[:, None]
            for k in range(3):
                v = tris[:, k]
                old = np.einsum("ij,ij->i", before[v] - pt, nrm)
                new = np.einsum("ij,ij->i", m.current_pos[v] - pt, nrm)
                side = np.where(old >= 0, 1.0, -1.0)
                approached = new * side < old * side - 1e-15
                assert np.all((new * side)[approached] >= p.softening_eta - 1e-12)


def test_graph_and_eager_paths_agree(g2k):
    m = golden_mesh(g2k)
    p = _params(g2k, iterations=5)
    eng = L.LayoutEngine(m, p)
    temps = L.temperature_schedule(p.initial_temp, p.decay_lambda, 5)
    eng.set_positions(g2k["states"][0])
    eng.run(temps, use_graph=True)
    a = eng.pos.clone()
    eng.set_positions(g2k["states"][0])
    eng.run(temps, use_graph=False)
    assert torch.equal(a, eng.pos)


def test_vertex_partition_reassembles_bit_identically(g2k):
    """Config-4 multi-GPU layout, emulated on one GPU: the ranks' partial steps
    (each owns a leaf-order slice, writes 0.0 elsewhere) summed == full step,
    for 5 chained iterations (1-GPU vs N-GPU bit-identical)."""
    m = golden_mesh(g2k)
    p = _params(g2k, iterations=5)
    temps = L.temperature_schedule(p.initial_temp, p.decay_lambda, 5)
    full = L.LayoutEngine(m, p)
    parts = [L.LayoutEngine(m, p, part=(r, 3)) for r in range(3)]
    pos = torch.as_tensor(g2k["states"][0]).cuda()
    full.pos.copy_(pos)
    for it in range(5):
        full.run(temps[it:it + 1], use_graph=False)
        acc = torch.zeros_like(pos)
        for e in parts:
            e.pos.copy_(pos)
            e.run(temps[it:it + 1], use_graph=False)
            acc += e.pos
        pos = acc
        assert torch.equal(pos, full.pos), it
    assert normwise(pos.cpu().numpy(), g2k["states"][5]) <= FREE_TOL


@pytest.mark.parametrize("kind,n", [("float_collisions", 20000), ("long_run", 20000), ("float_collisions", 3000),
                                    ("signed_zero", 5000), ("constant_x", 4000), ("outlier_cluster", 20000)])
def test_kdtree_device_sort_exact_order(kind, n):
    """The device sort (bucket ranks, MDC_SORT_BUCKET) must give the exact
    (coord, id) order whatever the distribution: distinct doubles sharing a
    float, exact ties, -0.0 vs +0.0, a constant column (one bucket), a far
    outlier squeezing the rest into a few buckets -- checked through the
    kd-tree membership against the oracle."""
    rng = np.random.default_rng(7)
    y = rng.normal(0, 3, n)
    if kind == "float_collisions":
        base = rng.normal(0, 3, n // 8)
        x = np.repeat(base, 8) * (1 + rng.integers(-3, 4, n) * 2.0 ** -45)  # same float, distinct doubles
        x[::97] = x[0]  # exact ties as well
    elif kind == "long_run":
        x = 1.0 + rng.integers(0, 4000, n) * 2.0 ** -40  # one float key, a 20000-long run
        y = rng.normal(0, 1, n)
    elif kind == "signed_zero":
        x = rng.normal(0, 1, n)
        x[rng.integers(0, n, n // 4)] = 0.0
        x[rng.integers(0, n, n // 4)] = -0.0
        y[::3] = -0.0
    elif kind == "constant_x":
        x = np.full(n, 0.75)
    else:
        x = rng.normal(0, 1e-3, n)
        x[123] = 1e6
        y[77] = -1e9
    pts = np.column_stack([x, y])
    gt = bhtree.KdTree(pts, leaf_size=32)
    ot = O.KdTree(pts, leaf_size=32)
    nn = ot.count
    for arr in ("lo", "hi", "left", "right"):
        assert np.array_equal(getattr(gt, arr)[:nn], getattr(ot, arr)[:nn]), arr
    for i in range(nn):
        assert set(gt.perm[gt.lo[i]:gt.hi[i]].tolist()) == set(ot.perm[ot.lo[i]:ot.hi[i]].tolist()), i
    assert np.array_equal(gt.bmin, ot.bmin[:nn]) and np.array_equal(gt.bmax, ot.bmax[:nn])


def test_teacher_forced_at_bench_scale():
    """The bench workload itself (config 3: 100k GMM points, PCA projection,
    Delaunay mesh): GPU steps against the fp64 oracle restatement at steps 0,
    1 and 250 of a GPU trajectory (teacher-forced: both take the same input
    state), <= 1e-12 normwise; plus zero orientation flips after 250 steps."""
    import bench

    cfg = bench.CONFIGS[3]
    ds, mesh, raw = bench.build_scene(cfg)
    params = L.LayoutParams.defaults_for(mesh, iterations=500)
    p = {k: getattr(params, k) for k in ("repulsion_c", "spring_scale", "desired_edge_d", "softening_eta",
                                         "bh_theta", "initial_temp", "decay_lambda")}
    temps = L.temperature_schedule(params.initial_temp, params.decay_lambda, 251)
    eng = L.LayoutEngine(mesh, params)
    eng.set_positions(mesh.original_pos)
    states = {0: mesh.original_pos.copy()}
    eng.run(temps[:1])
    states[1] = eng.pos.cpu().numpy()
    eng.run(temps[1:250])
    states[250] = eng.pos.cpu().numpy()
    signs0 = np.sign(mesh.signed_areas(mesh.original_pos))
    assert np.array_equal(np.sign(mesh.signed_areas(states[250])), signs0)
    for k in (0, 1, 250):
        eng.set_positions(states[k])
        eng.run(temps[k:k + 1], use_graph=False)
        got = eng.pos.cpu().numpy()
        ref = O.layout_step(states[k], mesh.csr_offsets, mesh.csr_targets, mesh.triangles, p, float(temps[k]))
        assert normwise(got, ref) <= TF_TOL, (k, normwise(got, ref))


@pytest.fixture(scope="module")
def g10k_traj():
    from conftest import load_golden

    return load_golden("g10k_traj")


def test_teacher_forced_500_step_reference_trajectory(g10k, g10k_traj):
    """SURVEY.md §8c(i) at config 2: the reference's own 500-step layout_run
    (layout.py:298-302, tests/golden/make_golden.py --traj) -- the GPU step
    applied to reference state k matches reference state k+1 (<= 1e-12
    normwise) for k in {0..4, 49, 99, 199, 299, 399, 498}, with the exact
    temperature; and the 500-step temperature is lambda^500 t_i."""
    m = golden_mesh(g10k)
    p = _params(g10k, iterations=500)
    its = list(g10k_traj["state_iters"])
    st, T = g10k_traj["states"], g10k_traj["temps"]
    worst = {}
    for k in g10k_traj["pairs"]:
        a, b = its.index(k), its.index(k + 1)
        m.current_pos = st[a].copy()
        nxt = L.layout_step(L.LayoutState(m, int(k), float(T[a]), st[a]), p)
        worst[int(k)] = normwise(nxt.relaxed_pos, st[b])
        assert nxt.temperature == T[b]
    print("teacher-forced 500-step trajectory:", worst)
    assert max(worst.values()) <= TF_TOL, worst
    temps = L.temperature_schedule(p.initial_temp, p.decay_lambda, 500)
    assert float(temps[-1]) * p.decay_lambda == pytest.approx(float(g10k_traj["final_temp"]), rel=1e-12)


def test_free_running_5_steps_config2(g10k, g10k_traj):
    """SURVEY.md §8c(ii) at config 2 (10k): 5 free-running GPU steps from the
    reference's state 0 against the reference's state 5, <= 1e-9 normwise."""
    m = golden_mesh(g10k)
    p = _params(g10k, iterations=5)
    its = list(g10k_traj["state_iters"])
    state = L.layout_run(m, p)
    err = normwise(state.relaxed_pos, g10k_traj["states"][its.index(5)])
    print("free-running 5 steps at 10k:", err)
    assert err <= FREE_TOL


@pytest.mark.parametrize("scene", ["c1", "g2k"])
def test_small_mesh_persistent_step_bit_identical(scene, request):
    """n <= 2048 runs every step of a call in one persistent CTA
    (layout_small_kernel: exact ranks, one-CTA walk, BH, combine, local
    update between block barriers).  It must equal the multi-kernel step
    (use_graph=False: the launch-per-phase path) bit for bit over 12 steps."""
    g = request.getfixturevalue(scene)
    m = golden_mesh(g)
    p = _params(g, iterations=12)
    temps = L.temperature_schedule(p.initial_temp, p.decay_lambda, 12)
    fused, multi = L.LayoutEngine(m, p), L.LayoutEngine(m, p)
    fused.set_positions(m.original_pos)
    multi.set_positions(m.original_pos)
    fused.run(temps, use_graph=True)
    multi.run(temps, use_graph=False)
    assert np.array_equal(fused.pos.cpu().numpy(), multi.pos.cpu().numpy())
    one = L.LayoutEngine(m, p)  # odd step counts end in the other buffer
    one.set_positions(m.original_pos)
    one.run(temps[:5], use_graph=True)
    multi.set_positions(m.original_pos)
    multi.run(temps[:5], use_graph=False)
    assert np.array_equal(one.pos.cpu().numpy(), multi.pos.cpu().numpy())
