"""Generate the golden parity fixtures by running the UPSTREAM reference.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

Every array written here comes straight out of the reference package
(`mdcontour`, imported from a temp copy by ``refload.py``): PCA
(`projection.py:50-79`), Delaunay + CSR/fan assembly (`mesh.py:362-467`),
layout trajectories (`layout.py:266-302`), Barnes-Hut forces
(`bhtree.py:69-95`), the individual force/clamp passes (`layout.py:160-256`),
MLS fields via `compute_field` (`field.py:582-659`), band indices
(`render.py:135-139`) and contour coverage (`render.py:116-126`).
The fixtures are committed; tests and the oracle check against them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from refload import load_reference  # noqa: E402


def gmm(n, d, seed):
    """SURVEY.md Appendix A.1 Gaussian-mixture generator."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(0, 4, (8, d))
    scales = rng.uniform(0.5, 1.5, 8)
    lab = rng.integers(0, 8, n)
    return centers[lab] + rng.normal(0, 1, (n, d)) * scales[lab, None]


def make_cars_like(rows=300, seed=11):
    """Same generator as the reference's tests/conftest.py:8-23."""
    rng = np.random.default_rng(seed)
    cyl = rng.choice([3, 4, 5, 6, 8], size=rows, p=[0.02, 0.5, 0.02, 0.26, 0.2])
    disp = cyl * 40 + rng.normal(0, 25, rows)
    hp = disp * 0.55 + rng.normal(0, 12, rows)
    weight = 1600 + disp * 4.5 + rng.normal(0, 180, rows)
    accel = 28 - hp * 0.08 + rng.normal(0, 1.6, rows)
    mpg = 48 - weight * 0.008 + rng.normal(0, 2.5, rows)
    year = rng.integers(70, 83, rows)
    origin = rng.choice([1, 2, 3], size=rows, p=[0.62, 0.18, 0.2])
    names = ["mpg", "cylinders", "horsepower", "weight", "acceleration", "year", "origin"]
    return names, np.column_stack([mpg, cyl, hp, weight, accel, year, origin]).astype(float)


def mesh_arrays(m):
    return dict(
        original_pos=m.original_pos,
        triangles=m.triangles.astype(np.int64),
        csr_offsets=m.csr_offsets.astype(np.int64),
        csr_targets=m.csr_targets.astype(np.int64),
        fan_offsets=m.fan_offsets.astype(np.int64),
        fan_nodes=m.fan_nodes.astype(np.int64),
    )


def scene(R, X, seed_mesh, iterations, keep_states):
    D, P, M, L = R["dataset"], R["projection"], R["mesh"], R["layout"]
    names = [f"d{i}" for i in range(X.shape[1])]
    ds = D.normalize(D.Dataset(names=names, data=X))
    model, cloud = P.pca_project(ds)
    mesh = M.delaunay(cloud, seed=seed_mesh)
    params = L.LayoutParams.defaults_for(mesh, iterations=iterations)
    state = L.initial_state(mesh, params)
    states = {0: state.relaxed_pos.copy()}
    temps = {0: state.temperature}
    for it in range(1, iterations + 1):
        state = L.layout_step(state, params)
        if it in keep_states:
            states[it] = state.relaxed_pos.copy()
            temps[it] = state.temperature
    return ds, model, cloud, mesh, params, state, states, temps


def params_dict(p):
    return dict(
        repulsion_c=p.repulsion_c, spring_scale=p.spring_scale, desired_edge_d=p.desired_edge_d,
        softening_eta=p.softening_eta, initial_temp=p.initial_temp, decay_lambda=p.decay_lambda,
        bh_theta=p.bh_theta,
    )


TRAJ_PAIRS = (0, 1, 2, 3, 4, 49, 99, 199, 299, 399, 498)


def make_traj():
    """g10k_traj.npz: the reference's own 500-step layout_run at config 2
    (10000 x 16, seed 2 -- the g10k scene, same mesh), keeping the state pairs
    (k, k+1) for k in TRAJ_PAIRS (SURVEY.md §8c(i) teacher-forced parity)."""
    R = load_reference()
    X = gmm(10000, 16, 2)
    keep = set(TRAJ_PAIRS) | {k + 1 for k in TRAJ_PAIRS}
    ds, model, cloud, mesh, params, state, states, temps = scene(R, X, 0, 500, keep)
    g10k = np.load(os.path.join(HERE, "g10k.npz"))
    for k, v in mesh_arrays(mesh).items():
        assert np.array_equal(g10k[k], v), f"mesh differs from g10k.npz: {k}"
    iters = np.array(sorted(keep))
    out = dict(state_iters=iters, states=np.stack([states[k] for k in iters]),
               temps=np.array([temps[k] for k in iters]), pairs=np.array(TRAJ_PAIRS),
               final=state.relaxed_pos, final_temp=np.float64(state.temperature))
    path = os.path.join(HERE, "g10k_traj.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def main():
    if "--traj" in sys.argv:
        return make_traj()
    R = load_reference()
    F, Rn, L, B, C = R["field"], R["render"], R["layout"], R["bhtree"], R["cli"]
    out = {}

    # ---- scene c1: config 1 (150 x 4, seed 1, 50 iterations) -------------
    X = gmm(150, 4, 1)
    ds, model, cloud, mesh, params, state, states, temps = scene(R, X, 0, 50, set(range(51)))
    c1 = dict(X=X, ds_data=ds.data, pca_mean=model.mean, pca_axes=model.axes,
              pca_eigenvalues=model.eigenvalues, pca_positions=cloud.positions,
              pca_viewport=np.array(cloud.viewport), **mesh_arrays(mesh))
    c1["states"] = np.stack([states[k] for k in range(51)])
    c1["temps"] = np.array([temps[k] for k in range(51)])
    for k, v in params_dict(params).items():
        c1[f"lp_{k}"] = np.float64(v)
    # Component forces at state 0 and state 25 (teacher-forced pieces).
    for k in (0, 25):
        pos = states[k]
        mesh.current_pos = pos.copy()
        c1[f"bh_{k}"] = B.repulsive_forces(pos, params.repulsion_c, params.softening_eta, params.bh_theta)
        c1[f"spring_{k}"] = L._spring_forces(pos, mesh, params)
        c1[f"nodeedge_{k}"] = L._node_edge_forces(pos, mesh, params)
        c1[f"total_{k}"] = L.total_forces(pos, mesh, params)
        rng = np.random.default_rng(100 + k)
        disp = rng.normal(0, params.desired_edge_d, pos.shape)
        c1[f"clampdisp_{k}"] = disp
        c1[f"clamp_{k}"] = L.clamp_factors(pos, disp, mesh.triangles, params.softening_eta)
    c1["bh_exact_0"] = B.repulsive_forces_exact(states[0], params.repulsion_c, params.softening_eta)

    # MLS fields on the relaxed layout (interpolate_layout t=1), 64 x 48.
    mesh.current_pos = states[50].copy()
    positions = states[50]
    W, H = 64, 48
    raw = [ds.raw_column(n) for n in ds.names]
    c1["raw"] = np.column_stack(raw)
    c1["field_positions"] = positions
    c1["field_wh"] = np.array([W, H])
    cases = []
    for dim in range(4):
        cases.append((f"affine_dim{dim}", "affine", None, ("dims", (dim,))))
    cases += [
        ("mean_dim0", "mean", None, ("dims", (0,))),
        ("mean_dim2_a05", "mean", 0.5, ("dims", (2,))),
        ("affine_dim1_a13", "affine", 1.3, ("dims", (1,))),
        ("affine_dim3_a20", "affine", 2.0, ("dims", (3,))),
        ("affine_dim0_a10", "affine", 1.0, ("dims", (0,))),
        ("rigid_dims01", "rigid", None, ("dims", (0, 1))),
        ("affine_dims23", "affine", None, ("dims", (2, 3))),
        ("affine_proj", "affine", None, ("projection", ())),
        ("mean_proj", "mean", None, ("projection", ())),
        ("rigid_proj", "rigid", 1.0, ("projection", ())),
        ("rigid_proj_a15", "rigid", 1.5, ("projection", ())),
        ("linear_dim0", "linear", None, ("dims", (0,))),
        ("linear_proj", "linear", None, ("projection", ())),
        ("linear_dims13", "linear", None, ("dims", (1, 3))),
    ]
    for name, variant, alpha, (mode, dims) in cases:
        if mode == "projection":
            tg = F.projection_targets(mesh)
        elif len(dims) == 1:
            tg = F.dimension_targets(ds, ds.names[dims[0]])
        else:
            tg = F.dimension_targets(ds, ds.names[dims[0]], ds.names[dims[1]])
        fld = F.compute_field(mesh, positions, tg, F.MlsParams(variant=variant, alpha=alpha), W, H)
        c1[f"field_{name}"] = fld.coords
        c1[f"targets_{name}"] = tg.targets
        c1[f"channels_{name}"] = np.int64(tg.active_channels)
        if mode == "dims" and len(dims) == 1:
            sp = C.auto_spacing(tg.targets[:, 0])
            c1[f"spacing_{name}"] = np.float64(sp)
            c1[f"bands_{name}"] = Rn._band_indices(fld, sp).astype(np.int32)
            c1[f"coverage_{name}"] = Rn.line_coverage(fld, sp, 1.5)
    c1["field_cases"] = np.array([c[0] for c in cases])
    c1["field_variants"] = np.array([c[1] for c in cases])
    c1["field_alphas"] = np.array([np.nan if c[2] is None else c[2] for c in cases])
    out["c1"] = c1

    # ---- scene g2k: 2000 x 8, 5 iterations, BH + a 40x30 field ----------
    X = gmm(2000, 8, 5)
    ds, model, cloud, mesh, params, state, states, temps = scene(R, X, 0, 5, set(range(6)))
    g = dict(pca_mean=model.mean, pca_axes=model.axes, pca_eigenvalues=model.eigenvalues,
             pca_positions=cloud.positions, **mesh_arrays(mesh))
    g["states"] = np.stack([states[k] for k in range(6)])
    g["temps"] = np.array([temps[k] for k in range(6)])
    for k, v in params_dict(params).items():
        g[f"lp_{k}"] = np.float64(v)
    g["bh_0"] = B.repulsive_forces(states[0], params.repulsion_c, params.softening_eta, params.bh_theta)
    g["bh_exact_0"] = B.repulsive_forces_exact(states[0], params.repulsion_c, params.softening_eta)
    mesh.current_pos = states[5].copy()
    tg = F.dimension_targets(ds, ds.names[0])
    fld = F.compute_field(mesh, states[5], tg, F.MlsParams(variant="affine"), 40, 30)
    g["field_affine_dim0"] = fld.coords
    g["targets_affine_dim0"] = tg.targets
    g["field_positions"] = states[5]
    fld = F.compute_field(mesh, states[5], tg, F.MlsParams(variant="linear"), 120, 90)
    g["field_linear_dim0"] = fld.coords
    out["g2k"] = g

    # ---- scene g10k: config-2 data (10000 x 16, seed 2) ------------------
    X = gmm(10000, 16, 2)
    ds, model, cloud, mesh, params, state, states, temps = scene(R, X, 0, 31, {1, 2, 30, 31})
    g = dict(pca_eigenvalues=model.eigenvalues, pca_axes=model.axes, **mesh_arrays(mesh))
    g["states"] = np.stack([states[k] for k in (0, 1, 2, 30, 31)])
    g["state_iters"] = np.array([0, 1, 2, 30, 31])
    g["temps"] = np.array([temps[k] for k in (0, 1, 2, 30, 31)])
    for k, v in params_dict(params).items():
        g[f"lp_{k}"] = np.float64(v)
    g["bh_30"] = B.repulsive_forces(states[30], params.repulsion_c, params.softening_eta, params.bh_theta)
    out["g10k"] = g

    # ---- PCA on the reference's cars-like fixture -----------------------
    names, data = make_cars_like()
    D, P = R["dataset"], R["projection"]
    ds = D.normalize(D.Dataset(names=names, data=data))
    model, cloud = P.pca_project(ds)
    out["cars"] = dict(data=data, ds_data=ds.data, pca_mean=model.mean, pca_axes=model.axes,
                       pca_eigenvalues=model.eigenvalues, pca_positions=cloud.positions,
                       pca_viewport=np.array(cloud.viewport))

    for name, arrays in out.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **arrays)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
