"""The one-to-one numba-seam replacements (mdc_{mean,affine,rigid}_field,
mdc_bh_forces) against the oracle, which is itself bit-exact against the
reference (test_oracle.py).  Same operation order, no FMA contraction:
bit-exact for the fast-path alphas, <= 1e-15 normwise for generic alpha."""
import ctypes

import numpy as np
import pytest
import torch

import oracle as O
from conftest import layout_params, normwise

from paper_1408_0677_b200 import _lib

pytestmark = pytest.mark.gpu


def _dev(a):
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("variant,alpha", [("affine", 1.5), ("mean", 1.0), ("rigid", 1.0),
                                           ("affine", 1.3), ("mean", 0.5), ("affine", 2.0)])
def test_seam_kernels_match_numba_restatement(c1, variant, alpha):
    lib = _lib.require_cuda()
    pos = c1["field_positions"]
    tv = c1["targets_affine_proj"]
    W, H = 64, 48
    vp = O.viewport(pos, W, H)
    pm, qm = pos.mean(axis=0), tv.mean(axis=0)
    pc, qc = pos - pm, tv - qm
    xs, ys = O.pixel_centers(vp, W, H)
    vx, vy = xs.ravel() - pm[0], ys.ravel() - pm[1]
    ref = O.mls_kernel(variant, vx, vy, pc, qc, alpha)
    q = (qc - pc) if variant == "mean" else qc
    t = [_dev(v) for v in (vx, vy, pc[:, 0], pc[:, 1], q[:, 0], q[:, 1])]
    out = torch.empty((len(vx), 2), dtype=torch.float64, device="cuda")
    P = [_lib.ptr(x) for x in t]
    s = _lib.stream_ptr()
    if variant == "affine":
        rc = lib.mdc_affine_field(len(vx), P[0], P[1], len(pc), P[2], P[3], P[4], P[5], alpha, 1e-12, _lib.ptr(out), s)
    elif variant == "mean":
        rc = lib.mdc_mean_field(len(vx), P[0], P[1], len(pc), P[2], P[3], P[4], P[5], alpha, _lib.ptr(out), s)
    else:
        rc = lib.mdc_rigid_field(len(vx), P[0], P[1], len(pc), P[2], P[3], P[4], P[5], alpha, _lib.ptr(out), s)
    _lib.check(rc, variant)
    got = out.cpu().numpy()
    if alpha in (1.0, 1.5, 0.5, 2.0) and variant != "rigid":
        assert np.array_equal(got, ref), normwise(got, ref)
    else:  # CUDA pow / hypot vs glibc: last-ulp differences
        assert normwise(got, ref) <= 1e-14


def test_seam_bh_forces_match_oracle(g2k):
    lib = _lib.require_cuda()
    p = layout_params(g2k)
    pts = g2k["states"][1]
    tree = O.KdTree(pts, leaf_size=32)
    ref = np.empty_like(pts)
    O.lib().orc_bh_forces(ctypes.c_int64(len(pts)), O._d(pts), O._i(tree.perm), O._i(tree.lo), O._i(tree.hi),
                          O._i(tree.left), O._i(tree.right), O._d(tree.com), O._d(tree.mass), O._d(tree.size),
                          O._d(tree.bmin), O._d(tree.bmax), ctypes.c_double(p["repulsion_c"]),
                          ctypes.c_double(p["softening_eta"]), ctypes.c_double(p["bh_theta"]), O._d(ref))
    d = [_dev(a) for a in (pts, tree.perm, tree.lo, tree.hi, tree.left, tree.right, tree.com, tree.mass,
                           tree.size, tree.bmin, tree.bmax)]
    out = torch.empty((len(pts), 2), dtype=torch.float64, device="cuda")
    _lib.check(lib.mdc_bh_forces(len(pts), *[_lib.ptr(x) for x in d], p["repulsion_c"], p["softening_eta"],
                                 p["bh_theta"], _lib.ptr(out), _lib.stream_ptr()), "mdc_bh_forces")
    got = out.cpu().numpy()
    # same tree, same DFS and summation order, no contraction: bit-exact
    assert np.array_equal(got, ref), normwise(got, ref)
