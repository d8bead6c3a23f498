"""Kd-tree Barnes-Hut repulsion on the GPU.

Mirror of the reference's ``bhtree`` module (bhtree.py:10-129): the same
median-split kd-tree (rebuilt on the device per call) and opening criterion,
evaluated by libmdc's warp-cooperative traversal.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib


class _TreePlan:
    """libmdc layout plan over an empty topology: tree + BH only."""

    def __init__(self, n: int, c: float, eta: float, theta: float, leaf: int):
        lib = _lib.require_cuda()
        self.lib = lib
        dev = torch.device("cuda", torch.cuda.current_device())
        self.zeros = torch.zeros(n + 1, dtype=torch.int32, device=dev)
        self.pos = torch.zeros((n, 2), dtype=torch.float64, device=dev)
        self.ws = torch.empty(int(lib.mdc_layout_workspace_bytes(n, leaf)), dtype=torch.uint8, device=dev)
        a = _lib.MdcLayoutArgs()
        a.n, a.ntri, a.leaf = n, 0, leaf
        a.c, a.spring, a.dlen, a.eta, a.theta = c, 1.0, 1.0, eta, theta
        z = _lib.ptr(self.zeros)
        a.csr_off = a.csr_tgt = a.inc_off = z
        a.pos = _lib.ptr(self.pos)
        a.workspace, a.workspace_bytes = _lib.ptr(self.ws), self.ws.numel()
        self.args = a
        h = ctypes.c_void_p()
        _lib.check(lib.mdc_layout_plan_create(ctypes.byref(a), ctypes.byref(h), _lib.stream_ptr()),
                   "mdc_layout_plan_create")
        self.h = h

    def __del__(self):
        try:
            self.lib.mdc_layout_plan_destroy(self.h)
        except Exception:
            pass


_PLANS: dict = {}


def _plan(n, c, eta, theta, leaf) -> _TreePlan:
    key = (n, c, eta, theta, leaf, torch.cuda.current_device())
    p = _PLANS.get(key)
    if p is None:
        if len(_PLANS) > 8:
            _PLANS.clear()
        p = _PLANS[key] = _TreePlan(n, c, eta, theta, leaf)
    return p


def repulsive_forces_device(points: torch.Tensor, c: float, eta: float, theta: float,
                            leaf_size: int = 32) -> torch.Tensor:
    """Barnes-Hut repulsion of an (n, 2) float64 CUDA tensor (bhtree.py:69-95)."""
    n = points.shape[0]
    out = torch.zeros_like(points)
    if n < 2:
        return out
    p = _plan(n, c, eta, theta, leaf_size)
    pts = points.contiguous()
    _lib.check(p.lib.mdc_layout_repulsion(p.h, _lib.ptr(pts), _lib.ptr(out), _lib.stream_ptr()),
               "mdc_layout_repulsion")
    return out


def repulsive_forces(points: np.ndarray, c: float, eta: float, theta: float,
                     leaf_size: int = 32) -> np.ndarray:
    """bhtree.py:69-95: net repulsive force on every point (numpy in/out)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if len(pts) < 2:
        return np.zeros_like(pts)
    t = torch.as_tensor(pts).cuda()
    return repulsive_forces_device(t, c, eta, theta, leaf_size).cpu().numpy()


class KdTree:
    """bhtree.py:10-66 flat node arrays, built on the GPU (int32 indices)."""

    def __init__(self, points: np.ndarray, leaf_size: int = 16):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        n = len(pts)
        p = _plan(n, 1.0, 1.0, 0.5, leaf_size)
        lib = p.lib
        nn = int(lib.mdc_layout_node_count(p.h))
        dev = p.pos.device
        t = torch.as_tensor(pts).to(dev)
        i32 = dict(dtype=torch.int32, device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        perm = torch.empty(n, **i32)
        lo, hi, left, right = (torch.empty(nn, **i32) for _ in range(4))
        com, bmin, bmax = (torch.empty((nn, 2), **f64) for _ in range(3))
        mass, size = torch.empty(nn, **f64), torch.empty(nn, **f64)
        _lib.check(lib.mdc_layout_kdtree(p.h, _lib.ptr(t), _lib.ptr(perm), _lib.ptr(lo), _lib.ptr(hi),
                                         _lib.ptr(left), _lib.ptr(right), _lib.ptr(com), _lib.ptr(mass),
                                         _lib.ptr(size), _lib.ptr(bmin), _lib.ptr(bmax), _lib.stream_ptr()),
                   "mdc_layout_kdtree")
        self.points = pts
        self.perm = perm.cpu().numpy().astype(np.int64)
        self.lo, self.hi = lo.cpu().numpy().astype(np.int64), hi.cpu().numpy().astype(np.int64)
        self.left, self.right = left.cpu().numpy().astype(np.int64), right.cpu().numpy().astype(np.int64)
        self.com, self.mass, self.size = com.cpu().numpy(), mass.cpu().numpy(), size.cpu().numpy()
        self.bmin, self.bmax = bmin.cpu().numpy(), bmax.cpu().numpy()
        self._count = nn


def repulsive_forces_exact(points: np.ndarray, c: float, eta: float) -> np.ndarray:
    """bhtree.py:123-129 direct O(n^2) sum (host; test oracle helper)."""
    d = points[:, None, :] - points[None, :, :]
    r2 = np.einsum("ijk,ijk->ij", d, d)
    with np.errstate(divide="ignore"):
        w = c / (r2 * np.sqrt(r2) + eta)
    np.fill_diagonal(w, 0.0)
    return np.einsum("ij,ijk->ik", w, d)
