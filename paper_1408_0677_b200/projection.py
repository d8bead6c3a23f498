"""PCA projection onto the top two principal axes, on the GPU.

Mirrors projection.py:16-79 of the reference (same dataclasses, defaults,
errors, sign convention); the numerics run in libmdc's ``mdc_pca``
(fp64 covariance with deterministic chunked reductions + one-CTA parallel
Jacobi eigensolver).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .dataset import Dataset


class VarianceZero(Exception):
    """All columns constant: no principal directions exist."""


@dataclass(frozen=True)
class ProjectionModel:
    mean: np.ndarray          # (d,)
    axes: np.ndarray          # (2, d), orthonormal rows
    eigenvalues: np.ndarray   # (2,), descending

    def transform(self, rows: np.ndarray) -> np.ndarray:
        return (rows - self.mean) @ self.axes.T


@dataclass(frozen=True)
class PointCloud2D:
    positions: np.ndarray     # (n, 2)
    viewport: tuple[float, float, float, float]


def expand_bounds(points: np.ndarray, margin: float = 0.05) -> tuple[float, float, float, float]:
    """projection.py:36-47 (host; bit-identical numpy arithmetic)."""
    x0, y0 = points.min(axis=0)
    x1, y1 = points.max(axis=0)
    dx = (x1 - x0) or 1.0
    dy = (y1 - y0) or 1.0
    return (float(x0 - margin * dx), float(y0 - margin * dy),
            float(x1 + margin * dx), float(y1 + margin * dy))


def pca_device(x: torch.Tensor):
    """Device PCA of an (n, d) float64 CUDA tensor.

    Returns (mean (d,), cov (d, d), eigenvalues (2,), axes (2, d),
    positions (n, 2)) as CUDA tensors, all produced by one ``mdc_pca`` call.
    """
    lib = _lib.require_cuda()
    x = x.contiguous()
    n, d = x.shape
    dev = x.device
    mean = torch.empty(d, dtype=torch.float64, device=dev)
    cov = torch.empty((d, d), dtype=torch.float64, device=dev)
    ev = torch.empty(2, dtype=torch.float64, device=dev)
    axes = torch.empty((2, d), dtype=torch.float64, device=dev)
    pos = torch.empty((n, 2), dtype=torch.float64, device=dev)
    ws = torch.empty(int(lib.mdc_pca_workspace_bytes(n, d)), dtype=torch.uint8, device=dev)
    with _lib.nvtx("pca"):
        _lib.check(lib.mdc_pca(ctypes.c_int64(n), ctypes.c_int32(d), _lib.ptr(x), _lib.ptr(mean),
                               _lib.ptr(cov), _lib.ptr(ev), _lib.ptr(axes), _lib.ptr(pos),
                               _lib.ptr(ws), _lib.stream_ptr()), "mdc_pca")
    return mean, cov, ev, axes, pos


def pca_project(ds: Dataset) -> tuple[ProjectionModel, PointCloud2D]:
    """projection.py:50-79 on the GPU."""
    if ds.row_count < 2 or (ds.constant and all(ds.constant)):
        raise VarianceZero("dataset has no varying column")
    if ds.dim_count < 2:
        raise VarianceZero("need at least two dimensions for a 2D projection")
    x = torch.as_tensor(np.ascontiguousarray(ds.data, dtype=np.float64)).cuda()
    mean, cov, ev, axes, pos = pca_device(x)
    cov_h = cov.cpu().numpy()
    if not np.any(cov_h):
        raise VarianceZero("covariance is identically zero")
    positions = pos.cpu().numpy()
    return (
        ProjectionModel(mean=mean.cpu().numpy(), axes=axes.cpu().numpy(),
                        eigenvalues=ev.cpu().numpy()),
        PointCloud2D(positions=positions, viewport=expand_bounds(positions)),
    )
