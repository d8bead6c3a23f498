"""PCA parity (projection.py:50-79) on the GPU: eigenvalues and axes to 1e-9."""
import numpy as np
import pytest

from conftest import normwise

from paper_1408_0677_b200 import dataset as D
from paper_1408_0677_b200 import projection as P

pytestmark = pytest.mark.gpu


def test_pca_matches_reference(c1, cars):
    for g in (c1, cars):
        ds = D.Dataset(names=[f"c{i}" for i in range(g["ds_data"].shape[1])], data=g["ds_data"])
        model, cloud = P.pca_project(ds)
        assert normwise(model.eigenvalues, g["pca_eigenvalues"]) <= 1e-9
        assert np.abs(model.axes - g["pca_axes"]).max() <= 1e-9
        assert np.abs(model.mean - g["pca_mean"]).max() <= 1e-12
        assert np.abs(cloud.positions - g["pca_positions"]).max() <= 1e-9 * np.abs(g["pca_positions"]).max()
        assert np.allclose(cloud.viewport, g["pca_viewport"], rtol=1e-9)


def test_pca_larger_d():
    rng = np.random.default_rng(3)
    x = rng.normal(size=(5000, 64)) @ rng.normal(size=(64, 64))
    ds = D.normalize(D.Dataset(names=[f"c{i}" for i in range(64)], data=x))
    model, cloud = P.pca_project(ds)
    xc = ds.data - ds.data.mean(axis=0)
    cov = xc.T @ xc / (len(x) - 1)
    w, v = np.linalg.eigh(cov)
    assert normwise(model.eigenvalues, w[::-1][:2]) <= 1e-9
    for k in range(2):
        vk = v[:, -1 - k]
        vk = vk if vk[np.argmax(np.abs(vk))] > 0 else -vk
        assert np.abs(model.axes[k] - vk).max() <= 1e-9


def test_variance_zero():
    ds = D.normalize(D.Dataset(names=["a", "b", "c"], data=np.ones((5, 3))))
    with pytest.raises(P.VarianceZero):
        P.pca_project(ds)
