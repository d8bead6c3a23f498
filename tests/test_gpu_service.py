"""Interactive session on the GPU (service.py mirror).

Ports the reference's tests/test_service.py (routes, status codes, byte-
identical repeats, cache invalidation on recompute, planarity after a
recompute, 409 on concurrent recompute) and the viewer-loop acceptance
criterion (test_acceptance.py:273-338: monotone relax scrub, overlay pixels
identical across dimensions, alpha-slider round trip < 1 s)."""
import io
import time

import numpy as np
import pytest

from paper_1408_0677_b200 import cli, field, layout, render, service

from test_gpu_cli import make_cars_like

pytestmark = pytest.mark.gpu


def _write_csv(path, names, data):
    with open(path, "w") as fh:
        fh.write(",".join(names) + "\n")
        for row in data:
            fh.write(",".join(f"{v:.6g}" for v in row) + "\n")
    return path


@pytest.fixture(scope="module")
def session(tmp_path_factory):
    names, data = make_cars_like(rows=300, seed=11)
    csv = _write_csv(tmp_path_factory.mktemp("svc") / "cars.csv", names, data)
    cfg = cli.PipelineConfig(input=str(csv), variant="mean", mode="contour", width=128, height=128,
                             iterations=30, seed=3)
    return service.load_session(cfg)


@pytest.fixture(scope="module")
def client(session):
    from fastapi.testclient import TestClient

    return TestClient(service.create_app(session))


def wait_idle(client, timeout=60.0):
    t0 = time.time()
    while time.time() - t0 < timeout:
        if not client.get("/api/status").json()["recomputing"]:
            return
        time.sleep(0.05)
    raise TimeoutError("layout recompute did not finish")


def test_meta_and_defaults(client, session):
    body = client.get("/api/meta").json()
    assert body["columns"] == session.ds.names
    assert body["rowCount"] == session.ds.row_count
    d = client.get("/api/defaults").json()
    assert d["alpha"]["min"] == 0.25 and d["alpha"]["max"] == 3.0
    assert set(d["variants"]) == {"linear", "mean", "affine", "rigid"}
    assert "adaptive" in d["modes"]


def test_positions_relax_endpoints(client, session):
    p0 = np.array(client.get("/api/positions", params={"relax": 0}).json()["positions"])
    p1 = np.array(client.get("/api/positions", params={"relax": 1}).json()["positions"])
    np.testing.assert_allclose(p0, session.mesh.original_pos, atol=1e-9)
    np.testing.assert_allclose(p1, session.snapshot.state.relaxed_pos, atol=1e-9)
    assert client.get("/api/positions", params={"relax": 2}).status_code == 400


def test_repeat_get_byte_identical_and_cached_on_gpu(client, session):
    q = "/api/render.png?dim=mpg&variant=mean&alpha=1.0&relax=0.7&mode=contour&w=96&h=96"
    hits = session.cache_hits
    a = client.get(q)
    b = client.get(q)
    assert a.status_code == 200 and a.headers["content-type"] == "image/png"
    assert a.content == b.content
    assert session.cache_hits == hits + 1
    key = (session.snapshot.revision, "mpg", "", "mean", 1.0, 0.7, 96, 96)
    fld = session._field_cache[key]
    assert fld.device_coords is not None and fld.device_coords.is_cuda
    assert np.array_equal(fld.device_coords.cpu().numpy(), fld.coords)


def test_render_matches_cli_pipeline(client, session):
    resp = client.get("/api/render.png", params={"dim": "weight", "variant": "mean", "relax": 1.0,
                                                 "mode": "contour", "w": 128, "h": 128})
    assert resp.status_code == 200
    pos = layout.interpolate_layout(session.snapshot.state, 1.0)
    img = cli.render_one(session.cfg, session.ds, session.mesh, pos, ("weight",))
    assert resp.content == img.to_png_bytes()


@pytest.mark.parametrize("params,status,key", [
    ({"dim": "mpg", "relax": 1.7}, 400, "relax"),
    ({"dim": "mpg", "variant": "cubic"}, 400, "variant"),
    ({"dim": "mpg", "alpha": 99.0}, 400, "alpha"),
    ({"dim": "mpg", "mode": "gradient"}, 400, "mode"),
    ({"dim": "mpg", "variant": "rigid"}, 400, "variant"),
    ({"dim": "mpg", "spacing": "-1"}, 400, "spacing"),
])
def test_invalid_params_yield_field_messages(client, params, status, key):
    r = client.get("/api/render.png", params=params)
    assert r.status_code == status
    assert key in r.json()["errors"]


def test_unknown_dimension_404(client):
    r = client.get("/api/render.png", params={"dim": "warp"})
    assert r.status_code == 404
    assert "columns" in r.json()


def test_all_modes_and_variants_render(client):
    for variant, mode, extra in (("affine", "discrete+contour", {}), ("linear", "adaptive", {}),
                                 ("rigid", "gradient", {"dim2": "horsepower"}), ("mean", "discrete", {})):
        r = client.get("/api/render.png", params={"dim": "mpg", "variant": variant, "mode": mode,
                                                  "w": 80, "h": 64, **extra})
        assert r.status_code == 200, (variant, mode, r.text)


def test_layout_recompute_bumps_revision_and_preserves_planarity(client, session):
    rev0 = client.get("/api/status").json()["revision"]
    signs0 = np.sign(session.mesh.signed_areas(session.mesh.original_pos))
    r = client.post("/api/layout", json={"iterations": 40, "lambda": 0.95})
    assert r.status_code == 202, r.text
    wait_idle(client)
    assert client.get("/api/status").json()["revision"] == rev0 + 1
    p1 = np.array(client.get("/api/positions", params={"relax": 1}).json()["positions"])
    assert np.all(np.sign(session.mesh.signed_areas(p1)) == signs0)


def test_concurrent_recompute_409(client):
    r1 = client.post("/api/layout", json={"iterations": 600, "lambda": 0.999})
    assert r1.status_code == 202
    r2 = client.post("/api/layout", json={"iterations": 10, "lambda": 0.9})
    assert r2.status_code == 409
    wait_idle(client, timeout=120.0)


def test_invalid_layout_params_rejected(client):
    assert client.post("/api/layout", json={"iterations": 10, "lambda": 1.5}).status_code == 422


def test_recompute_invalidates_field_cache(client):
    q = "/api/render.png?dim=mpg&variant=mean&relax=1&mode=contour&w=64&h=64"
    before = client.get(q).content
    client.post("/api/layout", json={"iterations": 80, "lambda": 0.9})
    wait_idle(client)
    after = client.get(q).content
    assert before != after


def test_viewer_loop_acceptance(tmp_path):
    """test_acceptance.py:273-338 against this service."""
    from fastapi.testclient import TestClient
    from PIL import Image

    names, data = make_cars_like(rows=300, seed=29)
    csv = _write_csv(tmp_path / "cars.csv", names, data)
    cfg = cli.PipelineConfig(input=str(csv), variant="mean", mode="contour", width=320, height=320,
                             iterations=120, seed=1)
    session = service.load_session(cfg)
    client = TestClient(service.create_app(session))

    orig = np.array(client.get("/api/positions", params={"relax": 0}).json()["positions"])
    prev = np.zeros(len(orig))
    for t in np.linspace(0.0, 1.0, 9):
        pos = np.array(client.get("/api/positions", params={"relax": t}).json()["positions"])
        dist = np.hypot(*(pos - orig).T)
        assert np.all(dist >= prev - 1e-9), f"non-monotone marker motion at relax={t}"
        prev = dist

    def fetch(dim):
        r = client.get("/api/render.png", params={"dim": dim, "variant": "mean", "relax": 1.0,
                                                  "mode": "contour", "w": 320, "h": 320})
        assert r.status_code == 200
        return np.array(Image.open(io.BytesIO(r.content)).convert("RGBA"))

    img_a, img_b = fetch("mpg"), fetch("weight")
    pos = layout.interpolate_layout(session.snapshot.state, 1.0)
    transform = field.ViewportTransform.fit(pos, 320, 320)
    spec = render.RenderSpec(spacing=1.0, point_radius=cfg.point_radius - 1.0)
    interior = render.point_mask((320, 320), pos, transform, spec)
    point_rgba = np.array(render.RenderSpec(spacing=1.0).point_color, dtype=np.uint8)
    assert np.all(img_a[interior] == point_rgba)
    np.testing.assert_array_equal(img_a[interior], img_b[interior])
    assert (img_a != img_b).any()

    times = []
    for alpha in (1.3, 0.8, 1.05):
        t0 = time.perf_counter()
        r = client.get("/api/render.png", params={"dim": "mpg", "variant": "mean", "alpha": alpha,
                                                  "relax": 1.0, "mode": "contour", "w": 320, "h": 320})
        times.append(time.perf_counter() - t0)
        assert r.status_code == 200 and r.content
    dt = sorted(times)[1]
    print("alpha slider round trips (s):", [round(t, 4) for t in times])
    assert dt < 1.0


def test_dim2_projection_is_404(client, session):
    """service.py:188-192: 'projection' is accepted as dim only; an unknown dim2
    (including 'projection') is a 404, never a 500."""
    r = client.get("/api/render.png", params={"dim": session.ds.names[0], "dim2": "projection"})
    assert r.status_code == 404
    assert client.get("/api/render.png", params={"dim": "projection"}).status_code == 200


def test_field_cache_is_bounded_and_drops_stale_revisions(session, monkeypatch):
    """The cache is an LRU (CACHE_MAX_ENTRIES) and only the DEVICE_KEEP most
    recent entries keep their GPU copy; a field built for a revision that was
    swapped out meanwhile is served but not cached."""
    monkeypatch.setattr(service, "CACHE_MAX_ENTRIES", 5)
    monkeypatch.setattr(service, "DEVICE_KEEP", 2)
    rev = session.snapshot.revision
    dim = session.ds.names[0]
    for i in range(8):
        service.render_png(session, dim=dim, alpha=0.5 + 0.1 * i, w=32, h=24)
    with session.lock:
        entries = list(session._field_cache.values())
    assert len(entries) == 5
    assert sum(e.device_coords is not None for e in entries) == 2
    assert entries[-1].device_coords is not None
    # a build for a stale revision is returned but not inserted
    before = len(session._field_cache)
    stale_key = (rev - 1, dim, "", "mean", 1.0, 1.0, 32, 24)
    out = session.cached_field(stale_key, lambda: entries[-1])
    assert out is entries[-1]
    assert stale_key not in session._field_cache and len(session._field_cache) == before
