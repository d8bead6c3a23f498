"""Interactive session: GPU-resident snapshot + field cache behind the viewer API.

Mirror of the reference's ``service`` module (service.py:1-292, SURVEY.md
§8f row 4).  One dataset per process; the layout relaxation runs only on an
explicit request on a worker thread (``mdc_layout_steps`` on the GPU);
every GET re-renders from the current immutable snapshot.  Fields are cached
by their full parameter key exactly as the reference does (service.py:40-84),
but the cached ``CoordinateField`` carries its GPU copy (``device_coords``),
so a cache hit renders, composites the point overlay and encodes with ONE
device->host copy of the RGBA8 image.  Identical query strings return
identical bytes until a recompute bumps the revision.

``create_app`` is a thin FastAPI adapter over ``render_png`` / ``relayout``
(same routes, status codes and error payloads as the reference); the viewer
bundle is not shipped.
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from dataclasses import dataclass, field as dc_field
from typing import Optional

import torch
from pydantic import BaseModel, Field

from . import dataset as dataset_mod
from . import field, layout, render
from .cli import PipelineConfig, prepare_session
from .render import auto_spacing

MAX_RESOLUTION = 8192


class LayoutRequest(BaseModel):
    """service.py:30-37: POST /api/layout body."""

    iterations: int = Field(default=500, ge=0, le=100_000)
    decay_lambda: float = Field(default=0.99, gt=0.0, lt=1.0, alias="lambda")
    initial_temp: Optional[float] = Field(default=None, gt=0.0)
    edge_length: Optional[float] = Field(default=None, gt=0.0)

    model_config = {"populate_by_name": True}


@dataclass
class Snapshot:
    """service.py:40-47: one immutable view of the session."""

    revision: int
    state: layout.LayoutState
    params: layout.LayoutParams


# Field-cache bounds.  The reference's cache is an unbounded dict of host
# arrays; here every entry can also hold a GPU fp64 copy (H*W*16 bytes), so
# the cache is an LRU over entries and only the most recent DEVICE_KEEP
# entries keep their device copy (older hits re-upload on render).
CACHE_MAX_ENTRIES = 64
DEVICE_KEEP = 4


@dataclass
class Session:
    """service.py:50-72 (field cache keyed by the full parameter tuple)."""

    cfg: PipelineConfig
    ds: dataset_mod.Dataset
    mesh: object
    snapshot: Snapshot
    lock: threading.Lock = dc_field(default_factory=threading.Lock)
    recomputing: bool = dc_field(default=False)
    _field_cache: OrderedDict = dc_field(default_factory=OrderedDict)
    cache_hits: int = 0
    cache_misses: int = 0

    def _touch(self, key):  # caller holds the lock
        self._field_cache.move_to_end(key)
        for i, k in enumerate(reversed(self._field_cache)):
            if i >= DEVICE_KEEP:
                self._field_cache[k].device_coords = None
        while len(self._field_cache) > CACHE_MAX_ENTRIES:
            self._field_cache.popitem(last=False)

    def cached_field(self, key, build):
        with self.lock:
            hit = self._field_cache.get(key)
            if hit is not None:
                self.cache_hits += 1
                self._touch(key)
        if hit is not None:
            return hit
        fld = build()
        with self.lock:
            self.cache_misses += 1
            if key[0] != self.snapshot.revision:
                # built from a snapshot that was swapped out meanwhile: serve it, do not cache it
                return fld
            # identical keys reuse bit-identical fields: first write wins
            fld = self._field_cache.setdefault(key, fld)
            self._touch(key)
            return fld

    def swap_snapshot(self, snap: Snapshot):
        with self.lock:
            self.snapshot = snap
            self._field_cache.clear()


def load_session(cfg: PipelineConfig) -> Session:
    """service.py:75-84 (PCA, mesh and the initial layout on the GPU)."""
    ds, model, tri, params, state = prepare_session(cfg)
    return Session(cfg=cfg, ds=ds, mesh=tri, snapshot=Snapshot(revision=0, state=state, params=params))


def defaults_payload(session: Session) -> dict:
    """service.py:91-113."""
    snap = session.snapshot
    return {
        "variants": list(field.VARIANTS),
        "modes": list(render.MODES),
        "alpha": {"min": field.ALPHA_RANGE[0], "max": field.ALPHA_RANGE[1], "perVariant": field.DEFAULT_ALPHA},
        "relax": {"min": 0.0, "max": 1.0, "default": 1.0},
        "resolution": {"default": [session.cfg.width, session.cfg.height], "max": MAX_RESOLUTION},
        "variant": session.cfg.variant,
        "mode": session.cfg.mode,
        "layout": {
            "iterations": snap.params.iterations,
            "lambda": snap.params.decay_lambda,
            "initialTemp": snap.params.initial_temp,
            "edgeLength": snap.params.desired_edge_d,
        },
    }


def meta_payload(session: Session) -> dict:
    return {"columns": session.ds.names, "rowCount": session.ds.row_count,
            "revision": session.snapshot.revision, "defaults": defaults_payload(session)}


class RequestError(Exception):
    """A rejected request: HTTP status + JSON payload (service.py's 400/404/409)."""

    def __init__(self, status: int, payload: dict):
        super().__init__(payload)
        self.status = status
        self.payload = payload


def positions_payload(session: Session, relax: float = 1.0) -> dict:
    """service.py:126-138."""
    if not 0.0 <= relax <= 1.0:
        raise RequestError(400, {"errors": {"relax": "must be in [0, 1]"}})
    snap = session.snapshot
    pos = layout.interpolate_layout(snap.state, relax)
    return {"revision": snap.revision, "relax": relax, "positions": [[float(x), float(y)] for x, y in pos]}


def render_png(session: Session, dim: str = "", dim2: str = "", variant: Optional[str] = None,
               alpha: Optional[float] = None, relax: float = 1.0, mode: Optional[str] = None,
               spacing: str = "auto", w: Optional[int] = None, h: Optional[int] = None) -> bytes:
    """service.py:140-217: validate, fetch/build the cached field, render on
    the GPU (field -> RGBA8 -> point overlay, all device-resident), encode."""
    cfg = session.cfg
    variant = variant or cfg.variant
    mode = mode or cfg.mode
    w = w or cfg.width
    h = h or cfg.height

    errors = {}
    if variant not in field.VARIANTS:
        errors["variant"] = f"must be one of {', '.join(field.VARIANTS)}"
    if mode not in render.MODES:
        errors["mode"] = f"must be one of {', '.join(render.MODES)}"
    if not 0.0 <= relax <= 1.0:
        errors["relax"] = "must be in [0, 1]"
    if alpha is not None and not (field.ALPHA_RANGE[0] <= alpha <= field.ALPHA_RANGE[1]):
        errors["alpha"] = f"must be in [{field.ALPHA_RANGE[0]}, {field.ALPHA_RANGE[1]}]"
    if not (w and h and 0 < w <= MAX_RESOLUTION and 0 < h <= MAX_RESOLUTION):
        errors["w"] = errors["h"] = f"resolution limited to {MAX_RESOLUTION}"
    spacing_val: float | str = "auto"
    if spacing != "auto":
        try:
            spacing_val = float(spacing)
            if spacing_val <= 0:
                errors["spacing"] = "must be positive"
        except ValueError:
            errors["spacing"] = "must be a number or 'auto'"
    if errors:
        raise RequestError(400, {"errors": errors})
    # service.py:183-192: 'projection' is a valid dim only; any unknown dim2 is a 404
    for name, allow_projection in ((dim, True), (dim2, False)):
        if name and not (allow_projection and name == "projection") and name not in session.ds.names:
            raise RequestError(404, {"error": f"unknown dimension {name!r}", "columns": session.ds.names})

    if not dim or dim == "projection":
        targets = field.projection_targets(session.mesh)
    elif dim2:
        targets = field.dimension_targets(session.ds, dim, dim2)
    else:
        targets = field.dimension_targets(session.ds, dim)
    if variant == "rigid" and targets.active_channels == 1:
        raise RequestError(400, {"errors": {"variant": "rigid is degenerate for a single dimension"}})
    if mode == "gradient" and targets.active_channels == 1:
        raise RequestError(400, {"errors": {"mode": "gradient requires two target dimensions"}})

    snap = session.snapshot
    key = (snap.revision, dim, dim2, variant, alpha, relax, w, h)
    pos = layout.interpolate_layout(snap.state, relax)

    def build():
        params = field.MlsParams(variant=variant, alpha=alpha)
        return field.compute_field(session.mesh, pos, targets, params, w, h, threads=cfg.threads)

    fld = session.cached_field(key, build)
    s = auto_spacing(targets.targets[:, 0]) if spacing_val == "auto" else spacing_val
    spec = render.RenderSpec(mode=mode, spacing=s, point_radius=cfg.point_radius)
    px = render.render_device(fld, spec)
    render.overlay_points_device(px, pos, fld.transform, spec)
    host = px.cpu().numpy()
    return render.RenderedImage(width=host.shape[1], height=host.shape[0], pixels=host).to_png_bytes()


def relayout(session: Session, iterations: int = 500, decay_lambda: float = 0.99,
             initial_temp: Optional[float] = None, edge_length: Optional[float] = None,
             wait: bool = False) -> dict:
    """service.py:219-249: start a layout recompute on a worker thread (409
    while one is running); the new snapshot replaces the old atomically and
    clears the field cache."""
    if not (0 <= iterations <= 100_000) or not (0.0 < decay_lambda < 1.0) or \
            (initial_temp is not None and initial_temp <= 0) or (edge_length is not None and edge_length <= 0):
        raise RequestError(422, {"error": "invalid layout parameters"})
    with session.lock:
        if session.recomputing:
            raise RequestError(409, {"error": "layout recompute already in progress"})
        session.recomputing = True
        target_revision = session.snapshot.revision + 1
    # the worker thread starts on the default device: pin the caller's (the session's) device
    dev = torch.cuda.current_device() if torch.cuda.is_available() else None

    def work():
        try:
            overrides = {"decay_lambda": decay_lambda}
            if initial_temp is not None:
                overrides["initial_temp"] = initial_temp
            if edge_length is not None:
                overrides["desired_edge_d"] = edge_length
            params = layout.LayoutParams.defaults_for(session.mesh, iterations=iterations, **overrides)
            session.mesh.current_pos = session.mesh.original_pos.copy()
            if dev is not None:
                torch.cuda.set_device(dev)
            state = layout.layout_run(session.mesh, params)
            session.swap_snapshot(Snapshot(target_revision, state, params))
        finally:
            with session.lock:
                session.recomputing = False

    th = threading.Thread(target=work, daemon=True)
    th.start()
    if wait:
        th.join()
    return {"accepted": True, "revision": target_revision}


def status_payload(session: Session) -> dict:
    with session.lock:
        return {"revision": session.snapshot.revision, "recomputing": session.recomputing}


def create_app(session: Session):
    """service.py:116-281 routes over the functions above (FastAPI)."""
    from fastapi import FastAPI, Query, Response
    from fastapi.responses import JSONResponse

    app = FastAPI(title="mdcontour-b200", docs_url=None, redoc_url=None)
    device = torch.cuda.current_device() if torch.cuda.is_available() else None

    def on_device(fn, *a, **kw):
        # request handlers run on a thread pool: pin the session's device
        if device is not None:
            torch.cuda.set_device(device)
        try:
            return fn(*a, **kw)
        except RequestError as exc:
            return JSONResponse(status_code=exc.status, content=exc.payload)

    @app.get("/api/meta")
    def meta():
        return meta_payload(session)

    @app.get("/api/defaults")
    def defaults():
        return defaults_payload(session)

    @app.get("/api/positions")
    def positions(relax: float = Query(default=1.0)):
        return on_device(positions_payload, session, relax)

    @app.get("/api/render.png")
    def render_route(dim: str = Query(default=""), dim2: str = Query(default=""),
                     variant: str = Query(default=None), alpha: float = Query(default=None),
                     relax: float = Query(default=1.0), mode: str = Query(default=None),
                     spacing: str = Query(default="auto"), w: int = Query(default=None),
                     h: int = Query(default=None)):
        out = on_device(render_png, session, dim=dim, dim2=dim2, variant=variant, alpha=alpha, relax=relax,
                        mode=mode, spacing=spacing, w=w, h=h)
        if isinstance(out, bytes):
            return Response(content=out, media_type="image/png")
        return out

    @app.post("/api/layout", status_code=202)
    def layout_route(req: LayoutRequest):
        return on_device(relayout, session, iterations=req.iterations, decay_lambda=req.decay_lambda,
                         initial_temp=req.initial_temp, edge_length=req.edge_length)

    @app.get("/api/status")
    def status():
        return status_payload(session)

    @app.get("/")
    def index():
        return Response("mdcontour-b200 service is running; the viewer bundle is not shipped.",
                        media_type="text/plain")

    return app


def serve(cfg: PipelineConfig, port: int = 8000, host: str = "127.0.0.1") -> None:
    """service.py:284-292."""
    import uvicorn

    session = load_session(cfg)
    uvicorn.run(create_app(session), host=host, port=port, log_level="warning")
