"""Triangle-mesh container (CSR + anchored fans) and the layout topology.

``TriMesh`` mirrors the reference's arrays (mesh.py:107-128) so meshes built
by either package drop into ``layout_step`` / ``compute_field``.  Mesh
CONSTRUCTION is outside the GPU hot path: the
``delaunay`` here triangulates with scipy's Qhull and canonicalises exactly
like the reference's ``_assemble`` (mesh.py:362-416), which yields the same
arrays as the reference's Bowyer-Watson for points in general position
(checked against the reference's own meshes in tests/test_mesh.py).

``layout_topology`` derives the int32 device-side topology the layout kernels
consume (CSR, padded triangles, per-vertex incident (triangle, corner) lists
in the per-corner bincount order of layout.py:240-255).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from fractions import Fraction

import numpy as np


class MeshError(Exception):
    pass


class DegenerateInput(MeshError):
    """All input points collinear: no triangulation exists."""


class ZeroAreaTriangle(MeshError):
    pass


def signed_area(a, b, c) -> float:
    """mesh.py:33-35."""
    return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]))


def limiting_lines(tri, positions):
    """mesh.py:82-104: midsegment line (point, inward unit normal) per vertex."""
    a, b, c = (np.asarray(positions[i], dtype=float) for i in tri)
    if signed_area(a, b, c) == 0.0:
        raise ZeroAreaTriangle(f"triangle {tuple(tri)} has zero area")
    verts = (a, b, c)
    out = []
    for k in range(3):
        v = verts[k]
        m1 = 0.5 * (v + verts[(k + 1) % 3])
        m2 = 0.5 * (v + verts[(k + 2) % 3])
        d = m2 - m1
        n = np.array([-d[1], d[0]])
        n /= np.linalg.norm(n)
        if np.dot(n, v - m1) < 0:
            n = -n
        out.append((m1, n))
    return out


@dataclass
class TriMesh:
    """mesh.py:107-128 field-for-field."""

    node_count: int
    original_pos: np.ndarray
    current_pos: np.ndarray
    csr_offsets: np.ndarray
    csr_targets: np.ndarray
    fan_offsets: np.ndarray
    fan_nodes: np.ndarray
    triangles: np.ndarray
    jitter_count: int = 0

    @property
    def edge_count(self) -> int:
        return len(self.csr_targets) // 2

    @property
    def triangle_count(self) -> int:
        return len(self.triangles)

    def neighbors(self, i: int) -> np.ndarray:
        return self.csr_targets[self.csr_offsets[i]: self.csr_offsets[i + 1]]

    def signed_areas(self, positions: np.ndarray | None = None) -> np.ndarray:
        """mesh.py:178-187."""
        p = self.current_pos if positions is None else positions
        a = p[self.triangles[:, 0]]
        b = p[self.triangles[:, 1]]
        c = p[self.triangles[:, 2]]
        return 0.5 * ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1])
                      - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0]))

    def fan_entries(self, i: int) -> np.ndarray:
        """mesh.py:157-158: the fan-stored second vertices of node i's anchored triangles."""
        return self.fan_nodes[self.fan_offsets[i]: self.fan_offsets[i + 1]]

    def node_triangles(self, i: int) -> list[tuple[int, int, int]]:
        """mesh.py:160-176: every triangle incident to node i as a CCW triple
        starting at its smallest vertex (the fan anchor)."""
        rows = self.triangles[np.any(self.triangles == i, axis=1)]
        out = []
        for t in rows:
            k = int(np.argmin(t))
            out.append((int(t[k]), int(t[(k + 1) % 3]), int(t[(k + 2) % 3])))
        return out

    def dump_text(self) -> str:
        """mesh.py:189-198: line-based debug dump ("mesh n t", one "p ox oy cx cy"
        row per node, one "t a b c" row per triangle; floats repr-exact)."""
        rows = [f"mesh {self.node_count} {self.triangle_count}"]
        rows += [f"p {float(o[0])!r} {float(o[1])!r} {float(c[0])!r} {float(c[1])!r}"
                 for o, c in zip(self.original_pos, self.current_pos)]
        rows += [f"t {int(a)} {int(b)} {int(c)}" for a, b, c in self.triangles]
        return "\n".join(rows) + "\n"

    def hull_nodes(self) -> np.ndarray:
        e = np.sort(np.concatenate([self.triangles[:, [0, 1]], self.triangles[:, [1, 2]],
                                    self.triangles[:, [2, 0]]]), axis=1)
        uniq, cnt = np.unique(e, axis=0, return_counts=True)
        return np.unique(uniq[cnt == 1].ravel()).astype(np.int64)


def assemble(original: np.ndarray, current: np.ndarray, tris: np.ndarray, jitter_count: int = 0) -> TriMesh:
    """Vectorised restatement of mesh.py:362-416 `_assemble`.

    Canonical triangle order (smallest vertex first, lexsorted), CSR
    neighbours sorted counter-clockwise by angle at ``original`` (ties by
    index), fans anchored at each triangle's smallest vertex.
    """
    n = len(original)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    a, b, c = tris[:, 0], tris[:, 1], tris[:, 2]
    rot0 = (a <= b) & (a <= c)
    rot1 = ~rot0 & (b <= a) & (b <= c)
    canon = np.where(rot0[:, None], tris,
                     np.where(rot1[:, None], tris[:, [1, 2, 0]], tris[:, [2, 0, 1]]))
    canon = canon[np.lexsort((canon[:, 2], canon[:, 1], canon[:, 0]))]

    src = np.concatenate([canon[:, 0], canon[:, 0], canon[:, 1], canon[:, 1], canon[:, 2], canon[:, 2]])
    dst = np.concatenate([canon[:, 1], canon[:, 2], canon[:, 0], canon[:, 2], canon[:, 0], canon[:, 1]])
    pairs = np.unique(np.stack([src, dst], axis=1), axis=0)
    src, dst = pairs[:, 0], pairs[:, 1]
    d = original[dst] - original[src]
    ang = np.arctan2(d[:, 1], d[:, 0])
    order = np.lexsort((dst, ang, src))
    src, dst = src[order], dst[order]
    csr_offsets = np.zeros(n + 1, dtype=np.int64)
    np.add.at(csr_offsets, src + 1, 1)
    csr_offsets = np.cumsum(csr_offsets)
    csr_targets = dst.astype(np.int64)

    # position of every (i, j) in i's CSR run, for the fan ordering
    rank = np.arange(len(src)) - csr_offsets[src]
    key = src * np.int64(n) + dst
    korder = np.argsort(key)
    ksorted = key[korder]

    def csr_rank(i, j):
        return rank[korder[np.searchsorted(ksorted, i * np.int64(n) + j)]]

    anchors, firsts = canon[:, 0], canon[:, 1]
    fo = np.lexsort((csr_rank(anchors, firsts), anchors))
    fan_nodes = firsts[fo].astype(np.int64)
    fan_offsets = np.zeros(n + 1, dtype=np.int64)
    np.add.at(fan_offsets, anchors + 1, 1)
    fan_offsets = np.cumsum(fan_offsets)
    return TriMesh(node_count=n, original_pos=original, current_pos=current,
                   csr_offsets=csr_offsets, csr_targets=csr_targets, fan_offsets=fan_offsets,
                   fan_nodes=fan_nodes, triangles=canon.astype(np.int64), jitter_count=jitter_count)


def _jitter_duplicates(points: np.ndarray, diag: float, rng: np.random.Generator):
    """mesh.py:336-359: split near-coincident points with a seeded jitter."""
    pts = points.copy()
    tol = 1e-9 * diag
    amp = 1e-6 * diag
    moved = 0
    for _ in range(16):
        cells: dict[tuple[int, int], int] = {}
        dup = []
        for i, (x, y) in enumerate(pts):
            key = (int(round(x / tol)), int(round(y / tol)))
            if key in cells:
                dup.append(i)
            else:
                cells[key] = i
        if not dup:
            break
        for i in dup:
            ang = rng.uniform(0.0, 2.0 * np.pi)
            r = amp * (0.5 + 0.5 * rng.uniform())
            pts[i, 0] += r * np.cos(ang)
            pts[i, 1] += r * np.sin(ang)
        moved += len(dup)
    return pts, moved


def parse_mesh_text(text: str) -> TriMesh:
    """mesh.py:201-217: inverse of TriMesh.dump_text (the CSR / fan arrays are
    rebuilt by ``assemble``)."""
    rows = [r.split() for r in text.splitlines() if r.strip()]
    if not rows or rows[0][0] != "mesh" or len(rows[0]) != 3:
        raise MeshError(f"bad mesh dump header: {' '.join(rows[0]) if rows else ''!r}")
    n, t = int(rows[0][1]), int(rows[0][2])
    if len(rows) < 1 + n + t:
        raise MeshError("truncated mesh dump")
    pts = np.array([[float(v) for v in r[1:5]] for r in rows[1:1 + n]], dtype=np.float64).reshape(n, 4)
    tris = np.array([[int(v) for v in r[1:4]] for r in rows[1 + n:1 + n + t]], dtype=np.int64).reshape(t, 3)
    return assemble(pts[:, :2].copy(), pts[:, 2:].copy(), tris, jitter_count=0)


_ORIENT_BOUND = 3.3306690738754716e-16  # Shewchuk's static orient2d bound (mesh.py:30-48)


def _orient_signs(ax, ay, bx, by, cx, cy) -> np.ndarray:
    """Exact orient2d signs, vectorised: the reference's float filter
    (mesh.py:38-48) on every row, Fraction arithmetic only where it is
    inconclusive."""
    ax, ay, bx, by, cx, cy = np.broadcast_arrays(*(np.asarray(v, dtype=np.float64) for v in (ax, ay, bx, by, cx, cy)))
    detleft = (ax - cx) * (by - cy)
    detright = (ay - cy) * (bx - cx)
    det = detleft - detright
    sign = np.sign(det).astype(np.int64)
    unsure = np.abs(det) <= _ORIENT_BOUND * (np.abs(detleft) + np.abs(detright))
    for i in np.flatnonzero(unsure):
        F = Fraction
        d = (F(ax[i]) - F(cx[i])) * (F(by[i]) - F(cy[i])) - (F(ay[i]) - F(cy[i])) * (F(bx[i]) - F(cx[i]))
        sign[i] = (d > 0) - (d < 0)
    return sign


def _cocircular_ties(pts: np.ndarray, simp: np.ndarray) -> int:
    """Interior edges whose opposite vertex lies exactly on the neighbouring
    triangle's circumcircle (exact incircle == 0): there the Delaunay
    triangulation is not unique and Qhull's choice may differ from the
    reference's Bowyer-Watson insertion order (mesh.py:220-334)."""
    tri = np.asarray(simp)
    e = np.concatenate([tri[:, [1, 2]], tri[:, [2, 0]], tri[:, [0, 1]]])
    opp = np.concatenate([tri[:, 0], tri[:, 1], tri[:, 2]])
    key = np.sort(e, axis=1)
    order = np.lexsort((key[:, 1], key[:, 0]))
    k = key[order]
    same = np.flatnonzero((k[1:] == k[:-1]).all(axis=1))
    if len(same) == 0:
        return 0
    i0, i1 = order[same], order[same + 1]
    t = i0 % len(tri)
    a, b, c = (pts[tri[t, j]] for j in range(3))
    d = pts[opp[i1]]
    adx, ady, bdx, bdy, cdx, cdy = a[:, 0] - d[:, 0], a[:, 1] - d[:, 1], b[:, 0] - d[:, 0], b[:, 1] - d[:, 1], \
        c[:, 0] - d[:, 0], c[:, 1] - d[:, 1]
    det = (adx * adx + ady * ady) * (bdx * cdy - cdx * bdy) + (bdx * bdx + bdy * bdy) * (cdx * ady - adx * cdy) + \
        (cdx * cdx + cdy * cdy) * (adx * bdy - bdx * ady)
    scale = np.abs(adx * adx + ady * ady) * (np.abs(bdx * cdy) + np.abs(cdx * bdy)) + \
        np.abs(bdx * bdx + bdy * bdy) * (np.abs(cdx * ady) + np.abs(adx * cdy)) + \
        np.abs(cdx * cdx + cdy * cdy) * (np.abs(adx * bdy) + np.abs(bdx * ady))
    ties = 0
    for i in np.flatnonzero(np.abs(det) <= 1.2e-15 * scale):
        F = Fraction
        A, B, C, D = (tuple(F(x) for x in p[i]) for p in (a, b, c, d))
        fa = [A[0] - D[0], A[1] - D[1], B[0] - D[0], B[1] - D[1], C[0] - D[0], C[1] - D[1]]
        dd = (fa[0] ** 2 + fa[1] ** 2) * (fa[2] * fa[5] - fa[4] * fa[3]) + \
            (fa[2] ** 2 + fa[3] ** 2) * (fa[4] * fa[1] - fa[0] * fa[5]) + \
            (fa[4] ** 2 + fa[5] ** 2) * (fa[0] * fa[3] - fa[2] * fa[1])
        ties += dd == 0
    return int(ties)


def delaunay(points, seed: int = 0, viewport=None) -> TriMesh:
    """Delaunay triangulation into a TriMesh (signature of mesh.py:419).

    Preprocessing mirrors the reference (jitter of coincident points,
    collinearity check); the triangulation itself comes from Qhull.
    """
    from scipy.spatial import Delaunay

    if hasattr(points, "positions"):
        viewport = viewport or points.viewport
        points = points.positions
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 2:
        raise MeshError("expected an (n, 2) point array")
    n = len(pts)
    if n < 3:
        raise DegenerateInput(f"need at least 3 points, got {n}")
    if viewport is None:
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        ext = np.where(hi > lo, hi - lo, 1.0)
        diag = float(np.hypot(*(1.1 * ext)))
    else:
        diag = float(np.hypot(viewport[2] - viewport[0], viewport[3] - viewport[1]))
    rng = np.random.default_rng(seed)
    pts, jitter_count = _jitter_duplicates(pts, diag, rng)
    # mesh.py:441-448: exact collinearity against the first two distinct points
    i1 = 1
    while i1 < n and pts[i1, 0] == pts[0, 0] and pts[i1, 1] == pts[0, 1]:
        i1 += 1
    if i1 >= n or not _orient_signs(pts[0, 0], pts[0, 1], pts[i1, 0], pts[i1, 1], pts[:, 0], pts[:, 1]).any():
        raise DegenerateInput("all points are collinear")
    try:
        simp = Delaunay(pts).simplices.astype(np.int64)
    except Exception as exc:  # scipy.spatial.QhullError: precision failure on near-degenerate input
        raise DegenerateInput(f"Qhull could not triangulate the (near-degenerate) input: {exc}") from exc
    p = pts[simp]
    sign = _orient_signs(p[:, 0, 0], p[:, 0, 1], p[:, 1, 0], p[:, 1, 1], p[:, 2, 0], p[:, 2, 1])
    if (sign == 0).any():
        raise ZeroAreaTriangle(f"Qhull returned {int((sign == 0).sum())} zero-area triangle(s)")
    simp = np.where((sign < 0)[:, None], simp[:, [0, 2, 1]], simp)
    if len(np.unique(simp)) != n:
        raise MeshError(f"triangulation left {n - len(np.unique(simp))} vertex/vertices isolated")
    ties = _cocircular_ties(pts, simp)
    if ties:
        warnings.warn(f"{ties} exactly cocircular edge(s): the Delaunay triangulation is not unique there and "
                      "may differ from the reference's Bowyer-Watson tie-breaking", RuntimeWarning, stacklevel=2)
    return assemble(pts.copy(), pts.copy(), simp, jitter_count)


def layout_topology(mesh) -> dict[str, np.ndarray]:
    """int32 device topology for the layout kernels.

    csr_off/csr_tgt: the mesh CSR (layout.py:216-231 sums in this order).
    tris: (T, 4) int32, column 3 padding (16-byte rows).
    inc_off/inc: per vertex, entries ``triangle << 2 | corner`` sorted by
    (corner, triangle) == the order in which np.bincount accumulates each
    corner pass of layout.py:240-255.
    """
    n = int(mesh.node_count)
    tris = np.asarray(mesh.triangles, dtype=np.int64).reshape(-1, 3)
    t = len(tris)
    if n >= 2**31 or t >= 2**29:
        raise MeshError("mesh too large for int32 topology")
    tri4 = np.zeros((t, 4), dtype=np.int32)
    tri4[:, :3] = tris
    vert = tris.T.ravel()                        # corner-major: k*T + t
    corner = np.repeat(np.arange(3), t)
    tidx = np.tile(np.arange(t), 3)
    order = np.lexsort((tidx, corner, vert))     # by vertex, then corner, then triangle
    inc = ((tidx[order] << 2) | corner[order]).astype(np.int32)
    inc_off = np.zeros(n + 1, dtype=np.int64)
    np.add.at(inc_off, vert + 1, 1)
    inc_off = np.cumsum(inc_off).astype(np.int32)
    return dict(
        csr_off=np.asarray(mesh.csr_offsets, dtype=np.int32),
        csr_tgt=np.asarray(mesh.csr_targets, dtype=np.int32),
        tris=tri4,
        inc_off=inc_off,
        inc=inc,
    )
