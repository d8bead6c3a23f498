"""Shared test helpers: golden meshes as TriMesh objects."""

from paper_1408_0677_b200.mesh import TriMesh


def golden_mesh(g, pos=None):
    orig = g["original_pos"]
    return TriMesh(
        node_count=len(orig),
        original_pos=orig.copy(),
        current_pos=(orig if pos is None else pos).copy(),
        csr_offsets=g["csr_offsets"],
        csr_targets=g["csr_targets"],
        fan_offsets=g["fan_offsets"],
        fan_nodes=g["fan_nodes"],
        triangles=g["triangles"],
    )
