"""Planarity-preserving force-directed layout on the GPU.

Drop-in mirror of the reference's ``layout`` module
(/root/reference/pkg/src/mdcontour/layout.py): ``LayoutParams`` /
``defaults_for`` / ``LayoutState`` / ``initial_state`` / ``layout_step`` /
``layout_run`` / ``interpolate_layout`` / ``count_orientation_flips`` keep
their signatures, defaults and errors.  Each Jacobi step runs in libmdc
(kd-tree build + warp-cooperative Barnes-Hut + one fused per-vertex
spring/node-edge/cap/clamp/update kernel, positions double-buffered in HBM);
``layout_run`` replays a captured CUDA graph per step and moves positions
across PCIe once per run, not once per step.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .mesh import layout_topology


class TOutOfRange(Exception):
    pass


@dataclass(frozen=True)
class LayoutParams:
    """layout.py:26-67."""

    repulsion_c: float
    spring_scale: float
    desired_edge_d: float
    softening_eta: float
    initial_temp: float
    decay_lambda: float
    iterations: int = 500
    bh_theta: float = 0.5

    def __post_init__(self):
        if self.repulsion_c <= 0 or self.spring_scale <= 0 or self.desired_edge_d <= 0:
            raise ValueError("force constants must be positive")
        if self.softening_eta <= 0 or self.initial_temp <= 0 or self.bh_theta <= 0:
            raise ValueError("softening, temperature, and opening angle must be positive")
        if not 0.0 < self.decay_lambda < 1.0:
            raise ValueError("decay_lambda must lie in (0, 1)")
        if self.iterations < 0:
            raise ValueError("iterations must be non-negative")

    @classmethod
    def defaults_for(cls, mesh, iterations: int = 500, **overrides) -> "LayoutParams":
        d = median_edge_length(mesh)
        base = dict(
            repulsion_c=d * d,
            spring_scale=1.0,
            desired_edge_d=d,
            softening_eta=1e-7 * d,
            initial_temp=d,
            decay_lambda=0.99,
            iterations=iterations,
            bh_theta=0.5,
        )
        base.update(overrides)
        return cls(**base)


def median_edge_length(mesh, positions: np.ndarray | None = None) -> float:
    """layout.py:70-76."""
    pos = mesh.original_pos if positions is None else positions
    src = np.repeat(np.arange(mesh.node_count), np.diff(mesh.csr_offsets))
    dst = mesh.csr_targets
    keep = src < dst
    lengths = np.hypot(*(pos[src[keep]] - pos[dst[keep]]).T)
    return float(np.median(lengths)) if len(lengths) else 1.0


@dataclass(frozen=True)
class LayoutState:
    mesh: object
    iteration: int
    temperature: float
    relaxed_pos: np.ndarray


def temperature_schedule(t0: float, lam: float, k: int) -> np.ndarray:
    """t_i for i = 0..k-1 by repeated multiplication, exactly as the
    reference advances ``state.temperature * decay_lambda`` (layout.py:284)."""
    out = np.empty(k)
    t = t0
    for i in range(k):
        out[i] = t
        t = t * lam
    return out


LEAF_SIZE = 32  # bhtree.py:74 passes leaf_size=32 on the layout path


class LayoutEngine:
    """Device-resident topology + libmdc plan for one mesh and parameter set."""

    def __init__(self, mesh, params: LayoutParams, device=None, leaf: int = LEAF_SIZE, part=(0, 1), pos=None):
        lib = _lib.require_cuda()
        self.lib = lib
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.params = params
        self.n = int(mesh.node_count)
        topo = layout_topology(mesh)
        dev = self.device
        self.topo = {k: torch.as_tensor(v).to(dev) for k, v in topo.items()}
        self.ntri = int(topo["tris"].shape[0])
        # `pos` may be an external (n, 2) fp64 device tensor, e.g. an
        # inter-process buffer for the peer-memory exchange
        self.pos = torch.empty((self.n, 2), dtype=torch.float64, device=dev) if pos is None else pos
        self.ws = torch.empty(int(lib.mdc_layout_workspace_bytes(self.n, leaf)), dtype=torch.uint8, device=dev)
        self.leaf = leaf
        self.part = (int(part[0]), int(part[1]))
        self._plans = {}
        self.temps = None
        self.gather_send = None  # all-gather exchange: packed owned-slice buffer (GatherLayout)

    def _args(self, dbg=None) -> _lib.MdcLayoutArgs:
        p = self.params
        a = _lib.MdcLayoutArgs()
        a.n, a.ntri, a.leaf = self.n, self.ntri, self.leaf
        a.c, a.spring, a.dlen = p.repulsion_c, p.spring_scale, p.desired_edge_d
        a.eta, a.theta = p.softening_eta, p.bh_theta
        a.csr_off, a.csr_tgt = _lib.ptr(self.topo["csr_off"]), _lib.ptr(self.topo["csr_tgt"])
        a.tris, a.inc_off, a.inc = _lib.ptr(self.topo["tris"]), _lib.ptr(self.topo["inc_off"]), _lib.ptr(self.topo["inc"])
        a.pos = _lib.ptr(self.pos)
        a.workspace, a.workspace_bytes = _lib.ptr(self.ws), self.ws.numel()
        a.part_rank, a.part_world = self.part
        if dbg is not None:
            a.dbg_bh, a.dbg_force, a.dbg_scale = (_lib.ptr(t) for t in dbg)
        return a

    def plan(self, debug: bool = False):
        key = "dbg" if debug else "run"
        if key not in self._plans:
            dbg = None
            if debug:
                self.dbg = (torch.empty((self.n, 2), dtype=torch.float64, device=self.device),
                            torch.empty((self.n, 2), dtype=torch.float64, device=self.device),
                            torch.empty(self.n, dtype=torch.float64, device=self.device))
                dbg = self.dbg
            self._args_keep = a = self._args(dbg)
            h = ctypes.c_void_p()
            _lib.check(self.lib.mdc_layout_plan_create(ctypes.byref(a), ctypes.byref(h), _lib.stream_ptr()),
                       "mdc_layout_plan_create")
            if self.gather_send is not None:  # before any step is captured into a graph
                _lib.check(self.lib.mdc_layout_set_gather(h, _lib.ptr(self.gather_send)), "mdc_layout_set_gather")
            self._plans[key] = h
        return self._plans[key]

    def set_positions(self, pos) -> None:
        self.pos.copy_(torch.as_tensor(np.ascontiguousarray(pos, dtype=np.float64)))

    def run(self, temps: np.ndarray, use_graph: bool = True, debug: bool = False) -> None:
        """len(temps) steps in place on ``self.pos`` (device)."""
        k = len(temps)
        if k == 0:
            return
        if self.temps is None or self.temps.numel() < k or debug:
            self.temps = torch.as_tensor(np.asarray(temps, dtype=np.float64)).to(self.device)
            # captured graphs bind the temps pointer: drop them with the buffer
            self._drop("run")
        else:
            self.temps[:k].copy_(torch.as_tensor(np.asarray(temps, dtype=np.float64)))
        h = self.plan(debug)
        with _lib.nvtx(f"layout.steps x{k}"):
            _lib.check(self.lib.mdc_layout_steps(h, k, _lib.ptr(self.temps), int(use_graph and not debug),
                                                 _lib.stream_ptr()), "mdc_layout_steps")

    PHASES = ("sorts", "tree", "bh_traversal", "bh_combine", "local")

    def profile_step(self, temperature: float, count: bool = True) -> dict:
        """One eager step on ``self.pos`` with per-phase device times
        (mdc_layout_profile) and, optionally, the BH interaction counts."""
        t = torch.tensor([float(temperature)], dtype=torch.float64, device=self.device)
        ms = (ctypes.c_float * 5)()
        cnt = (ctypes.c_int64 * 4)()
        _lib.check(self.lib.mdc_layout_profile(self.plan(), _lib.ptr(t), ctypes.cast(ms, ctypes.c_void_p),
                                               ctypes.cast(cnt, ctypes.c_void_p) if count else None,
                                               _lib.stream_ptr()), "mdc_layout_profile")
        out = {"ms": dict(zip(self.PHASES, (float(v) for v in ms)))}
        if count:
            out["leaf_pairs"], out["monopoles"], out["node_tests"], out["lane_slots"] = (int(v) for v in cnt)
        return out

    def repulsion(self, pts: torch.Tensor) -> torch.Tensor:
        out = torch.empty_like(pts)
        _lib.check(self.lib.mdc_layout_repulsion(self.plan(), _lib.ptr(pts), _lib.ptr(out), _lib.stream_ptr()),
                   "mdc_layout_repulsion")
        return out

    def _drop(self, key):
        h = self._plans.pop(key, None)
        if h is not None:
            self.lib.mdc_layout_plan_destroy(h)

    def __del__(self):
        try:
            for key in list(self._plans):
                self._drop(key)
        except Exception:
            pass


def _engine(mesh, params: LayoutParams) -> LayoutEngine:
    """One engine per (mesh, params), cached on the mesh like the reference
    caches its constraint grouping (layout.py:270-273)."""
    cache = mesh.__dict__.setdefault("_mdc_layout_engines", {})
    key = (params.repulsion_c, params.spring_scale, params.desired_edge_d, params.softening_eta,
           params.bh_theta, torch.cuda.current_device())
    eng = cache.get(key)
    if eng is None:
        eng = LayoutEngine(mesh, params)
        cache[key] = eng
    return eng


def initial_state(mesh, params: LayoutParams) -> LayoutState:
    return LayoutState(mesh=mesh, iteration=0, temperature=params.initial_temp,
                       relaxed_pos=mesh.current_pos.copy())


def layout_step(state: LayoutState, params: LayoutParams) -> LayoutState:
    """layout.py:266-286: one synchronous annealed update from a frozen snapshot."""
    mesh = state.mesh
    eng = _engine(mesh, params)
    eng.set_positions(mesh.current_pos)
    eng.run(np.array([state.temperature]), use_graph=False)
    mesh.current_pos = eng.pos.cpu().numpy()
    return LayoutState(mesh=mesh, iteration=state.iteration + 1,
                       temperature=state.temperature * params.decay_lambda,
                       relaxed_pos=mesh.current_pos.copy())


def layout_run(mesh, params: LayoutParams) -> LayoutState:
    """layout.py:298-302: ``params.iterations`` steps, device-resident."""
    state = initial_state(mesh, params)
    k = params.iterations
    if k == 0:
        return state
    temps = temperature_schedule(state.temperature, params.decay_lambda, k + 1)
    eng = _engine(mesh, params)
    eng.set_positions(mesh.current_pos)
    eng.run(temps[:k], use_graph=True)
    mesh.current_pos = eng.pos.cpu().numpy()
    return LayoutState(mesh=mesh, iteration=k, temperature=float(temps[k]),
                       relaxed_pos=mesh.current_pos.copy())


def layout_debug_step(mesh, pos: np.ndarray, params: LayoutParams, temperature: float):
    """One step from ``pos`` returning (new_pos, bh, total_force, clamp_s) --
    the per-component teacher-forced parity hook (layout.py:259-280)."""
    eng = _engine(mesh, params)
    eng.set_positions(pos)
    eng.run(np.array([temperature]), use_graph=False, debug=True)
    bh, force, s = (t.cpu().numpy() for t in eng.dbg)
    return eng.pos.cpu().numpy(), bh, force, s


class IpcBuffer:
    """A device buffer shareable with other processes (cudaIpc, mdc_ipc_*):
    ``tensor`` views it in this process, ``handle`` (64 bytes) opens it in a
    peer process (``IpcBuffer.open``)."""

    def __init__(self, shape, dtype=torch.float64):
        self.lib = _lib.require_cuda()
        self.shape, self.dtype = tuple(shape), dtype
        nbytes = int(np.prod(self.shape)) * torch.empty((), dtype=dtype).element_size()
        ptr, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        _lib.check(self.lib.mdc_ipc_alloc(nbytes, ctypes.byref(ptr), handle), "mdc_ipc_alloc")
        self.ptr, self.handle = ptr.value, handle.raw
        self.tensor = _wrap_device(self.ptr, self.shape, dtype)

    @staticmethod
    def open(handle: bytes) -> int:
        lib = _lib.require_cuda()
        ptr = ctypes.c_void_p()
        _lib.check(lib.mdc_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)), "mdc_ipc_open")
        return ptr.value

    @staticmethod
    def close(ptr: int) -> None:
        _lib.check(_lib.require_cuda().mdc_ipc_close(ctypes.c_void_p(ptr)), "mdc_ipc_close")

    def free(self) -> None:
        if self.ptr:
            self.tensor = None
            _lib.check(self.lib.mdc_ipc_free(ctypes.c_void_p(self.ptr)), "mdc_ipc_free")
            self.ptr = None


def _wrap_device(ptr: int, shape, dtype) -> torch.Tensor:
    """A torch view of raw device memory (__cuda_array_interface__, no copy)."""
    typestr = {torch.float64: "<f8", torch.float32: "<f4", torch.int32: "<i4"}[dtype]

    class _View:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_View(), device=torch.device("cuda", torch.cuda.current_device()))


def layout_run_partitioned(mesh, params: LayoutParams, group=None, exchange: str = "allgather") -> LayoutState:
    """layout_run with the vertices partitioned over the ranks of ``group``
    (SURVEY.md §8e, config 4): every rank rebuilds the kd-tree from the full
    snapshot and updates its leaf-order slice of the vertices; the slices are
    reassembled each iteration by

    * ``allgather`` (default, the north_star's exchange): the step packs the
      owned slice in leaf order, one all_gather_into_tensor (NCCL over
      NVLink on the GPU box) collects every slice, ``mdc_layout_scatter``
      writes them back in vertex order -- n x 16 bytes received per rank;
    * ``allreduce``: non-owned entries are exactly 0.0 and one SUM
      all-reduce adds the slices (about twice the bytes);
    * ``p2p``: the step kernel stores its slice into every rank's next
      position buffer over NVLink (cudaIpc-mapped peer buffers, one host
      barrier per step).

    All three are bit-identical to the single-GPU trajectory."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    state = initial_state(mesh, params)
    k = params.iterations
    temps = temperature_schedule(state.temperature, params.decay_lambda, k + 1)
    if exchange not in ("allgather", "allreduce", "p2p"):
        raise ValueError(f"exchange must be 'allgather', 'allreduce' or 'p2p', got {exchange!r}")
    if exchange == "p2p" and world > 1:
        pos = _run_p2p(mesh, params, temps[:k], world, rank, group)
    elif exchange == "allgather" and world > 1:
        ag = GatherLayout(mesh, params, group)
        ag.eng.set_positions(mesh.current_pos)
        for it in range(k):
            ag.step(temps[it:it + 1])
        pos = ag.eng.pos.cpu().numpy()
    else:
        eng = LayoutEngine(mesh, params, part=(rank, world))
        eng.set_positions(mesh.current_pos)
        for it in range(k):
            eng.run(temps[it:it + 1], use_graph=True)
            if world > 1:
                dist.all_reduce(eng.pos, op=dist.ReduceOp.SUM, group=group)
        pos = eng.pos.cpu().numpy()
    mesh.current_pos = pos
    return LayoutState(mesh=mesh, iteration=k, temperature=float(temps[k]) if k else params.initial_temp,
                       relaxed_pos=mesh.current_pos.copy())


class GatherLayout:
    """Vertex-partitioned layout with the all-gather exchange: per step, the
    captured step graph (tree + BH + local update of this rank's leaf-order
    slice, packed into ``send``), one ``all_gather_into_tensor`` and one
    scatter kernel back to vertex order (``mdc_layout_scatter``)."""

    def __init__(self, mesh, params: LayoutParams, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.eng = LayoutEngine(mesh, params, part=(self.rank, self.world))
        n = self.eng.n
        self.chunk = -(-n // self.world)
        dev = self.eng.device
        self.send = torch.zeros((self.chunk, 2), dtype=torch.float64, device=dev)
        self.recv = torch.empty((self.world * self.chunk, 2), dtype=torch.float64, device=dev)
        self.eng.gather_send = self.send  # applied to every plan the engine creates

    def step(self, temps) -> None:
        self.eng.run(temps, use_graph=True)
        with _lib.nvtx("layout.allgather"):
            self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        _lib.check(self.eng.lib.mdc_layout_scatter(self.eng.plan(), _lib.ptr(self.recv), self.chunk,
                                                   _lib.stream_ptr()), "mdc_layout_scatter")


class P2PLayout:
    """Vertex-partitioned layout whose per-iteration exchange is done by the
    step kernel itself: each rank stores its owned vertices' new positions
    into every rank's next-parity buffer (cudaIpc-mapped, NVLink stores);
    one stream sync + host barrier per step orders the ranks."""

    def __init__(self, mesh, params: LayoutParams, temps, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        n = int(mesh.node_count)
        self.bufs = [IpcBuffer((n, 2)), IpcBuffer((n, 2))]
        handles = [None] * self.world
        dist.all_gather_object(handles, (self.bufs[0].handle, self.bufs[1].handle), group=group)
        self.opened = []
        peers = [[0] * self.world, [0] * self.world]
        for r in range(self.world):
            for par in (0, 1):
                if r == self.rank:
                    peers[par][r] = self.bufs[par].ptr
                else:
                    ptr = IpcBuffer.open(handles[r][par])
                    self.opened.append(ptr)
                    peers[par][r] = ptr
        self.eng = LayoutEngine(mesh, params, part=(self.rank, self.world), pos=self.bufs[0].tensor)
        self.plan = self.eng.plan()
        arr0 = (ctypes.c_void_p * self.world)(*peers[0])
        arr1 = (ctypes.c_void_p * self.world)(*peers[1])
        _lib.check(self.eng.lib.mdc_layout_set_peers(self.plan, self.world, arr0, arr1), "mdc_layout_set_peers")
        self.temps = torch.as_tensor(np.asarray(temps, dtype=np.float64)).to(self.eng.device)
        self.it = 0

    def reset(self, positions) -> None:
        """Start a trajectory from ``positions`` (every rank passes the same)."""
        self.eng.set_positions(positions)
        _lib.check(self.eng.lib.mdc_layout_reset_counter(self.plan, _lib.stream_ptr()), "mdc_layout_reset_counter")
        self.it = 0
        torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)

    def step(self) -> None:
        _lib.check(self.eng.lib.mdc_layout_step_parity(self.plan, self.it & 1, _lib.ptr(self.temps), 1,
                                                       _lib.stream_ptr()), "mdc_layout_step_parity")
        self.it += 1
        torch.cuda.current_stream().synchronize()  # this rank's peer stores are done
        self.dist.barrier(group=self.group)         # ... and every other rank's

    def positions(self) -> torch.Tensor:
        """The current snapshot (a view of this rank's buffer)."""
        return self.bufs[self.it & 1].tensor

    def close(self) -> None:
        self.eng = None
        self.dist.barrier(group=self.group)  # nobody frees while a peer still maps the buffers
        for ptr in self.opened:
            IpcBuffer.close(ptr)
        self.opened = []
        torch.cuda.synchronize()
        for b in self.bufs:
            b.free()


def _run_p2p(mesh, params, temps, world, rank, group):
    run = P2PLayout(mesh, params, temps, group)
    try:
        run.reset(mesh.current_pos)
        for _ in range(len(temps)):
            run.step()
        return run.positions().cpu().numpy()
    finally:
        run.close()


# ---- scalar force laws (layout.py:87-116; Eqs. 1-3 of the paper) ----------
# Per-pair restatements for tests and inspection; the step evaluates the same
# laws on the GPU (bh_kernel / local_kernel).

def repulsive_force(v, vi, params: LayoutParams) -> np.ndarray:
    """Softened inverse-square push of v away from vi: C d / (|d|^3 + eta)."""
    d = np.asarray(v, dtype=float) - np.asarray(vi, dtype=float)
    r = float(np.hypot(d[0], d[1]))
    return params.repulsion_c / (r ** 3 + params.softening_eta) * d


def spring_force(v, vi, params: LayoutParams) -> np.ndarray:
    """Log spring along a mesh edge, zero at the desired edge length D."""
    d = np.asarray(v, dtype=float) - np.asarray(vi, dtype=float)
    r = float(np.hypot(d[0], d[1]))
    if r == 0.0:
        return np.zeros(2)
    return -params.spring_scale * np.log((r + params.softening_eta) / params.desired_edge_d) * d


def node_edge_force(v, vi, vj, params: LayoutParams) -> np.ndarray:
    """Push of v away from the line through its opposite edge (vi, vj)."""
    v = np.asarray(v, dtype=float)
    a = np.asarray(vi, dtype=float)
    e = np.asarray(vj, dtype=float) - a
    ee = float(e @ e)
    if ee == 0.0:
        return np.zeros(2)
    r = a + float((v - a) @ e) / ee * e - v  # foot of the perpendicular minus v
    nr = float(np.hypot(r[0], r[1]))
    if nr < 1e-12:
        return np.zeros(2)
    return -params.repulsion_c / (nr ** 2 + params.softening_eta) * (r / nr)


def clamp_displacement(node_idx: int, proposed, mesh, params: LayoutParams) -> np.ndarray:
    """layout.py:187-213, one node: ``proposed`` scaled so the node crosses no
    limiting line of an incident triangle (direction kept)."""
    proposed = np.asarray(proposed, dtype=float)
    if not proposed.any():
        return proposed.copy()
    pos = mesh.current_pos
    p = pos[node_idx]
    factor = 1.0
    for tri in mesh.triangles[np.any(mesh.triangles == node_idx, axis=1)]:
        a, b, c = pos[tri[0]], pos[tri[1]], pos[tri[2]]
        mab, mbc, mca = 0.5 * (a + b), 0.5 * (b + c), 0.5 * (c + a)
        for pt, other in ((mab, mca), (mab, mbc), (mbc, mca)):
            nrm = np.array([pt[1] - other[1], other[0] - pt[0]])
            ln = float(np.hypot(nrm[0], nrm[1]))
            if ln == 0.0:
                continue
            nrm = nrm / ln
            signed = float((p - pt) @ nrm)
            allowed = max(0.0, abs(signed) - params.softening_eta)
            toward = -(1.0 if signed >= 0.0 else -1.0) * float(proposed @ nrm)
            if toward > allowed:
                factor = min(factor, allowed / toward)
    return proposed * max(factor, 0.0)


def clamp_factors(pos: np.ndarray, disp: np.ndarray, tris: np.ndarray, eta: float, groups=None) -> np.ndarray:
    """layout.py:160-184 on the GPU (mdc_layout_clamp_factors): per-node factor
    in [0, 1] keeping every node eta clear of every limiting line of every
    triangle it belongs to.  ``groups`` (the reference's cached grouping) is
    accepted and unused."""
    lib = _lib.require_cuda()
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    disp = np.ascontiguousarray(disp, dtype=np.float64)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    n = len(pos)
    if len(tris) == 0:
        return np.ones(n)
    corner = np.repeat(np.arange(3, dtype=np.int64)[None, :], len(tris), axis=0).ravel()
    tri_id = np.repeat(np.arange(len(tris), dtype=np.int64), 3)
    node = tris.ravel()
    order = np.argsort(node, kind="stable")
    inc = ((tri_id << 2) | corner)[order].astype(np.int32)
    inc_off = np.concatenate([[0], np.cumsum(np.bincount(node, minlength=n))]).astype(np.int32)
    tris4 = np.zeros((len(tris), 4), dtype=np.int32)
    tris4[:, :3] = tris
    dev = torch.device("cuda", torch.cuda.current_device())
    t = [torch.as_tensor(x).to(dev) for x in (pos, disp, tris4, inc_off, inc)]
    out = torch.empty(n, dtype=torch.float64, device=dev)
    _lib.check(lib.mdc_layout_clamp_factors(n, *(_lib.ptr(x) for x in t), float(eta), _lib.ptr(out),
                                            _lib.stream_ptr()), "mdc_layout_clamp_factors")
    return out.cpu().numpy()


def total_forces(pos: np.ndarray, mesh, params: LayoutParams) -> np.ndarray:
    """layout.py:259-263 on the GPU: Barnes-Hut + spring + node-edge forces at
    ``pos`` (the step's force before the temperature cap and the clamp)."""
    _, _, force, _ = layout_debug_step(mesh, np.asarray(pos, dtype=np.float64), params, params.initial_temp)
    return force


def dump_layout_text(state: LayoutState) -> str:
    """layout.py:323-329: the mesh dump followed by "layout <iteration>
    <temperature>" and one "r x y" row per node (floats repr-exact)."""
    rows = [state.mesh.dump_text().rstrip("\n"), f"layout {state.iteration} {state.temperature!r}"]
    rows += [f"r {float(x)!r} {float(y)!r}" for x, y in state.relaxed_pos]
    return "\n".join(rows) + "\n"


def parse_layout_text(text: str) -> LayoutState:
    """layout.py:332-350: inverse of dump_layout_text."""
    from .mesh import parse_mesh_text

    rows = [r for r in text.splitlines() if r.strip()]
    k = next(i for i, r in enumerate(rows) if r.startswith("layout "))
    mesh = parse_mesh_text("\n".join(rows[:k]))
    _, iteration, temperature = rows[k].split()
    relaxed = np.array([[float(v) for v in r.split()[1:3]] for r in rows[k + 1:]], dtype=np.float64)
    if len(relaxed) != mesh.node_count:
        raise ValueError("relaxed position count does not match the mesh")
    return LayoutState(mesh=mesh, iteration=int(iteration), temperature=float(temperature), relaxed_pos=relaxed)


def interpolate_layout(state: LayoutState, t: float) -> np.ndarray:
    """layout.py:305-309."""
    if not 0.0 <= t <= 1.0:
        raise TOutOfRange(f"relax parameter must be in [0, 1], got {t}")
    return (1.0 - t) * state.mesh.original_pos + t * state.relaxed_pos


def count_orientation_flips(mesh, positions: np.ndarray) -> int:
    """layout.py:312-320."""
    def areas(p):
        a, b, c = p[mesh.triangles[:, 0]], p[mesh.triangles[:, 1]], p[mesh.triangles[:, 2]]
        return 0.5 * ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0]))
    ref = np.sign(areas(mesh.original_pos))
    cur = np.sign(areas(positions))
    return int(np.count_nonzero(ref != cur))
