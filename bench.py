#!/usr/bin/env python
"""Benchmark of the north-star workload (BASELINE.json):

  MLS Mpixel.dim/s -- affine MLS (alpha 1.5, fp32) of all d target dims over a
  W x H raster, fused band epilogue + fp64 snap, row-band sharded over the
  ranks (point data broadcast once per frame over NCCL); plus the layout
  metric (vertex-iters/s of `iterations` planarity-preserving steps).

Default workload: config 3 (100k points x 32 dims, 3840 x 2160, 500 layout
iterations) on synthetic Gaussian-mixture data.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3]
  python bench.py --impl reference ...   # the CPU reference arm (oracle port)
"""

from __future__ import annotations

import argparse
import hashlib
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(n=150, d=4, seed=1, W=256, H=256, iters=50),
    2: dict(n=10_000, d=16, seed=2, W=1920, H=1080, iters=500),
    3: dict(n=100_000, d=32, seed=3, W=3840, H=2160, iters=500),
    4: dict(n=1_000_000, d=64, seed=4, W=7680, H=4320, iters=500),
}
METRIC = "MLS Mpixel·dim/s (4K, N=100k, d=32) at 1/2/4/8 GPU; layout vertex-iters/s"
UNIT = "Mpixel*dim/s"


def gmm(n, d, seed):
    """SURVEY.md Appendix A.1 Gaussian-mixture generator."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(0, 4, (8, d))
    scales = rng.uniform(0.5, 1.5, 8)
    lab = rng.integers(0, 8, n)
    return centers[lab] + rng.normal(0, 1, (n, d)) * scales[lab, None]


def workload_name(cfg):
    return (f"config{cfg['id']}: affine MLS alpha=1.5 fp32, {cfg['n']} points x {cfg['d']} dims, "
            f"{cfg['W']}x{cfg['H']}, fused bands + RGBA8 band shading + snap; layout {cfg['iters']} iterations")


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md "clocks DURING the timed region")

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU arm (oracle = C restatement of the reference, all host threads)

def cpu_mls_sample(positions, raw, cfg, target_s=10.0, dims=4, nrows=16):
    """Time the reference's affine kernel (_kernels.affine_field, restated in
    C: oracle/mdc_oracle.c, all host threads) the way the reference renders:
    one call per dimension with targets (q_k, 0) (cli.py:143-165), on
    `nrows` rows spread top to bottom over the frame (every `stride`-th
    column when a full row would overrun the time budget), `dims` dims."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    O.set_threads(os.cpu_count() or 1)
    W, H = cfg["W"], cfg["H"]
    rows = sorted({int(r) for r in np.linspace(0, H - 1, nrows)})
    vp = O.viewport(positions, W, H)
    xs, ys = O.pixel_centers(vp, W, H)
    pm = positions.mean(axis=0)
    pc = positions - pm

    def run(cols, k):
        tv = np.column_stack([raw[:, k], np.zeros(len(raw))])
        qm = tv.mean(axis=0)
        O.mls_kernel("affine", xs[rows][:, cols].ravel() - pm[0], ys[rows][:, cols].ravel() - pm[1], pc,
                     tv - qm, 1.5)

    probe = np.arange(0, W, max(1, W // 64))
    t0 = time.perf_counter()
    run(probe, 0)
    per_px = (time.perf_counter() - t0) / (len(rows) * len(probe))
    stride = max(1, int(np.ceil(per_px * len(rows) * W * dims / target_s)))
    cols = np.arange(0, W, stride)
    t0 = time.perf_counter()
    for k in range(dims):
        run(cols, k)
    dt = time.perf_counter() - t0
    px = len(rows) * len(cols)
    return {"value": px * dims / dt / 1e6, "unit": UNIT, "cores": O.max_threads(),
            "kind": "port", "seconds": dt,
            "sample": f"affine_field restated in C (oracle/mdc_oracle.c), one call per dim: {len(rows)} rows "
                      f"spread over the frame x {len(cols)} px (every {stride}th column), {dims} dims, "
                      f"N={len(positions)} controls at the laid-out positions, fp64"}


def cpu_layout_sample(mesh, params, states, steps=10):
    """layout_step restated in C (oracle, all host threads): `steps` steps from
    iteration 0 and `steps` from iteration 250."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    p = {k: getattr(params, k) for k in ("repulsion_c", "spring_scale", "desired_edge_d",
                                         "softening_eta", "bh_theta", "initial_temp", "decay_lambda")}
    dt, done = 0.0, []
    for it, pos in sorted(states.items()):
        temp = params.initial_temp * params.decay_lambda ** it
        t0 = time.perf_counter()
        O.layout_run(pos, mesh.csr_offsets, mesh.csr_targets, mesh.triangles, p, steps, temperature=temp)
        dt += time.perf_counter() - t0
        done.append(it)
    nsteps = steps * len(done)
    return {"value": mesh.node_count * nsteps / dt, "unit": "vertex-iters/s",
            "cores": O.max_threads(), "kind": "port",
            "sample": f"{steps} layout_steps restated in C from each of iterations {done}, N={mesh.node_count}"}


def config_dict(cfg, world):
    """One config dict for both arms (the driver compares them)."""
    return {"workload": workload_name(cfg), "points": cfg["n"], "dims": cfg["d"], "width": cfg["W"],
            "height": cfg["H"], "layout_iterations": cfg["iters"], "parallelism": f"rowband{world}",
            "l2": "flushed between frames (256 MiB write)"}


def laid_out_positions(cfg, mesh):
    """The GPU arm's positions after 250 and `iters` layout iterations, from
    bench_data/ (written by tools/make_bench_positions.py from this repo's
    deterministic GPU layout); PCA positions when no fixture matches."""
    path = os.path.join(ROOT, "bench_data", f"config{cfg['id']}_positions.npz")
    try:
        z = np.load(path)
        # the CPU arm's PCA (oracle) may differ from the GPU's in the last bits:
        # same mesh topology and positions equal to 1e-9 of the extent
        ext = float(np.ptp(mesh.original_pos))
        if int(z["iters"]) == cfg["iters"] and z["pos_final"].shape == mesh.original_pos.shape and \
                str(z["triangles_sha256"]) == hashlib.sha256(
                    np.ascontiguousarray(mesh.triangles.astype(np.int64)).tobytes()).hexdigest() and \
                np.allclose(z["original_pos"], mesh.original_pos, rtol=0, atol=1e-9 * ext):
            return {0: mesh.original_pos, 250: z["pos_250"]}, z["pos_final"]
    except (OSError, KeyError):
        pass
    return {0: mesh.original_pos}, mesh.original_pos


def build_scene(cfg, device_pca=True):
    from paper_1408_0677_b200 import dataset as D
    from paper_1408_0677_b200 import mesh as M
    from paper_1408_0677_b200 import projection as P

    X = gmm(cfg["n"], cfg["d"], cfg["seed"])
    ds = D.normalize(D.Dataset(names=[f"d{i}" for i in range(cfg["d"])], data=X))
    if device_pca:
        model, cloud = P.pca_project(ds)
        positions = cloud.positions
    else:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        positions = O.pca_project(ds.data)[3]
    mesh = M.delaunay(positions, seed=0)
    raw = np.column_stack([ds.raw_column(nm) for nm in ds.names])
    return ds, mesh, raw


def run_reference(args, cfg, rank):
    if rank != 0:
        return
    from paper_1408_0677_b200.layout import LayoutParams

    ds, mesh, raw = build_scene(cfg, device_pca=False)
    params = LayoutParams.defaults_for(mesh, iterations=cfg["iters"])
    states, positions = laid_out_positions(cfg, mesh)
    sample_s = max(1.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        cpu_mls_sample(positions, raw, cfg, target_s=sample_s)
    vals, secs = [], []
    for _ in range(args.steps):
        s = cpu_mls_sample(positions, raw, cfg, target_s=sample_s)
        vals.append(s["value"])
        secs.append(s["seconds"])
    value = statistics.median(vals)
    lay = cpu_layout_sample(mesh, params, states, steps=10 if cfg["n"] <= 200_000 else 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args.gpus),
        "cpu_baseline": {k: s[k] for k in ("value", "unit", "cores", "kind", "sample")} | {"value": value},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "layout": {"metric": "vertex-iters/s", **lay},
    }
    print(json.dumps(line), flush=True)


def measure_peaks(lib, torch):
    """Live FFMA / DFMA peaks on this GPU (FLOP/s), CUDA-event timed."""
    sms = lib.mdc_num_sms()
    sink = torch.zeros(4, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    out = {}
    for name, fn, iters in (("fp32", lib.mdc_peak_ffma, 4096), ("fp64", lib.mdc_peak_dfma, 1024)):
        blocks = sms * 8
        fn(ctypes.c_void_p(sink.data_ptr()), blocks, 64, s)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(3):
            e0.record()
            fn(ctypes.c_void_p(sink.data_ptr()), blocks, iters, s)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        flops = blocks * 256.0 * iters * 16 * 8 * 2
        out[name] = flops / (best * 1e-3)
    return out


# fp64 pipe ops per BH unit (bh_kernel source): leaf pair = 2 sub + 2 fma (r2)
# + 5 (sqrt from the rsqrt.approx seed + 2nd-order series) + 1 fma (r2 r + eta)
# + 3 (rcp.approx + correction) + 2 fma (force) = 15; monopole = 16 (+1 mass);
# opening test = 9 (box offsets, squared distance, size^2 vs theta^2 d2 with the
# guard band; the exact IEEE sqrt path is only taken inside the band).
BH_OPS = {"leaf_pairs": 15, "monopoles": 16, "node_tests": 9}
LOCAL_BYTES_PER_VERTEX = 204  # SURVEY.md §8d algorithmic bytes per vertex-iteration


def layout_roofline(eng, params, lib, torch):
    """Per-phase device times of one eager step after the timed run
    (mdc_layout_profile) and the two layout roofs of SURVEY.md §8d: BH on the
    FP64 pipe (executed lane-ops x 2 vs the live DFMA peak) and the local
    sweep against HBM (algorithmic bytes; the working set is L2-resident, so
    frac may exceed 1)."""
    prof = eng.profile_step(params.initial_temp * params.decay_lambda ** params.iterations)
    ms = prof["ms"]
    n = eng.n
    peaks = measure_peaks(lib, torch)
    ops = sum(BH_OPS[k] * prof[k] for k in BH_OPS)
    bh_tflops = 2 * ops / (ms["bh_traversal"] * 1e-3) / 1e12
    hbm = _measured_hbm_gbs()
    local_gbs = LOCAL_BYTES_PER_VERTEX * n / (ms["local"] * 1e-3) / 1e9
    return {
        "phases_ms_one_eager_step": ms,
        "bh": {"bound": "fp64", "achieved": bh_tflops, "peak": peaks["fp64"] / 1e12, "unit": "TFLOP/s",
               "frac": bh_tflops * 1e12 / peaks["fp64"],
               "interactions_per_vertex": (prof["leaf_pairs"] - n + prof["monopoles"]) / n,
               "node_tests_per_vertex": prof["node_tests"] / n,
               "lane_efficiency": (prof["leaf_pairs"] + prof["node_tests"]) / max(1, prof["lane_slots"]),
               "ops_def": "fp64 lane-ops x 2 / bh_kernel time; 15/leaf pair, 16/monopole, 9/opening test",
               "peak_source": "measured DFMA microbenchmark (mdc_peak_dfma), this run"},
        "local": {"bound": "hbm", "achieved": local_gbs, "peak": hbm, "unit": "GB/s", "frac": local_gbs / hbm,
                  "bytes_per_vertex": LOCAL_BYTES_PER_VERTEX,
                  "note": "algorithmic bytes (SURVEY.md §8d); working set L2-resident at this N",
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
    }


def _kernel_traffic(cfg, W, H, d, use_tc):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture, when this run is the captured workload (else None)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "r02_mls_tc_kernel_traffic.json")))
    except (OSError, ValueError):
        return None
    if use_tc and t.get("frame") == [W, H] and t.get("n") == cfg["n"] and t.get("d") == d:
        return t["traffic_bytes"]
    return None


def _measured_hbm_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback (6.65 TB/s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layout-iters", type=int, default=None)
    ap.add_argument("--no-layout", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--frame", default=None, help="override the raster, WxH (profiling only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tc", action="store_true", help="force the SIMT MLS kernel (A/B)")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 (reference precision) line")
    ap.add_argument("--dist-backend", default="nccl",
                    help="torch.distributed backend (gloo: host-mediated collectives, lets several ranks "
                         "share one GPU for a functional check of the N>1 path; never a bench number)")
    ap.add_argument("--layout-partition", action="store_true",
                    help="vertex-partition the layout over the ranks (default for config 4)")
    ap.add_argument("--layout-exchange", default="allgather", choices=["allgather", "p2p", "allreduce"],
                    help="partitioned layout: step kernel stores into every rank's buffer over NVLink "
                         "(p2p, cudaIpc) or a SUM all-reduce per iteration")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = dict(CONFIGS[args.config], id=args.config)
    if args.layout_iters is not None:
        cfg["iters"] = args.layout_iters
    if args.frame:
        cfg["W"], cfg["H"] = (int(v) for v in args.frame.lower().split("x"))

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist

    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    from paper_1408_0677_b200 import _lib
    from paper_1408_0677_b200 import field as F
    from paper_1408_0677_b200 import layout as L

    lib = _lib.require_cuda()
    dev = torch.device("cuda", local)

    ds, mesh, raw = build_scene(cfg)
    params = L.LayoutParams.defaults_for(mesh, iterations=cfg["iters"])

    # ---- layout: `iters` steps, device-resident, CUDA graph per step -------
    layout_res = None
    positions = mesh.original_pos
    partition = world > 1 and (args.layout_partition or args.config == 4)
    if not args.no_layout:
        temps = L.temperature_schedule(params.initial_temp, params.decay_lambda, cfg["iters"])
        p2p = partition and args.layout_exchange == "p2p"
        ag = partition and args.layout_exchange == "allgather"
        if p2p:  # the step kernel stores its slice into every rank's buffer
            run = L.P2PLayout(mesh, params, temps)
            eng = run.eng
        elif ag:  # packed owned slices, one NCCL all-gather per iteration
            gat = L.GatherLayout(mesh, params)
            eng = gat.eng
        else:
            eng = L.LayoutEngine(mesh, params, part=(rank, world) if partition else (0, 1))

        def reset():
            if p2p:
                run.reset(mesh.original_pos)
            else:
                eng.set_positions(mesh.original_pos)

        def layout_pass(k):
            if p2p:
                for _ in range(k):
                    run.step()
            elif ag:
                for it in range(k):
                    gat.step(temps[it:it + 1])
            elif partition:  # one SUM all-reduce of positions per iteration
                for it in range(k):
                    eng.run(temps[it:it + 1])
                    dist.all_reduce(eng.pos, op=dist.ReduceOp.SUM)
            else:
                eng.run(temps[:k])

        reset()
        # warm-up: one full pass captures every graph the timed pass replays
        # (single-step and 32-step graphs)
        layout_pass(cfg["iters"])
        reset()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        layout_pass(cfg["iters"])
        e1.record()
        e1.synchronize()
        lay_ms = e0.elapsed_time(e1)
        positions = (run.positions() if p2p else eng.pos).cpu().numpy()
        flips = L.count_orientation_flips(mesh, positions)
        t = torch.tensor([lay_ms], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # the whole mesh advances `iters` steps; replicas repeat the same work, so
        # they are not counted as extra throughput
        units = cfg["n"] * cfg["iters"]
        layout_res = {"metric": "vertex-iters/s", "unit": "vertex-iters/s",
                      "value": units / (t.item() * 1e-3),
                      "ms_total": t.item(), "iterations": cfg["iters"], "points": cfg["n"],
                      "orientation_flips": flips,
                      "scaling": ("strong (vertex-partitioned, step kernel stores into peer buffers over "
                                  "NVLink, host barrier per iteration)" if p2p else
                                  "strong (vertex-partitioned, one all-gather of the packed owned slices per "
                                  "iteration)" if ag else
                                  "strong (vertex-partitioned, SUM all-reduce per iteration)") if partition
                      else "replicas only (each rank runs the whole layout; value is one replica's)"}
        if p2p:
            run.close()
        if rank == 0:
            # rooflines of one whole-mesh step (a partitioned plan covers a slice)
            peng = L.LayoutEngine(mesh, params) if partition else eng
            if partition:
                peng.set_positions(positions)
            layout_res["roofline"] = layout_roofline(peng, params, lib, torch)

    # ---- MLS frame: d dims, row band per rank ---------------------------
    from paper_1408_0677_b200.field import MlsProblem

    W, H, d = cfg["W"], cfg["H"], cfg["d"]
    spacing = np.array([_auto_spacing(raw[:, k]) for k in range(d)])
    prob = MlsProblem(positions, raw, "affine", W, H, dtype="f32", tensor_cores=not args.no_tc)
    from paper_1408_0677_b200.shard import broadcast_controls, row_band

    r0, r1 = row_band(rank, world, H)
    rows = r1 - r0
    out = torch.empty((d, rows, W), dtype=torch.float32, device=dev)
    bands = torch.empty((d, rows, W), dtype=torch.int32, device=dev)
    # north_star (3): band shading fused into the MLS epilogue (RGBA8 per pixel-channel)
    from paper_1408_0677_b200.render import DEFAULT_COLORMAP

    rgba = torch.empty((d, rows, W), dtype=torch.int32, device=dev)
    pal_t = torch.as_tensor(F.palette_rgba8(DEFAULT_COLORMAP).view(np.int32)).to(dev)
    sp_t = torch.as_tensor(spacing).to(dev)
    nonfinite = torch.zeros((), dtype=torch.int32, device=dev)
    a = prob.args(out, (rows * W, W, 1), r0, r1, bands, (rows * W, W), sp_t, nonfinite, rgba=rgba, palette=pal_t)
    snap_ws = F._snap_workspace(int(lib.mdc_snap_workspace_bytes(W, rows)), dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    ctrl = [prob.pc_t, prob.q_t, prob.pm_t, prob.qm_t, prob.pos_t, prob.tvals_t]
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    kev = []

    def frame(timed):
        broadcast_controls(ctrl, src=0)  # point data once per frame (NCCL / NVLink)
        flush.fill_(1)
        nonfinite.zero_()
        if timed:
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0.record(stream)
        _lib.check(lib.mdc_mls_field(ctypes.byref(a), sptr), "mdc_mls_field")
        if timed:
            k1.record(stream)
            kev.append((k0, k1))
        _lib.check(lib.mdc_mls_snap(ctypes.byref(a), _lib.ptr(prob.pos_t), _lib.ptr(prob.tvals_t),
                                    ctypes.c_double(prob.eps), _lib.ptr(snap_ws), sptr), "mdc_mls_snap")

    for _ in range(args.warmup):
        frame(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            frame(True)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_total = t0.elapsed_time(t1)
    kernel_ms = statistics.mean(k0.elapsed_time(k1) for k0, k1 in kev)
    tt = torch.tensor([ms_total, kernel_ms], device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_total, kernel_ms = tt.tolist()
    ms_step = ms_total / args.steps
    value = W * H * d / (ms_step * 1e-3) / 1e6
    if int(nonfinite.item()) != 0:
        raise RuntimeError("non-finite field values")

    # ---- e2e through the public API (host buffers in, field out) -----------
    e2e = None if args.no_e2e else run_e2e(args, positions, raw, spacing, W, H, d, r0, r1, dev, world)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel --------------------------------
    peaks = measure_peaks(lib, torch)
    pairs = rows * W * cfg["n"]
    alg_flops = pairs * (19 + 6 * d)  # SURVEY.md §8d per-pair figure (one-pass formulation)
    use_tc = (not args.no_tc) and d >= 8
    if use_tc:
        nc = 16 if d <= 16 else (32 if d <= 32 else (64 if d <= 64 else 128))  # mls_tc.cu pick_nc
        chunks = -(-d // nc)
        # SIMT FP32 lane-ops per pair (FFMA2/FADD2/FMUL2 count 2): pass-1 moments 13
        # (alpha = 3/2: sum 1/r replaces sum w dy^2), pass-2 G evaluation + tf32
        # split 10 per channel chunk (ncu SASS count: profiles/r02_mls_tc_kernel_fp32_lane_ops.txt)
        fma_instr = pairs * (13 + 10 * chunks)
        mixed = nc > 32  # wide chunks: tf32 main + 2 bf16 corrections = 2 tf32-equivalent passes
        tc_flops = pairs * chunks * (2 if mixed else 3) * 2 * nc
        kname = (f"mls_tc_kernel<alpha=1.5, N={nc}> (tcgen05 pass 2: "
                 + ("kind::tf32 + kind::f16 bf16 corrections)" if mixed else "kind::tf32 3xTF32)"))
    else:
        dc = 1
        while dc < d and dc < 8:
            dc *= 2
        chunks = -(-d // dc)
        fma_instr = pairs * (14 + 9 * chunks + d)
        tc_flops = 0
        kname = f"mls_kernel<float, AFFINE, alpha=1.5, DC={dc}, R=2> (SIMT)"
    sec = kernel_ms * 1e-3
    achieved = 2 * fma_instr / sec / 1e12          # FP32-pipe FLOP-equivalents (FMA-pipe op = 2)
    peak = peaks["fp32"] / 1e12
    tf32_peak = 0.5 * _measured_bf16_tflops()       # dense tf32 = 1/2 bf16 (measured bf16, MEASURED_PEAKS.json)
    traffic, alg_bytes = _kernel_traffic(cfg, W, H, d, use_tc), pairs // cfg["n"] * d * 12 + cfg["n"] * (16 + 4 * d)
    roofline = {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_def": "dram__bytes_read.sum + dram__bytes_write.sum of one launch from the committed "
                               "ncu --set full capture of this workload (profiles/r02_mls_tc_kernel_traffic.json)",
                "algorithmic_bytes": alg_bytes,
                "algorithmic_bytes_def": "fp32 field + int32 bands + RGBA8 band shading per pixel-channel, + "
                                         "controls (16 B) and fp32 targets per control",
                "kernel": kname, "kernel_ms": kernel_ms,
                "achieved_def": "FP32-pipe lane-ops executed x 2 (one FMA-pipe lane-op = one FFMA = 2 FLOP) / kernel time",
                "peak_source": "measured FFMA microbenchmark (mdc_peak_ffma), this run",
                "algorithmic_tflops": alg_flops / sec / 1e12,
                "algorithmic_def": "SURVEY.md §8d 19+6d FLOP per (pixel, control) pair",
                "tensor_tflops": tc_flops / sec / 1e12 if tc_flops else 0.0,
                "tensor_peak_tflops": tf32_peak, "tensor_frac": (tc_flops / sec / 1e12) / tf32_peak if tc_flops else 0.0,
                "fp64_peak_tflops": peaks["fp64"] / 1e12,
                "kernel_share_of_step": kernel_ms / ms_step}

    fp64 = None if args.no_fp64 else run_fp64(positions, raw, cfg, W, H, d, dev, lib, peaks)

    cpu = None
    if not args.no_cpu and world == 1:  # the CPU baseline is quoted at N=1 only
        cpu = cpu_mls_sample(positions, raw, cfg, target_s=args.cpu_seconds)
        cpu.pop("seconds", None)
        if layout_res is not None:
            states, fixture = laid_out_positions(cfg, mesh)
            layout_res["cpu_baseline"] = cpu_layout_sample(mesh, params, states, steps=2)
            layout_res["positions_equal_cpu_arm_fixture"] = bool(np.array_equal(fixture, positions))

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, world),
        "gpu_launches": (6 if use_tc else 5) * args.steps,
        "clocks": clk.summary(),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "fp64": fp64,
        "layout": layout_res,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_fp64(positions, raw, cfg, W, H, d, dev, lib, peaks, band_div=8):
    """The reference's own precision: the same workload through the fp64
    parity kernel (mls_kernel<double>, reference arithmetic _kernels.py:70-124,
    1e-10 contract), on a band of H/band_div rows through the frame centre
    (per-pixel cost is uniform; a full 4K frame takes seconds in fp64),
    CUDA-event timed, L2 flushed first.  Roofline: executed fp64 lane-ops per
    (pixel, control) pair from the committed ncu capture
    (profiles/r02_mls_fp64_ops.json) x 2 / kernel time vs the live DFMA peak."""
    import torch

    from paper_1408_0677_b200 import _lib
    from paper_1408_0677_b200.field import MlsProblem

    prob = MlsProblem(positions, raw, "affine", W, H, dtype="f64")
    rows = max(1, H // band_div)
    r0 = (H - rows) // 2
    out = torch.empty((d, rows, W), dtype=torch.float64, device=dev)
    warm = prob.args(out, (rows * W, W, 1), r0, r0 + min(rows, 8))
    a = prob.args(out, (rows * W, W, 1), r0, r0 + rows)
    stream = torch.cuda.current_stream()
    _lib.check(lib.mdc_mls_field(ctypes.byref(warm), stream.cuda_stream), "mdc_mls_field")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    flush.fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _lib.check(lib.mdc_mls_field(ctypes.byref(a), stream.cuda_stream), "mdc_mls_field")
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    pairs = rows * W * cfg["n"]
    res = {"value": rows * W * d / (ms * 1e-3) / 1e6, "unit": UNIT, "dtype": "f64", "kernel_ms": ms,
           "sample": f"{rows} rows x {W} px through the frame centre (1/{band_div} of the frame), all {d} dims, "
                     f"N={cfg['n']} controls",
           "kernel": "mls_kernel<double, AFFINE, alpha=1.5> (SIMT, fp64 parity mode)"}
    try:
        ops = json.load(open(os.path.join(ROOT, "profiles", "r02_mls_fp64_ops.json")))
        if ops.get("d") == d:
            achieved = 2 * pairs * ops["fp64_lane_ops_per_pair"] / (ms * 1e-3)
            res["roofline"] = {"bound": "fp64", "achieved": achieved / 1e12, "peak": peaks["fp64"] / 1e12,
                               "unit": "TFLOP/s", "frac": achieved / peaks["fp64"],
                               "fp64_lane_ops_per_pair": ops["fp64_lane_ops_per_pair"],
                               "achieved_def": "executed fp64 lane-ops (ncu SASS count, DFMA/DADD/DMUL) x 2 / "
                                               "kernel time", "peak_source": "measured DFMA microbenchmark"}
    except (OSError, ValueError, KeyError):
        pass
    return res


def run_e2e(args, positions, raw, spacing, W, H, d, r0, r1, dev, world):
    """The same frame through the public API: pinned host inputs -> H2D ->
    kernels -> D2H of the fp32 field, every step (field.compute_fields_to_host:
    per-band D2H overlapped with the next band's kernels)."""
    import torch
    import torch.distributed as dist

    from paper_1408_0677_b200 import field as F

    rows = r1 - r0
    pin_pos = torch.from_numpy(np.ascontiguousarray(positions)).pin_memory()
    pin_raw = torch.from_numpy(np.ascontiguousarray(raw)).pin_memory()
    host_out = torch.empty((d, rows, W), dtype=torch.float32).pin_memory()
    host_rgba = torch.empty((d, rows, W, 4), dtype=torch.uint8).pin_memory()
    from paper_1408_0677_b200.render import DEFAULT_COLORMAP

    mp = F.MlsParams("affine")
    ne = max(1, min(args.steps, 3))
    h2d = [0]

    def e2e_step():
        # public API with host buffers in and out: the frame's row bands are
        # copied back while the next band computes (compute_fields_to_host)
        h2d[0] = F.compute_fields_to_host(pin_pos, pin_raw, mp, W, H, host_out,
                                          row_range=(r0, r1), dtype="f32", band_spacing=spacing,
                                          rgba_out=host_rgba, colormap=DEFAULT_COLORMAP)

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    c0 = time.perf_counter()
    for _ in range(ne):
        e2e_step()
    c1 = time.perf_counter()
    e_ms = torch.tensor([(c1 - c0) * 1e3 / ne], device=dev)
    if world > 1:
        dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
    return {"value": W * H * d / (e_ms.item() * 1e-3) / 1e6, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d[0]), "d2h_bytes_per_step": int(host_out.numel() * 4 + host_rgba.numel()),
            "ms_per_step": e_ms.item(), "timing": "wall clock, synchronized, max over ranks"}


def _measured_bf16_tflops():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 1590.0  # B200_PROFILING.md fallback


def _auto_spacing(values):
    from paper_1408_0677_b200.render import auto_spacing
    return auto_spacing(values)


if __name__ == "__main__":
    main()
