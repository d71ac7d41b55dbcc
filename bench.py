#!/usr/bin/env python
"""bench.py — SteepGS hot path on B200 (BASELINE.json metric: "fwd+bwd+splitting-matrix ms/view
@1M Gaussians; densify Gaussians/s; x1-8 GPU").

One step = the whole hot path over one batch of V views per GPU:
restore the densified planes from the pristine copy (checkpoint restore, cudaMemcpy2D) ->
project -> bin/sort -> render fwd -> l1 gradient -> render bwd (moments) -> per-Gaussian bwd + S
-> [NCCL allreduce of grads + S across ranks, N > 1] -> SDC densify.
Workload: BASELINE configs[1] (C2): 1.0M Gaussians, 980x545, synthetic surface-like scene (seeded,
SURVEY §8(d1)); views are sharded over ranks (rank r takes ring views r::N, weak scaling).

value = ms per view for the whole job = max-over-ranks step time / (V * N).
Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (bounded sample).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "fwd+bwd+splitting-matrix ms/view @1M Gaussians; densify Gaussians/s; x1-8 GPU"
UNIT = "ms/view"
FP32_LANES_PER_SM = 128
N_SM = 148
# algorithmic work per unit
BWD_LANE_OPS_PER_PAIR = 45.0   # contributing pair in the backward replay
FWD_LANE_OPS_PER_PAIR = 20.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm_gbs=float(d["hbm_gbs"]), sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)), src="measured")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9:
                continue
            try:
                sm.append(float(c[1]))
                mx.append(float(c[2]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if c[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return dict(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=max(mx) if mx else None,
                    reasons=sorted(reasons), samples=len(sm))


def clock_probe(stream, cycles=20_000_000):
    """SM clock (MHz) right after the timed region: torch.cuda._sleep spins one thread for `cycles`
    SM cycles (clock64); CUDA events around it give the wall time on the device."""
    import torch
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(cycles // 10)
    a.record(stream)
    torch.cuda._sleep(cycles)
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b)
    return round(cycles / (ms * 1e3), 1) if ms > 0 else None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------------------------------------
# CPU oracle (baseline + reference arm): bounded sample of the same workload
# ------------------------------------------------------------------------------------------------
def oracle_view(cfg, params, cam, dl_full):
    """One WHOLE view of the hot path on the CPU oracle (O1-O4 per view): fp32
    decision chain + fp64 projection of all n Gaussians, then fwd + bwd + S (per pair, fp64) over
    every pixel.  Returns (ms, sample description)."""
    import oracle
    t0 = time.perf_counter()
    dec = oracle.decide(params, cam)
    oracle.render(params, cam, dl_dimage=dl_full, decision=dec)
    ms = 1e3 * (time.perf_counter() - t0)
    desc = (f"whole views of {cfg.name} ({cfg.n} Gaussians, {cfg.width}x{cfg.height}): fp32 decision chain over "
            f"all Gaussians + fp64 fwd+bwd+S over every pixel (oracle/oracle.c, OpenMP)")
    return ms, desc


def oracle_window_estimate(cfg, params, cam, dl_full):
    """Labelled extra (round 1's estimate): a centred 96x64 window scaled by pixel count.  It
    over-estimates a whole view (the decision chain and candidate projection do not scale with
    pixels), so it is reported beside the whole-view timing, never as the baseline."""
    import oracle
    w, h = min(96, cfg.width), min(64, cfg.height)
    x0, y0 = (cfg.width - w) // 2, (cfg.height - h) // 2
    t0 = time.perf_counter()
    dec = oracle.decide(params, cam)
    t1 = time.perf_counter()
    oracle.render(params, cam, window=(x0, y0, w, h), dl_dimage=dl_full[:, y0:y0 + h, x0:x0 + w], decision=dec)
    t2 = time.perf_counter()
    frac = (w * h) / float(cfg.width * cfg.height)
    return 1e3 * ((t1 - t0) + (t2 - t1) / frac), f"{w}x{h} window scaled by 1/{1 / frac:.0f}"


def cpu_baseline(cfg, params, cams, reps=3):
    """Median of `reps` whole ring views on the host cores (median of 3 at C2)."""
    import oracle
    oracle.build()
    dl = synth.dl_dimage(1, cfg.width, cfg.height, 7)[0]
    ts = []
    desc = ""
    for k in range(reps):
        ms, desc = oracle_view(cfg, params, cams[k % len(cams)], dl)
        ts.append(ms)
    est, edesc = oracle_window_estimate(cfg, params, cams[0], dl)
    return dict(value=round(statistics.median(ts), 1), unit=UNIT, cores=oracle.num_threads(), kind="oracle",
                sample=f"median of {reps} {desc}", per_view_ms=[round(t, 1) for t in ts],
                window_estimate=dict(value=round(est, 1), unit=UNIT, sample=edesc, note="extra, not the baseline"))


def run_reference(args):
    """The reference arm (tier framing: the oracle as it stands on the host cores).  Each step is one
    whole view of the same workload (ring views in turn); the line's value is the mean ms/view."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    cfg = synth.CONFIGS[args.config]
    params = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=max(args.steps, 1))
    dl = synth.dl_dimage(1, cfg.width, cfg.height, 7)[0]
    t_run = time.perf_counter()
    for k in range(args.warmup):
        oracle_view(cfg, params, cams[k % len(cams)], dl)
    ts = []
    desc = ""
    for k in range(args.steps):
        ms, desc = oracle_view(cfg, params, cams[k % len(cams)], dl)
        ts.append(ms)
    wall = time.perf_counter() - t_run
    v = float(np.mean(ts)) if ts else 0.0
    cores = oracle.num_threads()
    out = dict(metric=METRIC, value=round(v, 2), unit=UNIT, n_gpus=args.gpus, steps=args.steps, warmup=args.warmup,
               ms_per_step=round(v, 2), higher_is_better=False, scaling="weak", vs_baseline=None, dtype="f64",
               data="synthetic", impl="reference",
               config=dict(workload=f"{cfg.name}: {cfg.cite}", n=cfg.n, width=cfg.width, height=cfg.height,
                           views_per_step=1),
               cpu_baseline=dict(value=round(v, 2), unit=UNIT, cores=cores, kind="oracle",
                                 sample=f"each step one of {desc}"),
               e2e=dict(value=round(v, 2), unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0),
               consistency=dict(timed_s=round(sum(ts) / 1e3, 2), run_wall_s=round(wall, 2),
                                fits_in_run=bool(sum(ts) / 1e3 <= wall)))
    print(json.dumps(out), flush=True)
    return 0


def to_u8(a):
    """Synthetic float targets in [0, 1] as 8-bit images (round to nearest)."""
    return np.ascontiguousarray(np.clip(np.rint(a * 255.0), 0, 255).astype(np.uint8))


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` (N > 1) without a torchrun environment: launch N ranks on this node ourselves
    (the driver's own command is torchrun; this makes a plain `python bench.py --gpus N` do the same
    instead of silently timing one GPU)."""
    import socket
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:   # noqa: BLE001
        have = 0
    if args.impl != "reference" and have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but this node has {have} CUDA device(s)", file=sys.stderr)
        return 3
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
def run_v1(args, cfg, p_np, pristine, dev, stream, views=16):
    """One view per step over `views` ring views: ms/view of the whole step
    (a1..a8) and of fwd+bwd+S alone (project .. gauss_bwd), CUDA events per stage, per-stage graphs."""
    import torch

    from paper_2505_05587_b200 import _lib
    from paper_2505_05587_b200.pipeline import Rasterizer
    n = cfg.n
    cap = pristine.shape[1]
    params = pristine.clone()
    grad_S = torch.zeros(20, cap, dtype=torch.float32, device=dev)
    cams = synth.cameras_for(cfg, views=views)
    tg_np = np.ascontiguousarray(synth.targets_for(cfg, views=views))
    tg = torch.from_numpy(to_u8(tg_np) if args.targets == "u8" else tg_np).to(dev)
    rz = Rasterizer(cap, 1, cfg.width, cfg.height, max_instances=int(3.0 * n), device=dev)

    def stages(v):
        def restore():
            _lib.copy_planes(params, pristine, n, 0, 3)
            _lib.copy_planes(params, pristine, n, 10, 1)
        return [("restore", restore), ("project", lambda: rz.project(params, n, [cams[v]])),
                ("bin_sort", rz.bin_sort), ("render_fwd", lambda: rz.render_fwd_l1(tg[v:v + 1])),
                ("render_bwd", rz.render_bwd_moments), ("gauss_bwd_S", lambda: rz.gauss_bwd(params, grad_S, accumulate=0)),
                ("densify", lambda: rz.densify(params, grad_S, n, cap, denom=1.0, want_lambda=False))]
    for v in range(views):                       # warm-up: every view once (projection uploads its camera)
        for _, f in stages(v):
            f()
    torch.cuda.synchronize()
    graphs, whole = {}, {}
    if not args.no_graph:
        for v in range(views):
            gs = []
            for nm, f in stages(v):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    f()
                gs.append(g)
            graphs[v] = gs
            g = torch.cuda.CUDAGraph()                  # the whole step as one graph (the value)
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                for _, f in stages(v):
                    f()
            whole[v] = g
    torch.cuda.synchronize()
    nst = len(stages(0))
    # the value: each view's whole step timed alone (one graph, events around it)
    wev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(views)]
    for v in range(views):
        wev[v][0].record(stream)
        if whole:
            whole[v].replay()
        else:
            for _, f in stages(v):
                f()
        wev[v][1].record(stream)
    torch.cuda.synchronize()
    # the breakdown: per-stage graphs with events between them
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nst + 1)] for _ in range(views)]
    for v in range(views):
        evs[v][0].record(stream)
        for k, (nm, f) in enumerate(stages(v)):
            if graphs:
                graphs[v][k].replay()
            else:
                f()
            evs[v][k + 1].record(stream)
    torch.cuda.synchronize()
    if rz.binning_arrays()["overflow"] != 0:
        raise RuntimeError("v1: tile-instance buffer overflow")
    names = [nm for nm, _ in stages(0)]
    per = {nm: float(np.median([evs[v][k].elapsed_time(evs[v][k + 1]) for v in range(views)]))
           for k, nm in enumerate(names)}
    tot = [wev[v][0].elapsed_time(wev[v][1]) for v in range(views)]
    tot_staged = [evs[v][0].elapsed_time(evs[v][nst]) for v in range(views)]
    fbs = [evs[v][1].elapsed_time(evs[v][names.index("gauss_bwd_S") + 1]) for v in range(views)]
    return dict(value=round(float(np.median(tot)), 5), unit=UNIT, views=views, views_per_step=1,
                value_with_stage_events=round(float(np.median(tot_staged)), 5),
                fwd_bwd_S_ms_per_view=round(float(np.median(fbs)), 5),
                stages_ms={k: round(v, 4) for k, v in per.items()},
                note="SURVEY 8(d1) headline definition: C2, one view per step (restore + a1..a8, densify "
                     "denom 1), median over 16 ring views, each step one graph replay; the stage breakdown and "
                     "fwd_bwd_S (project .. gauss_bwd, 8(d2)) from a second pass with per-stage graphs and events")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--views", type=int, default=8, help="views per GPU per step")
    ap.add_argument("--sh-degree", type=int, default=None, help="f3: view-dependent SH colour of this degree")
    ap.add_argument("--ssim", type=float, default=None, help="f3: loss (1 - l) l1 + l (1 - SSIM) with l = this")
    ap.add_argument("--budget-frac", type=float, default=None,
                    help="densify with the increment budget K = frac * n (App. A.2; SURVEY C4's ~10% split)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel eagerly (no per-stage CUDA graphs)")
    ap.add_argument("--h2d-at", default="after_sort", choices=["start", "after_sort"],
                    help="e2e: start step k+1's target copy with step k, or after step k's bin_sort (the copy's "
                         "DMA writes then overlap the ALU-bound render kernels, not the L2-resident sort)")
    ap.add_argument("--targets", default="u8", choices=["u8", "f32"],
                    help="target image format uploaded per step (u8: 8-bit, decoded * (1/255) on the device)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-v1", action="store_true", help="skip the 1-view-per-step line (SURVEY §8(d1))")
    ap.add_argument("--collective", default="nccl", choices=["nccl", "fused"],
                    help="N > 1: NCCL allreduce of grads + S, or k_gauss_bwd scattering to the column owners over "
                         "peer memory + owner reduce/broadcast (torch symmetric memory)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_under_torchrun(args)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2505_05587_b200 import _lib
    from paper_2505_05587_b200.pipeline import Rasterizer
    from paper_2505_05587_b200.parallel import allreduce_accumulators

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg = synth.CONFIGS[args.config]
    V = args.views
    n = cfg.n
    cap = 2 * n
    p_np = synth.scene_for(cfg)
    all_cams = synth.cameras_for(cfg, views=V * ws)
    cams = all_cams[rank::ws]                                 # view sharding
    tg_all = synth.targets_for(cfg, views=V * ws)
    tg_np = np.ascontiguousarray(tg_all[rank::ws])
    u8 = args.targets == "u8" and args.ssim is None        # the SSIM loss kernels take float targets
    if u8:   # the targets as 8-bit images (a photograph's format), decoded * (1/255) by the fused l1 epilogue
        tg_np = to_u8(tg_np)

    pristine = torch.zeros(14, cap, dtype=torch.float32, device=dev)
    pristine[:, :n] = torch.from_numpy(p_np).to(dev)
    params = pristine.clone()
    grad_S = torch.zeros(20, cap, dtype=torch.float32, device=dev)
    reducer = None
    if args.collective == "fused" and ws > 1:
        if args.sh_degree is not None:
            raise SystemExit("bench.py: --collective fused has no SH colour path (use nccl)")
        from paper_2505_05587_b200.parallel import FusedGradReduce
        reducer = FusedGradReduce(cap, device=dev)   # symmetric-memory grad_S + partial buffers
        grad_S = reducer.grad_S

    def collective():
        if reducer is not None:
            reducer.exchange(n, accumulate=0)         # owners reduce + broadcast over NVLink (P2P)
        else:
            allreduce_accumulators(grad_S, n=n)       # NCCL, [k, :n] rows in one group
    targets = torch.from_numpy(tg_np).to(dev)
    rz = Rasterizer(cap, V, cfg.width, cfg.height, max_instances=int(3.0 * V * n), device=dev)
    shd = args.sh_degree
    sh_rest = grad_sh = loss_ws = None
    if shd is not None:                                       # f3 workload: DC = planes 11-13 + rest
        nrest = 3 * ((shd + 1) ** 2 - 1)
        sh_rest = torch.zeros(max(nrest, 1), cap, dtype=torch.float32, device=dev)[:nrest]
        sh_rest[:, :n] = torch.from_numpy(synth.sh_coefficients(n, shd, 4000 + int(cfg.name[1:]))).to(dev)
        grad_sh = torch.zeros_like(sh_rest)
    if args.ssim is not None:
        loss_ws = torch.empty(_lib.loss_workspace_size(V, cfg.height, cfg.width), dtype=torch.uint8, device=dev)
    pair_counts = torch.zeros(2, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    stage_names = ["restore", "project", "bin_sort", "render_fwd", "l1_grad", "render_bwd", "gauss_bwd_S",
                   "allreduce", "densify"]

    def stage_fns(tgt):
        """The step as (stage, callable or None) in stage_names order; None = nothing in this stage."""
        def restore():
            _lib.copy_planes(params, pristine, n, 0, 3)      # undo last step's densify (positions,
            _lib.copy_planes(params, pristine, n, 10, 1)     # opacity) -- checkpoint restore, no kernel

        def bwd():
            if reducer is not None:                   # a6 with its output scattered to the column owners
                reducer.scatter(rz, params, n)
                return
            if shd is not None:
                rz.sh_bwd(params, grad_S, sh_rest, shd, grad_sh, 0)
            rz.gauss_bwd(params, grad_S, accumulate=0 | (4 if shd is not None else 0))
        fused = args.ssim is None
        return [
            ("restore", restore),
            ("project", lambda: rz.project(params, n, cams, sh_rest, shd)),
            ("bin_sort", rz.bin_sort),
            # a3 + a4 fused (l1 gradient in the forward's epilogue) unless the SSIM term is on
            ("render_fwd", (lambda: rz.render_fwd_l1(tgt)) if fused else rz.render_fwd),
            ("l1_grad", None if fused else (lambda: _lib.l1_ssim_grad(rz.image, tgt, args.ssim, 1.0, rz.dL, rz.loss,
                                                                      loss_ws))),
            ("render_bwd", rz.render_bwd_moments),
            ("gauss_bwd_S", bwd),
            ("allreduce", collective if ws > 1 else None),
            ("densify", lambda: rz.densify(params, grad_S, n, cap, denom=float(V * ws), want_lambda=False,
                                           budget=None if args.budget_frac is None else int(args.budget_frac * n))),
        ]

    # Per-stage CUDA graphs (captured after the warm-up; one set per target buffer): a replay
    # launches a stage's kernels and memsets back to back with no host launch overhead between them;
    # the stage boundaries stay eager so the per-stage CUDA events of the timed region bracket them.
    # The NCCL allreduce stays eager.  Kernels inside a graph are counted when it is captured.
    graphs = {}
    step_graphs = {}
    graph_launches = [0]
    launch_mode = ["eager" if args.no_graph else
                   "one CUDA graph per step (NCCL allreduce eager, between two graphs) for the timed steps; "
                   "per-stage CUDA graphs with CUDA events between them for the stage breakdown"]

    def capture(tgt):
        key = tgt.data_ptr()
        if key in graphs:
            return
        gs = {}
        for nm, fn in stage_fns(tgt):
            if fn is None or nm == "allreduce":
                continue
            g = torch.cuda.CUDAGraph()
            l0 = _lib.launch_count()
            try:
                with torch.cuda.graph(g, capture_error_mode="thread_local"):   # NCCL watchdog threads may query events
                    fn()
            except RuntimeError as exc:   # keep the stage eager rather than lose the run
                torch.cuda.synchronize()
                launch_mode[0] = f"per-stage CUDA graphs; {nm} eager (capture failed: {str(exc).splitlines()[0][:80]})"
                print(f"bench: graph capture of {nm} failed, stage runs eagerly: {exc}", file=sys.stderr)
                continue
            gs[nm] = (g, _lib.launch_count() - l0)
        graphs[key] = gs
        # the whole step as graph segments split after bin_sort (the e2e copy of the next step's targets
        # waits for an event recorded there) and at the (eager) NCCL allreduce
        segs, cur = [], []
        for nm, fn in stage_fns(tgt):
            if fn is None:
                continue
            if nm == "allreduce":
                segs.append(cur)
                segs.append("allreduce")
                cur = []
            else:
                cur.append(fn)
                if nm == "bin_sort":
                    segs.append(cur)
                    segs.append("sorted")
                    cur = []
        segs.append(cur)
        out = []
        for sg in segs:
            if sg in ("allreduce", "sorted"):
                out.append((sg, None, 0))
                continue
            if not sg:
                continue
            g = torch.cuda.CUDAGraph()
            l0 = _lib.launch_count()
            try:
                with torch.cuda.graph(g, capture_error_mode="thread_local"):
                    for fn in sg:
                        fn()
            except RuntimeError as exc:
                torch.cuda.synchronize()
                print(f"bench: step-graph capture failed, per-stage graphs used: {exc}", file=sys.stderr)
                return
            out.append(("graph", g, _lib.launch_count() - l0))
        step_graphs[key] = out

    def step_whole(tgt=None, sorted_ev=None):
        """One step through the step graphs (timed steps and e2e); falls back to step()."""
        tgt = targets if tgt is None else tgt
        sgs = step_graphs.get(tgt.data_ptr()) if not args.no_graph else None
        if not sgs:
            step(tgt=tgt, sorted_ev=sorted_ev)
            return
        for kind, g, nl in sgs:
            if kind == "allreduce":
                collective()
            elif kind == "sorted":
                if sorted_ev is not None:
                    sorted_ev.record(stream)
            else:
                g.replay()
                graph_launches[0] += nl

    def step(ev=None, tgt=None, sorted_ev=None):
        tgt = targets if tgt is None else tgt
        gs = graphs.get(tgt.data_ptr()) if not args.no_graph else None
        if ev is not None:
            ev[0].record(stream)
        for k, (nm, fn) in enumerate(stage_fns(tgt)):
            if gs is not None and nm in gs:
                g, nl = gs[nm]
                g.replay()
                graph_launches[0] += nl
            elif fn is not None:
                fn()
            if ev is not None and fn is not None:   # an empty stage records no event (each costs ~4 us)
                ev[k + 1].record(stream)
            if sorted_ev is not None and nm == "bin_sort":
                sorted_ev.record(stream)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3) if args.warmup >= 3 else args.warmup):
        step()
    barrier()
    if not args.no_graph:
        capture(targets)
        for _ in range(2):   # first replays upload the graphs: both launch modes warm before timing
            step()
            step_whole()
        barrier()
    pair_counts.zero_()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(10)] for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    graph_launches[0] = 0
    sampler = ClockSampler(local)
    time.sleep(0.3)
    barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        step_whole()
    t_end.record(stream)
    barrier()
    launches = _lib.launch_count() - launches0 + graph_launches[0]   # kernels of the timed steps
    # stage breakdown: the same steps again with per-stage graphs and CUDA events between them (each
    # event costs ~4 us of device time, so this pass is not the headline)
    t_st0 = torch.cuda.Event(enable_timing=True)
    t_st1 = torch.cuda.Event(enable_timing=True)
    t_st0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_st1.record(stream)
    barrier()
    clocks = sampler.stop()
    clocks["probe_mhz"] = clock_probe(stream)
    elapsed = t_start.elapsed_time(t_end)
    if ws > 1:
        tt = torch.tensor([elapsed], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    ms_step = elapsed / args.steps
    ms_step_staged = t_st0.elapsed_time(t_st1) / args.steps
    # stage i spans from the last event recorded before it to its own (empty stages: 0)
    recorded = [0] + [i + 1 for i, (_, fn) in enumerate(stage_fns(targets)) if fn is not None]
    stage_ms = {}
    for i, nm in enumerate(stage_names):
        if i + 1 not in recorded:
            stage_ms[nm] = 0.0
            continue
        prev = max(r for r in recorded if r <= i)
        stage_ms[nm] = float(np.mean([evs[k][prev].elapsed_time(evs[k][i + 1]) for k in range(args.steps)]))

    # every timed step's binning fitted its buffers (a step whose tile instances overflowed
    # max_instances would have rendered a truncated list): the overflow flag is sticky per bin_sort,
    # and the scene is the same each step, so the last step's flag decides
    if rz.binning_arrays()["overflow"] != 0:
        print("bench.py: tile-instance buffer overflow in the timed steps", file=sys.stderr)
        return 4

    # ---- counts for the roofline model: one counting forward after the timed region (the timed
    # forward runs the non-counting kernel instance), then device -> host ----
    _lib.copy_planes(params, pristine, n, 0, 3)
    _lib.copy_planes(params, pristine, n, 10, 1)
    rz.project(params, n, cams)
    rz.bin_sort()
    rz.render_fwd(pair_counts)
    b = rz.binning_arrays()
    n_vis, n_inst = b["n_visible"], b["n_instances"]
    comp_pairs, eval_pairs = (int(x) for x in pair_counts.cpu().tolist())
    n_split = int(rz.n_split.item())
    px = cfg.width * cfg.height
    tiles = ((cfg.width + 15) // 16) * ((cfg.height + 15) // 16)
    peaks = measured_peaks()
    hbm = peaks["hbm_gbs"]
    # the ALU peak at the SM clock the kernels ran at: the device-side probe right after the timed
    # region (nvidia-smi's 200 ms samples mostly miss a ~40 ms timed region and catch idle clocks)
    sm_mhz = clocks.get("probe_mhz") or clocks["sm_mhz"] or peaks["sm_max_mhz"]
    alu_peak = N_SM * FP32_LANES_PER_SM * sm_mhz * 1e6       # lane-ops/s at the measured clock
    # algorithmic (compulsory) bytes per launch of each stage
    byts = {
        "restore": 2 * 16 * n,
        "project": 56 * n + V * 16 * n + 64 * n_vis,
        "bin_sort": V * 16 * n + 8 * n_vis + 20 * n_inst + 8 * tiles * V,
        "render_fwd": 4 * n_inst + 64 * n_vis + 20 * px * V + 24 * px * V,   # + target read, dL write (fused a4)
        "l1_grad": 0,
        "render_bwd": 4 * n_inst + 64 * n_vis + 28 * px * V + 48 * n_vis,
        "gauss_bwd_S": 56 * n + 4 * V * n + 96 * n_vis + 80 * n,
        "densify": 24 * n + 8 * n + 24 * n + n_split * (56 + 56 + 80),
    }
    stages = {}
    for nm in stage_names:
        t = stage_ms[nm]
        e = dict(ms=round(t, 4))
        if nm in byts and t > 0:
            gbs = byts[nm] / (t * 1e-3) / 1e9
            e.update(alg_bytes=int(byts[nm]), gbs=round(gbs, 1), hbm_frac=round(gbs / hbm, 4))
        stages[nm] = e
    bwd_ops = BWD_LANE_OPS_PER_PAIR * comp_pairs
    stages["render_bwd"].update(alu_lane_ops=bwd_ops, alu_frac=round(bwd_ops / (stage_ms["render_bwd"] * 1e-3) / alu_peak, 4))
    stages["render_fwd"].update(alu_lane_ops=FWD_LANE_OPS_PER_PAIR * comp_pairs,
                                alu_frac=round(FWD_LANE_OPS_PER_PAIR * comp_pairs / (stage_ms["render_fwd"] * 1e-3) / alu_peak, 4))
    kernel_stages = [s for s in stage_names if s not in ("restore", "allreduce")]
    dom = max(kernel_stages, key=lambda s: stage_ms[s])
    if dom in ("render_bwd", "render_fwd"):
        ops = stages[dom]["alu_lane_ops"]
        ach = ops / (stage_ms[dom] * 1e-3) / 1e12
        roofline = dict(bound="alu", kernel=dom, achieved=round(ach, 3), peak=round(alu_peak / 1e12, 3),
                        unit="T lane-op/s", frac=round(ach * 1e12 / alu_peak, 4), traffic=None,
                        units_per_launch=dict(contributing_pairs=comp_pairs,
                                              lane_ops_per_pair=BWD_LANE_OPS_PER_PAIR if dom == "render_bwd" else FWD_LANE_OPS_PER_PAIR),
                        peak_basis=f"{N_SM} SMs x {FP32_LANES_PER_SM} FP32 lanes x median SM clock {sm_mhz:.0f} MHz")
    else:
        ach = byts[dom] / (stage_ms[dom] * 1e-3) / 1e9
        roofline = dict(bound="hbm", kernel=dom, achieved=round(ach, 1), peak=hbm, unit="GB/s",
                        frac=round(ach / hbm, 4), traffic=None, peak_basis=f"MEASURED_PEAKS.json ({peaks['src']})")
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture (profiles/)
    kname = {"render_bwd": "k_render_bwd2", "render_fwd": "k_render_fwd", "gauss_bwd_S": "k_gauss_bwd",
             "project": "k_project"}.get(dom)
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if kname and os.path.exists(tfile):
        with open(tfile) as f:
            tr = json.load(f).get(kname)
        if tr and int(tr.get("views", -1)) == V and args.config == "C2":
            roofline["traffic"] = tr["bytes_per_launch"]
            roofline["traffic_unit"] = "bytes per launch (dram read + write)"
            roofline["traffic_alg_bytes"] = int(byts[dom])
            roofline["traffic_source"] = tr["source"]
    path_bytes = sum(byts[s] for s in byts)
    path_ms = sum(stage_ms[s] for s in byts)
    value = ms_step / (V * ws)

    # ---- e2e: host buffers through the public API (H2D of the targets, D2H of loss + n_split) ----
    # Every step copies its V target images from pinned host memory and reads its loss and split
    # count back; the H2D copy of step k+1 runs on a copy stream under step k's kernels (double-
    # buffered targets), the D2H read ends each step with a host synchronisation.
    e2e = None
    if not args.no_e2e:
        tg_host = torch.from_numpy(tg_np).pin_memory()
        loss_host = [torch.zeros(V, dtype=torch.float32).pin_memory() for _ in range(2)]
        ns_host = [torch.zeros(1, dtype=torch.int64).pin_memory() for _ in range(2)]
        results = [torch.cuda.Event(), torch.cuda.Event()]
        seen = []
        tbuf = [targets, torch.empty_like(targets)]
        copy_stream = torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]

        sorted_evs = [torch.cuda.Event(), torch.cuda.Event()]

        def h2d(slot, after=None):
            with torch.cuda.stream(copy_stream):
                copy_stream.wait_event(consumed[slot])
                if after is not None:
                    copy_stream.wait_event(after)
                tbuf[slot].copy_(tg_host, non_blocking=True)
                copied[slot].record(copy_stream)

        def run_e2e(nsteps):
            # step k's loss and split count are read back into pinned slot k & 1; the host waits for
            # step k - 1's read-back (and consumes it) before issuing step k + 1, so every step's result
            # reaches the host inside the timed region while the device always has the next step queued
            h2d(0)
            for k in range(nsteps):
                slot = k & 1
                if k + 1 < nsteps and args.h2d_at == "start":
                    h2d(slot ^ 1)
                stream.wait_event(copied[slot])
                step_whole(tgt=tbuf[slot], sorted_ev=sorted_evs[slot])
                if k + 1 < nsteps and args.h2d_at == "after_sort":
                    h2d(slot ^ 1, after=sorted_evs[slot])
                consumed[slot].record(stream)
                loss_host[slot].copy_(rz.loss, non_blocking=True)
                ns_host[slot].copy_(rz.n_split, non_blocking=True)
                results[slot].record(stream)
                if k >= 1:
                    results[slot ^ 1].synchronize()
                    seen.append((float(loss_host[slot ^ 1].sum()), int(ns_host[slot ^ 1][0])))
            results[(nsteps - 1) & 1].synchronize()
            seen.append((float(loss_host[(nsteps - 1) & 1].sum()), int(ns_host[(nsteps - 1) & 1][0])))

        for ev in consumed:
            ev.record(stream)
        if not args.no_graph:
            capture(tbuf[1])
        run_e2e(2)
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        z = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run_e2e(args.steps)
        z.record(stream)
        barrier()
        et = a.elapsed_time(z)
        if ws > 1:
            tt = torch.tensor([et], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            et = float(tt.item())
        e2e = dict(value=et / args.steps / (V * ws), unit=UNIT,
                   h2d_bytes_per_step=int(tg_host.numel() * tg_host.element_size()),
                   d2h_bytes_per_step=int(loss_host[0].numel() * 4 + 8),
                   note="H2D of step k+1 overlapped with step k on a copy stream (issued "
                        + ("with step k" if args.h2d_at == "start" else "after step k's bin_sort")
                        + "); each step's loss and n_split read back to pinned host memory and consumed by the "
                          "host one step later")

    # ---- v1: SURVEY §8(d1)'s headline definition — C2 at ONE view per step, timed over 16 ring
    # views (the per-Gaussian stages, i.e. the parameter read in project, gauss_bwd's grad_S write and
    # densify, are charged to a single view); same stages, per-stage graphs, densify with denom 1 ----
    v1 = None
    if not args.no_v1 and ws == 1:
        v1 = run_v1(args, cfg, p_np, pristine, dev, stream)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, p_np, all_cams)

    if rank == 0:
        out = dict(
            metric=METRIC, value=round(value, 5), unit=UNIT, n_gpus=ws, steps=args.steps, warmup=args.warmup,
            ms_per_step=round(ms_step, 4), ms_per_step_with_stage_events=round(ms_step_staged, 4), higher_is_better=False, scaling="weak", vs_baseline=None, dtype="f32",
            data="synthetic",
            config=dict(workload=f"{cfg.name}: {cfg.cite}" + (f" + SH degree {shd}" if shd is not None else "")
                        + (f" + SSIM loss (lambda {args.ssim})" if args.ssim is not None else "")
                        + (f" + densify budget {args.budget_frac:g} n" if args.budget_frac is not None else ""),
                        n=n, width=cfg.width, height=cfg.height,
                        views_per_gpu_per_step=V, views_per_step=V * ws, capacity=cap,
                        parallelism=f"view-sharded dp{ws}" + ((" + NCCL allreduce(grads+S)" if reducer is None else
                                                                " + fused gauss_bwd reduce-scatter / owner broadcast "
                                                                "over NVLink (symmetric memory)") if ws > 1 else ""),
                        l2="no flush: per-step working set (params 56 MB + splats 48 B x V x n + sort/moment "
                           "buffers) exceeds the 126 MB L2",
                        scene="synthetic surface-like (SURVEY 8(d1)), procedural targets",
                        targets=("uint8 [V][3][H][W] (8-bit images), decoded as float(t) * (1/255) in the fused l1 "
                                 "epilogue" if u8 else "float32 [V][3][H][W]"),
                        launch=launch_mode[0]),
            roofline=roofline,
            path_hbm=dict(alg_bytes_per_step=int(path_bytes), ms=round(path_ms, 4),
                          frac=round(path_bytes / (path_ms * 1e-3) / 1e9 / hbm, 4), peak_gbs=hbm),
            stages=stages,
            counts=dict(n_visible=n_vis, n_instances=n_inst, contributing_pairs=comp_pairs, evaluated_pairs=eval_pairs,
                        n_split=n_split, split_frac=round(n_split / n, 4)),
            densify_gaussians_per_s=round(n / (stage_ms["densify"] * 1e-3), 1),
            gaussians_per_s=round(n * V * ws / (ms_step * 1e-3), 1),
            v1=v1, e2e=e2e, cpu_baseline=cpu, clocks=clocks, gpu_launches=int(launches),
            gpu_launches_per_step=round(launches / args.steps, 2),
        )
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
