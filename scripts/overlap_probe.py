"""Probe: one 8-view step on one stream vs. two 4-view halves on two streams (fork after the restore,
join before the second half's gauss_bwd).  Prints ms/step for each schedule.  GPU only."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2505_05587_b200 import _lib  # noqa: E402
from paper_2505_05587_b200.pipeline import Rasterizer  # noqa: E402


def main():
    cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    V, n = 8, cfg.n
    cap = 2 * n
    dev = torch.device("cuda", 0)
    p_np = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=V)
    tg = torch.from_numpy(np.ascontiguousarray(synth.targets_for(cfg, views=V))).to(dev)
    pristine = torch.zeros(14, cap, dtype=torch.float32, device=dev)
    pristine[:, :n] = torch.from_numpy(p_np).to(dev)
    params = pristine.clone()
    grad_S = torch.zeros(20, cap, dtype=torch.float32, device=dev)
    rz8 = Rasterizer(cap, V, cfg.width, cfg.height, max_instances=int(3.0 * V * n), device=dev)
    h = V // 2
    rzA = Rasterizer(cap, h, cfg.width, cfg.height, max_instances=int(3.0 * h * n), device=dev)
    rzB = Rasterizer(cap, h, cfg.width, cfg.height, max_instances=int(3.0 * h * n), device=dev)
    main_s = torch.cuda.current_stream()

    def restore():
        _lib.copy_planes(params, pristine, n, 0, 3)
        _lib.copy_planes(params, pristine, n, 10, 1)

    def half(rz, c, t):
        rz.project(params, n, c)
        rz.bin_sort()
        rz.render_fwd_l1(t)
        rz.render_bwd_moments()

    def serial8():
        restore()
        half(rz8, cams, tg)
        rz8.gauss_bwd(params, grad_S, accumulate=0)
        rz8.densify(params, grad_S, n, cap, denom=float(V), want_lambda=False)

    def serial44():
        restore()
        half(rzA, cams[:h], tg[:h])
        half(rzB, cams[h:], tg[h:])
        rzA.gauss_bwd(params, grad_S, accumulate=0)
        rzB.gauss_bwd(params, grad_S, accumulate=1)
        rzA.densify(params, grad_S, n, cap, denom=float(V), want_lambda=False)

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(10)]

    def serial8_marks():
        evs[0].record(main_s)
        restore()
        evs[1].record(main_s)
        rz8.project(params, n, cams)
        evs[2].record(main_s)
        rz8.bin_sort()
        evs[3].record(main_s)
        rz8.render_fwd_l1(tg)
        evs[4].record(main_s)
        evs[5].record(main_s)
        rz8.render_bwd_moments()
        evs[6].record(main_s)
        rz8.gauss_bwd(params, grad_S, accumulate=0)
        evs[7].record(main_s)
        evs[8].record(main_s)
        rz8.densify(params, grad_S, n, cap, denom=float(V), want_lambda=False)
        evs[9].record(main_s)

    for _ in range(3):
        serial8()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream(device=dev)
    cs.wait_stream(main_s)
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            serial8()
    torch.cuda.synchronize()

    def graph8():
        g.replay()

    xev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(10)]

    def serial8_xmarks():
        xev[0].record()
        restore()
        xev[1].record()
        rz8.project(params, n, cams)
        xev[2].record()
        rz8.bin_sort()
        xev[3].record()
        rz8.render_fwd_l1(tg)
        xev[4].record()
        xev[5].record()
        rz8.render_bwd_moments()
        xev[6].record()
        rz8.gauss_bwd(params, grad_S, accumulate=0)
        xev[7].record()
        xev[8].record()
        rz8.densify(params, grad_S, n, cap, denom=float(V), want_lambda=False)
        xev[9].record()

    gx = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gx):
        serial8_xmarks()
    torch.cuda.synchronize()

    def graph8_xmarks():
        gx.replay()

    stage_graphs = []
    for fn in (restore, lambda: rz8.project(params, n, cams), rz8.bin_sort, lambda: rz8.render_fwd_l1(tg),
               rz8.render_bwd_moments, lambda: rz8.gauss_bwd(params, grad_S, accumulate=0),
               lambda: rz8.densify(params, grad_S, n, cap, denom=float(V), want_lambda=False)):
        sg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(sg):
            fn()
        stage_graphs.append(sg)
    torch.cuda.synchronize()

    def stage_graphs_marks():
        evs[0].record(main_s)
        for k, sg in enumerate(stage_graphs):
            sg.replay()
            evs[k + 1].record(main_s)

    streams = {}

    def make_two(prioA, prioB):
        sA = torch.cuda.Stream(device=dev, priority=prioA)
        sB = torch.cuda.Stream(device=dev, priority=prioB)
        e0, eA, eB = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()

        def two():
            restore()
            e0.record(main_s)
            sA.wait_event(e0)
            sB.wait_event(e0)
            with torch.cuda.stream(sA):
                half(rzA, cams[:h], tg[:h])
                rzA.gauss_bwd(params, grad_S, accumulate=0)
                eA.record(sA)
            with torch.cuda.stream(sB):
                half(rzB, cams[h:], tg[h:])
                sB.wait_event(eA)
                rzB.gauss_bwd(params, grad_S, accumulate=1)
                eB.record(sB)
            main_s.wait_event(eB)
            rzA.densify(params, grad_S, n, cap, denom=float(V), want_lambda=False)
        streams[(prioA, prioB)] = (sA, sB)
        return two

    scheds = {"serial8": serial8, "serial8_marks": serial8_marks, "graph8": graph8, "graph8_xmarks": graph8_xmarks, "stage_graphs_marks": stage_graphs_marks, "serial4+4": serial44, "two_streams": make_two(0, 0),
              "two_streams_B_high": make_two(0, -1), "two_streams_A_high": make_two(-1, 0)}
    res = {}
    for rep in range(2):
        for nm, f in scheds.items():
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 20
            a.record(main_s)
            for _ in range(K):
                f()
            z.record(main_s)
            torch.cuda.synchronize()
            res.setdefault(nm, []).append(a.elapsed_time(z) / K)
            time.sleep(0.1)
    for nm, v in res.items():
        print(f"{nm:22s} ms/step {min(v):.4f}  ({', '.join(f'{x:.4f}' for x in v)})", flush=True)


if __name__ == "__main__":
    main()
