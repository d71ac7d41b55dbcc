"""Diagnostics for tests/test_gpu_fuzz.py::test_fuzz_full_path at given seeds (GPU): every gradient /
S element outside the strict §3.4 tolerance, with its oracle value, abs_ora, the plane maximum and the
ratio of its error to each tolerance term; and the ambiguous-pixel count per view.

usage: python scripts/fuzz_diag.py SEED [SEED ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from gpu_run import run_backward, run_forward  # noqa: E402
from test_gpu_fuzz import _case  # noqa: E402


def main():
    oracle.build()
    for seed in map(int, sys.argv[1:]):
        p, cams, rp = _case(seed)
        n, V = p.shape[1], len(cams)
        W, H = cams[0]["width"], cams[0]["height"]
        rz, pt = run_forward(p, cams, rp)
        decs = [oracle.decide(p, c, rp) for c in cams]
        dl = synth.dl_dimage(V, W, H, 1000 + seed)
        o = np.zeros((20, n)); a = np.zeros((20, n)); aS = np.zeros((6, n))
        amb = []
        for v, cam in enumerate(cams):
            r = oracle.render(p, cam, rp, decision=decs[v])
            amb.append(int(r["amb_px"].sum()))
            dl[v][:, r["amb_px"] != 0] = 0.0
        for v, cam in enumerate(cams):
            r = oracle.render(p, cam, rp, dl_dimage=dl[v], decision=decs[v])
            o += r["grad"]; a += r["absg"]; aS += r["absS"]
        g = run_backward(rz, pt, dl)
        a[14:20] = np.maximum(a[14:20], aS)   # the S planes' term magnitudes (as _grad_close with absS)
        d = np.abs(g - o)
        tol = 1e-3 * np.abs(o) + 1e-5 * a + 1e-30
        bad = np.argwhere(d > tol)
        print(f"seed {seed}: n={n} V={V} {W}x{H} rp={rp} amb_px per view={amb} ({W * H} px)")
        pm = np.abs(o).max(axis=1)
        for k, i in bad[np.argsort(-(d[bad[:, 0], bad[:, 1]] / tol[bad[:, 0], bad[:, 1]]))][:12]:
            print(f"   plane {k:2d} G{i:4d}: gpu {g[k, i]: .6e} ora {o[k, i]: .6e} err {d[k, i]:.2e} "
                  f"abs_ora {a[k, i]:.2e} plane_max {pm[k]:.2e}  err/(1e-3|ora|) {d[k, i] / (1e-3 * abs(o[k, i]) + 1e-300):.2f} "
                  f"err/(1e-5 abs) {d[k, i] / (1e-5 * a[k, i] + 1e-300):.2f} err/(1e-6 max) {d[k, i] / (1e-6 * pm[k] + 1e-300):.2f}")


if __name__ == "__main__":
    main()
