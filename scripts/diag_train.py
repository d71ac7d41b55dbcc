"""Diagnostic: worst parameter error of the Trainer vs oracle/train.py, in units of lr, per Adam eps."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np, torch, synth
from oracle.train import train
from gpu_run import raster_of
from paper_2505_05587_b200 import Adam, Schedule, Trainer
SM = dict(alpha_min=0.0, alpha_max=1.0, t_min=0.0, dilation=0.0, bg=(0.0, 0.0, 0.0), tile=16)
LR = (1e-3, 5e-3, 1e-3, 5e-2, 2.5e-3)
GROUP = np.array([0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 4, 4, 4])
cfg = synth.CONFIGS["C1"]
p, cams, tg = synth.scene_for(cfg), synth.ring_cameras(8, 64, 64, 7), synth.target_images(8, 64, 64, 8)
def b(t):
    idx = [(2 * t + k) % 8 for k in range(2)]
    return [cams[i] for i in idx], tg[idx]
variant = sys.argv[1] if len(sys.argv) > 1 else "budget"
kw = dict(budget=16, eps_grad=None) if variant == "budget" else (dict(budget=None, eps_grad=1e-3) if variant == "gate"
                                                                 else dict(budget=None, eps_grad=None))
for eps in (1e-15,):
    for T in (4, 6, 7, 9, 10):
        ora = train(p, 64, 4096, b, T=T, t_start=4, t_split=3, lr=LR, eps=eps, rp=SM, **kw)
        tr = Trainer(torch.from_numpy(p).cuda(), 64, 4096, 2, 64, 64, raster_of(SM), Adam(LR, 0.9, 0.999, eps),
                     Schedule(4, 3, -1e-6, 0.5, kw["eps_grad"], kw["budget"]))
        for t in range(1, T + 1):
            c, y = b(t)
            tr.step(c, torch.from_numpy(np.ascontiguousarray(y)).cuda())
        got = tr.params[:, :tr.n].double().cpu().numpy()
        ok = tr.n == ora["n"]
        if not ok:
            print(eps, T, "n mismatch", tr.n, ora["n"]); continue
        e = np.abs(got - ora["params"]) / np.asarray(LR)[GROUP][:, None]
        k = np.unravel_index(np.argmax(e), e.shape)
        print(f"eps={eps} T={T} n={tr.n} max err/lr per plane:", np.round(e.max(1), 5), "worst", k,
              "p99.9", np.quantile(e, 0.999))
