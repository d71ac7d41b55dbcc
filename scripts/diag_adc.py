"""Diagnostic: ADC training loop, Trainer vs oracle/train.py — worst error per plane / Gaussian."""
import os, sys
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
cap = 1024
zs = {t: np.random.default_rng(100 + t).normal(size=(6, cap)).astype(np.float32) for t in (4, 7, 10)}
adc = dict(eps_adc=6e-5, tau_adc=0.07, clone_step=float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3, scale_factor=0.8)
for T in (5, 7, 8, 10):
    ora = train(p, 64, cap, b, T=T, t_start=4, t_split=3, lr=LR, eps=1e-15, rp=SM, density="adc", adc=adc,
                normals=lambda t: zs[t].astype(np.float64))
    sched = Schedule(4, 3, density="adc", eps_adc=adc["eps_adc"], tau_adc=adc["tau_adc"], clone_step=adc["clone_step"],
                     scale_factor=0.8)
    tr = Trainer(torch.from_numpy(p).cuda(), 64, cap, 2, 64, 64, raster_of(SM), Adam(LR, 0.9, 0.999, 1e-15), sched,
                 normals_fn=lambda t: torch.from_numpy(zs[t]).cuda())
    for t in range(1, T + 1):
        c, y = b(t)
        tr.step(c, torch.from_numpy(np.ascontiguousarray(y)).cuda())
    got = tr.params[:, :tr.n].double().cpu().numpy()
    if tr.n != ora["n"]:
        print(T, "n mismatch", tr.n, ora["n"]); continue
    e = np.abs(got - ora["params"]) / np.asarray(LR)[GROUP][:, None]
    k = np.unravel_index(np.argmax(e), e.shape)
    print(f"T={T} n={tr.n} splits={ora['n_split']} max err/lr per plane:", np.round(e.max(1), 4), "worst at", k)
