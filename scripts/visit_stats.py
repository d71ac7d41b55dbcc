import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import synth
from gpu_run import to_dev
from paper_2505_05587_b200.pipeline import Rasterizer
cfg = synth.CONFIGS["C2"]; n = cfg.n; V = 8
p = synth.scene_for(cfg); cams = synth.cameras_for(cfg, views=V)
rz = Rasterizer(2 * n, V, cfg.width, cfg.height, max_instances=int(3.0 * V * n))
P = torch.zeros(14, 2 * n, device="cuda"); P[:, :n] = to_dev(p)
pc = torch.zeros(4, dtype=torch.int64, device="cuda")
rz.project(P, n, cams); rz.bin_sort(); rz.render_fwd(pc); torch.cuda.synchronize()
c = pc.cpu().tolist()
print("comp pairs", c[0], "evaluated", c[1], "fwd visits (8x4, before warp done)", c[2], "visits with >= 1 composite", c[3], "frac", c[3] / max(c[2], 1))
