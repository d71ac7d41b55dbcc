"""Warp-visit statistics from the forward's per-instance sub-block masks (binning.inst_mask): how many
(warp, splat) visits the backward / forward would make with 8x4 warp blocks (1 px per lane, the round-1
layout) vs 8x8 blocks (2 px per lane) vs 16x8.  C2, 2 views."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from gpu_run import to_dev  # noqa: E402
from paper_2505_05587_b200.pipeline import Rasterizer  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n, V = cfg.n, 2
p = synth.scene_for(cfg)
cams = synth.cameras_for(cfg, views=V)
rz = Rasterizer(2 * n, V, cfg.width, cfg.height, max_instances=int(3.0 * V * n))
P = torch.zeros(14, 2 * n, device="cuda")
P[:, :n] = to_dev(p)
rz.project(P, n, cams)
rz.bin_sort()
rz.render_fwd()
torch.cuda.synchronize()
b = rz.binning_arrays()
ni = b["n_instances"]
off = rz.binning.inst_mask - rz.sort_ws.data_ptr()
m = rz.sort_ws[off:off + ni].cpu().numpy().astype(np.int64)
pc = np.array([bin(i).count("1") for i in range(256)])
v84 = pc[m].sum()
b88 = ((m | (m >> 2)) & 0b00110011)
v88 = pc[b88].sum()
b168 = (((m | (m >> 1)) & 0b01010101) | (((m | (m >> 1)) >> 2) & 0b01010101))
v168 = pc[b168 & 0b00010001].sum()
print(f"{cfg.name}: instances {ni}, 8x4 visits {v84} ({v84 / ni:.2f}/inst), 8x8 visits {v88} ({v88 / ni:.2f}/inst, "
      f"ratio {v88 / v84:.3f}), 16x8 visits {v168} (ratio {v168 / v84:.3f}), empty masks {(m == 0).sum()}")
