"""Algorithm 1 (SteepGS training loop) on the CPU oracle.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module.  It composes the fp64 oracle (render + densify from liboracle.so) with a textbook Adam
written out in numpy fp64; it shares nothing with the CUDA product.

Readings (C17-C20):
  C17  "update each Gaussian parameters via standard gradient descent" = the optimiser
       3DGS trains with: Adam (Kingma & Ba 2015, Alg. 1), one lr per parameter group (mean,
       log-scale, quaternion, opacity logit, rgb), bias corrections with the global step count t.
  C18  Schedule: a step t is a densify step iff t >= t_start and (t - t_start) % T_split
       == 0; such a step takes no gradient step (Alg. 1's if/else).  Every other step renders its
       batch, takes one Adam step and accumulates G (position gradient) and S.
  C19  Accumulation windows: G and S restart after step t_start - T_split and after every densify
       step, so each densify sees the T_split - 1 gradient steps since the last one and divides by
       T_split as written.
  C20  Split parents and both offspring restart with zero Adam moments (they are new Gaussians,
       P:L547); the step count t is global.
The per-step loss is the batch mean of the per-view L1 (Eq. eqn:loss with lambda = 0):
dL/dimage = sign(image - target) / (3 H W V).
"""
from __future__ import annotations

import numpy as np

from . import densify as _densify
from . import render as _render
from .adc import adc_densify
from .ssim import loss_and_grad as ssim_loss_and_grad

# plane -> parameter group (mean, log-scale, quaternion, opacity logit, rgb)
PLANE_GROUP = np.array([0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 4, 4, 4])


def adam_step(p, g, m, v, lr, beta1, beta2, eps, t):
    """Kingma & Ba 2015, Algorithm 1, one step on [14][n] fp64 arrays (in place).  lr: 5 group lrs."""
    lr_plane = np.asarray(lr, dtype=np.float64)[PLANE_GROUP][:, None]
    m *= beta1
    m += (1.0 - beta1) * g
    v *= beta2
    v += (1.0 - beta2) * g * g
    m_hat = m / (1.0 - beta1 ** t)
    v_hat = v / (1.0 - beta2 ** t)
    p -= lr_plane * m_hat / (np.sqrt(v_hat) + eps)


def adam_step_dense(p, g, m, v, lr, beta1, beta2, eps, t):
    """The same Adam step with one learning rate for every plane (SH rest coefficients, f3)."""
    m *= beta1
    m += (1.0 - beta1) * g
    v *= beta2
    v += (1.0 - beta2) * g * g
    p -= lr * (m / (1.0 - beta1 ** t)) / (np.sqrt(v / (1.0 - beta2 ** t)) + eps)


def is_densify_step(t: int, t_start: int, t_split: int) -> bool:
    return t >= t_start and (t - t_start) % t_split == 0


def window_restarts_after(t: int, t_start: int, t_split: int) -> bool:
    return t == t_start - t_split or is_densify_step(t, t_start, t_split)


def train(params0, n0: int, capacity: int, batches, T: int, t_start: int, t_split: int, lr, beta1=0.9,
          beta2=0.999, eps=1e-15, rp=None, eps_split=-1e-6, eta=0.5, eps_grad=None, budget=None,
          density="sdc", adc=None, normals=None, sh_degree=None, sh_rest0=None, sh_lr=2.5e-3 / 20,
          ssim_lambda=None, grad_gate=None, min_opacity=None):
    """Run steps t = 1..T.  batches(t) -> (cams, targets [V][3][H][W]) for gradient steps.
    density = "adc": the 3DGS baseline (oracle/adc.py) with adc = dict(eps_adc, tau_adc, clone_step,
    scale_factor) and normals(t) -> [6][>=n] standard normals for that densify step.
    sh_degree (f3): SH colours (DC = planes 11-13, rest [3 (K - 1)][n] from sh_rest0), the rest
    coefficients trained by Adam with the single rate sh_lr and copied to offspring.
    ssim_lambda (f3): per-view loss (1 - lambda) l1 + lambda (1 - SSIM) (oracle/ssim.py), batch mean.
    grad_gate (C24): SDC splits only Gaussians whose mean view-space gradient norm >= grad_gate.
    min_opacity: after each densify, Gaussians whose opacity logit is below the fp32 logit of
    min_opacity are removed (3DGS's pruning), the rest keep their order.
    Returns dict(params [14][n], n, n_split, lambda_min [n] and ||G / T_split|| [n] per densify step, loss per
    gradient step); for "adc" lambda_min holds the mean view-gradient statistic and g_norm ||Sigma||_2.
    pos_sens [n]: for the parity test's per-Gaussian position tolerance, an upper bound on how far an
    offspring's position moves when its parent's S-bar carries the parity tolerance of S (DESIGN.md
    §3.4: |dS| <= 1e-3 |S| + 1e-5 sum|per-pair S|): with E that perturbation, Davis-Kahan gives
    ||dv|| <= 2 ||E||_F / gap (gap = lambda_2 - lambda_1 of S-bar), and the displacement eps v with
    eps = eta sqrt(v^T Sigma v) moves by <= 2 eta sqrt(lambda_max(Sigma)) ||dv||; summed along the
    Gaussian's lineage (both offspring inherit the parent's bound)."""
    P = np.zeros((14, capacity))
    P[:, :n0] = np.asarray(params0, dtype=np.float64)[:, :n0]
    m = np.zeros((14, capacity))
    v = np.zeros((14, capacity))
    G = np.zeros((3, capacity))
    S = np.zeros((6, capacity))
    S_abs = np.zeros((6, capacity))   # sum of |per-pair S| (the parity tolerance's absolute term)
    sens = np.zeros(capacity)          # pos_sens (see the docstring)
    st_sum = np.zeros(capacity)        # ADC statistic: sum of ||dL/dPi(p)|| over visible views
    st_cnt = np.zeros(capacity)
    n = n0
    opt_t = 0
    nrest = 3 * ((sh_degree + 1) ** 2 - 1) if sh_degree is not None else 0
    SHr = np.zeros((nrest, capacity)); mr = np.zeros((nrest, capacity)); vr = np.zeros((nrest, capacity))
    if nrest:
        SHr[:, :n0] = np.asarray(sh_rest0, dtype=np.float64)[:nrest, :n0]

    def spawn_rest(dest, reset):
        if nrest:
            for i in np.flatnonzero(dest >= 0):
                SHr[:, dest[i]] = SHr[:, i]
            mr[:, reset] = 0.0
            vr[:, reset] = 0.0
    splits, losses, lams, gnorms = [], [], [], []
    pruned, logits = [], []
    for t in range(1, T + 1):
        if is_densify_step(t, t_start, t_split) and density == "adc":
            d = adc_densify(P, G, st_sum, st_cnt, n, capacity, adc["eps_adc"], adc["tau_adc"], adc["clone_step"],
                            adc["scale_factor"], float(t_split), normals(t))
            if d["n_new"] < 0:
                raise RuntimeError("capacity exceeded")
            with np.errstate(invalid="ignore", divide="ignore"):
                lams.append(np.where(st_cnt[:n] > 0, st_sum[:n] / st_cnt[:n], 0.0))
            gnorms.append(np.exp(2.0 * P[3:6, :n]).max(0))
            ns = d["n_new"]
            P = np.zeros((14, capacity))
            P[:, :n + ns] = d["params"]
            reset = np.zeros(capacity, bool)
            reset[:n] = d["kind"] == 2
            reset[n:n + ns] = True
            m[:, reset] = 0.0
            v[:, reset] = 0.0
            spawn_rest(d["dest"], reset)
            n += ns
            splits.append(ns)
        elif is_densify_step(t, t_start, t_split):
            acc = np.zeros((20, capacity))
            acc[0:3] = G
            if grad_gate is not None:       # Alg. 1's condition on G as 3DGS's statistic (C24)
                acc[0], acc[1], acc[2] = st_sum, st_cnt, 0.0
            acc[14:20] = S
            d = _densify(P, acc, n, capacity, denom=float(t_split), eps_split=eps_split, eta=eta,
                         eps_grad=eps_grad, budget=budget, grad_gate=grad_gate)
            if d["n_split"] < 0:
                raise RuntimeError("capacity exceeded")
            lams.append(d["lambda_min"].copy())
            if grad_gate is not None:
                with np.errstate(invalid="ignore", divide="ignore"):
                    gnorms.append(np.where(st_cnt[:n] > 0, st_sum[:n] / st_cnt[:n], 0.0))
            else:
                gnorms.append(np.linalg.norm(G[:, :n], axis=0) / t_split)
            sp = np.flatnonzero(d["mask"])
            if sp.size:
                Sb = S[:, sp] / t_split
                E = (1e-3 * np.abs(S[:, sp]) + 1e-5 * S_abs[:, sp]) / t_split
                fro = np.sqrt(E[0] ** 2 + E[3] ** 2 + E[5] ** 2 + 2 * (E[1] ** 2 + E[2] ** 2 + E[4] ** 2))
                ev = np.array([np.linalg.eigvalsh(np.array([[a[0], a[1], a[2]], [a[1], a[3], a[4]], [a[2], a[4], a[5]]]))
                               for a in Sb.T])
                gap = np.maximum(ev[:, 1] - ev[:, 0], 1e-300)
                dv = np.minimum(2.0 * fro / gap, 2.0)
                smax = np.exp(2.0 * P[3:6, sp]).max(0)                 # lambda_max(Sigma) = max_k s_k^2
                add = 2.0 * abs(eta) * np.sqrt(smax) * dv if eta > 0 else 0.0 * dv
                sens[sp] += add
                sens[d["dest"][sp]] = sens[sp]
            P = d["params"]
            ns = d["n_split"]
            reset = np.zeros(capacity, bool)
            reset[:n] = d["mask"] != 0
            reset[n:n + ns] = True
            m[:, reset] = 0.0
            v[:, reset] = 0.0
            spawn_rest(d["dest"], reset)
            n += ns
            splits.append(ns)
        else:
            cams, targets = batches(t)
            V = len(cams)
            grad = np.zeros((20, n))
            gsh = np.zeros((nrest, n))
            shkw = dict(sh_rest=SHr[:, :n], sh_degree=sh_degree) if sh_degree is not None else {}
            loss = 0.0
            bw_abs = np.zeros((20, n))
            for k, cam in enumerate(cams):
                fw = _render(P[:, :n], cam, rp, **shkw)
                img = fw["image"]
                H, W = img.shape[1:]
                r = img - np.asarray(targets[k], dtype=np.float64)
                scale = 1.0 / (3.0 * H * W * V)
                if ssim_lambda is None:
                    loss += scale * np.abs(r).sum()
                    dl = np.sign(r) * scale
                else:
                    lv, gv = ssim_loss_and_grad(img, targets[k], ssim_lambda)
                    loss += lv / V
                    dl = gv / V
                bw = _render(P[:, :n], cam, rp, dl_dimage=dl, decision=fw["decision"], **shkw)
                grad += bw["grad"]
                bw_abs += bw["absg"]
                if nrest:
                    gsh += bw["grad_sh"]
                vis = fw["decision"]["visible"] != 0
                # C22: the statistic is the norm of the per-VIEW loss gradient dL_view/dPi(p); the batch
                # loss is the mean over the V views, so its gradient is scaled back by V
                st_sum[:n] += np.where(vis, V * np.hypot(bw["grad_mu"][0], bw["grad_mu"][1]), 0.0)
                st_cnt[:n] += vis
            losses.append(loss)
            opt_t += 1
            adam_step(P[:, :n], grad[:14], m[:, :n], v[:, :n], lr, beta1, beta2, eps, opt_t)
            if nrest:
                adam_step_dense(SHr[:, :n], gsh, mr[:, :n], vr[:, :n], sh_lr, beta1, beta2, eps, opt_t)
            G[:, :n] += grad[0:3]
            S[:, :n] += grad[14:20]
            S_abs[:, :n] += bw_abs[14:20]
        if is_densify_step(t, t_start, t_split) and min_opacity is not None:
            thr = float(np.float32(np.log(min_opacity / (1.0 - min_opacity))))
            keep = np.flatnonzero(P[10, :n] >= thr)
            logits.append(P[10, :n].copy())
            sens[:keep.size] = sens[keep]
            sens[keep.size:] = 0.0
            for arr in (P, m, v, SHr, mr, vr):
                if arr.shape[0]:
                    arr[:, :keep.size] = arr[:, keep]
                    arr[:, keep.size:] = 0.0
            pruned.append(n - keep.size)
            n = keep.size
        if window_restarts_after(t, t_start, t_split):
            G[:] = 0.0
            S[:] = 0.0
            S_abs[:] = 0.0
            st_sum[:] = 0.0
            st_cnt[:] = 0.0
    return dict(params=P[:, :n].copy(), n=n, n_split=splits, loss=losses, lambda_min=lams, g_norm=gnorms,
                sh_rest=SHr[:, :n].copy(), n_pruned=pruned, logits_at_prune=logits,
                pos_sens=sens[:n].copy())
