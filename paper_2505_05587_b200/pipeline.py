"""Host-side orchestration of the hot path on torch-owned device buffers.

`Rasterizer` owns the per-call buffers for a fixed (capacity, V, W, H) and issues the C-ABI calls
in order on one CUDA stream with no host synchronisation (the whole step is graph-capturable).
PyTorch is used for memory and streams only; every computation happens in libsteepgs.
"""
from __future__ import annotations

import dataclasses

import torch

from . import _lib

N_PLANES = 14
N_ACC = 20


@dataclasses.dataclass
class Raster:
    alpha_min: float = 1.0 / 255.0
    alpha_max: float = 0.99
    t_min: float = 1e-4
    dilation: float = 0.3
    bg: tuple = (0.0, 0.0, 0.0)

    def c(self):
        return _lib.raster_params(self.alpha_min, self.alpha_max, self.t_min, self.dilation, self.bg, 16)


SMOOTH = Raster(0.0, 1.0, 0.0, 0.0)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2505_05587_b200 needs a CUDA device of compute capability 10.x (no CPU fallback)")
    major, _ = torch.cuda.get_device_capability()
    if major != 10:
        raise RuntimeError("paper_2505_05587_b200 is built for sm_100a only")


class Rasterizer:
    def __init__(self, capacity: int, V: int, width: int, height: int, raster: Raster | None = None,
                 max_instances: int | None = None, device="cuda"):
        require_cuda()
        self.cap, self.V, self.W, self.H = int(capacity), int(V), int(width), int(height)
        self.raster = raster or Raster()
        self.rp = self.raster.c()
        self.device = torch.device(device)
        d = self.device
        VN = self.V * self.cap
        self.max_instances = int(max_instances if max_instances is not None else max(4 * VN, 1 << 16))
        self.splats = torch.empty(max(VN, 1) * _lib.SPLAT_BYTES, dtype=torch.uint8, device=d)
        self.depth_key = torch.empty(max(VN, 1), dtype=torch.int32, device=d)
        self.tile_rect = torch.empty(max(VN, 1) * 2, dtype=torch.int32, device=d)
        self.tiles_touched = torch.empty(max(VN, 1), dtype=torch.int32, device=d)
        ws = _lib.bin_sort_workspace_size(self.cap, self.V, self.W, self.H, self.max_instances)
        self.sort_ws = torch.empty(ws, dtype=torch.uint8, device=d)
        HW = self.W * self.H
        self.image = torch.empty(self.V, 3, self.H, self.W, dtype=torch.float32, device=d)
        self.final_T = torch.empty(self.V, self.H, self.W, dtype=torch.float32, device=d)
        self.n_contrib = torch.empty(self.V, self.H, self.W, dtype=torch.int32, device=d)
        self.dL = torch.empty(self.V, 3, self.H, self.W, dtype=torch.float32, device=d)
        self.loss = torch.zeros(self.V, dtype=torch.float32, device=d)
        self.moments = torch.zeros(max(VN, 1) * 12, dtype=torch.float32, device=d)  # must start at zero
        self.dens_ws = torch.empty(_lib.densify_workspace_size(self.cap), dtype=torch.uint8, device=d)
        self.split_mask = torch.empty(self.cap, dtype=torch.uint8, device=d)
        self.dest_index = torch.empty(self.cap, dtype=torch.int32, device=d)
        self.lambda_min = torch.empty(self.cap, dtype=torch.float32, device=d)
        self.n_split = torch.zeros(1, dtype=torch.int64, device=d)
        self.dens_status = torch.zeros(1, dtype=torch.int32, device=d)
        self.binning = None
        self.cams_arr = None
        self.n = 0
        self._HW = HW

    # ---- a1 ----
    def project(self, params: torch.Tensor, n: int, cams: list[dict], sh_rest: torch.Tensor | None = None,
                sh_degree: int | None = None):
        """a1; with sh_degree (0..3) the colour comes from spherical harmonics (f3): DC = planes 11-13,
        sh_rest [3 ((deg + 1)^2 - 1)][ld_sh]."""
        assert len(cams) == self.V and params.shape[0] == N_PLANES and n <= self.cap
        self.n = int(n)
        self.cams_arr = _lib.cameras(cams)
        if sh_degree is None:
            _lib.project(params, params.shape[1], self.n, self.cams_arr, self.V, self.rp, self.splats, self.depth_key,
                         self.tile_rect, self.tiles_touched)
        else:
            _lib.project_sh(params, params.shape[1], self.n, sh_rest, sh_degree, self.cams_arr, self.V, self.rp,
                            self.splats, self.depth_key, self.tile_rect, self.tiles_touched)

    # ---- a2 ----
    def bin_sort(self, check: bool = False):
        """a2.  check=True reads the instance count back (one host sync) and, if it exceeds
        max_instances, grows the instance buffers to 1.5x the count and sorts again; without it an
        overflow is only flagged on the device (binning_arrays()["overflow"]) and the step is invalid."""
        self.binning = _lib.bin_sort(self.depth_key, self.tile_rect, self.tiles_touched, self.n, self.cams_arr, self.V,
                                     self.rp, self.sort_ws, self.max_instances)
        if check:
            base = self.sort_ws.data_ptr()
            off = self.binning.n_instances - base
            inst = int(self.sort_ws[off:off + 8].view(torch.int64).item())
            if inst > self.max_instances:
                self.max_instances = int(inst * 1.5) + 1024
                ws = _lib.bin_sort_workspace_size(self.cap, self.V, self.W, self.H, self.max_instances)
                self.sort_ws = torch.empty(ws, dtype=torch.uint8, device=self.device)
                self.binning = _lib.bin_sort(self.depth_key, self.tile_rect, self.tiles_touched, self.n, self.cams_arr,
                                             self.V, self.rp, self.sort_ws, self.max_instances)

    # ---- a3 ----
    def render_fwd(self, pair_counts: torch.Tensor | None = None):
        _lib.render_fwd(self.splats, self.n, self.binning, self.cams_arr, self.V, self.rp, self.image, self.final_T,
                        self.n_contrib, pair_counts)

    def render_fwd_l1(self, targets: torch.Tensor, scale: float | None = None, with_loss: bool = True,
                      pair_counts: torch.Tensor | None = None):
        """a3 + a4 fused: the forward writes dL/dimage = scale sign(image - target) (default scale
        1/(3HW), the per-view mean) and the per-view loss in its epilogue.  targets: float32, or uint8
        (decoded as target * (1/255) in fp32 on the device)."""
        sc = 1.0 / (3 * self._HW) if scale is None else scale
        fn = _lib.render_fwd_l1_u8 if targets.dtype == torch.uint8 else _lib.render_fwd_l1   # 8-bit: decoded * (1/255)
        if targets.dtype not in (torch.uint8, torch.float32) or not targets.is_contiguous():
            raise TypeError("targets: contiguous float32 or uint8 [V][3][H][W]")
        fn(self.splats, self.n, self.binning, self.cams_arr, self.V, self.rp, self.image, self.final_T, self.n_contrib,
           targets, sc, self.dL, self.loss if with_loss else None, pair_counts)

    # ---- a4 ----
    def l1_grad(self, targets: torch.Tensor, with_loss: bool = True):
        count = 3 * self._HW
        _lib.l1_grad(self.image, targets, self.V, count, 1.0 / count, self.dL, self.loss if with_loss else None)

    # ---- a5 + a6 ----
    def render_bwd(self, params: torch.Tensor, grad_S: torch.Tensor, dL: torch.Tensor | None = None,
                   accumulate: int = 0, view_grad_stats: torch.Tensor | None = None):
        dl = self.dL if dL is None else dL
        _lib.render_bwd_split(params, params.shape[1], self.n, self.splats, self.binning, self.cams_arr, self.V,
                              self.rp, self.final_T, self.n_contrib, dl, self.moments, grad_S, grad_S.shape[1],
                              accumulate, self.tiles_touched if view_grad_stats is not None else None,
                              view_grad_stats)

    def render_bwd_moments(self, dL: torch.Tensor | None = None):
        """a5 only (per-pixel replay -> moments)."""
        _lib.render_bwd_moments(self.splats, self.n, self.binning, self.cams_arr, self.V, self.rp, self.final_T,
                                self.n_contrib, self.dL if dL is None else dL, self.moments)

    def gauss_bwd(self, params: torch.Tensor, grad_S: torch.Tensor, accumulate: int = 0,
                  view_grad_stats: torch.Tensor | None = None):
        """a6 only (moments -> dL/dparams and S; optionally the ADC view-gradient statistics, f4)."""
        _lib.gauss_bwd_split(params, params.shape[1], self.n, self.cams_arr, self.V, self.rp,
                             self.moments, grad_S, grad_S.shape[1], accumulate,
                             self.tiles_touched if view_grad_stats is not None else None, view_grad_stats)

    def sh_bwd(self, params: torch.Tensor, grad_S: torch.Tensor, sh_rest, sh_degree: int, grad_sh,
               accumulate: int = 0):
        """f3: SH colour backward (between render_bwd_moments and gauss_bwd(accumulate | 4))."""
        _lib.sh_bwd(params, self.n, sh_rest, sh_degree, self.cams_arr, self.V, self.moments, grad_S, grad_sh,
                    accumulate)

    # ---- a8 ----
    def densify(self, params: torch.Tensor, grad_S: torch.Tensor, n: int, capacity: int, eps_split=-1e-6, eta=0.5,
                eps_abs=0.0, denom=1.0, want_lambda=True, eps_grad=None, budget=None, grad_gate=None):
        """SDC densify (Thm 2).  eps_grad: compactest gate (App. A.2); budget: split at most this many;
        grad_gate: Alg. 1's condition on G as 3DGS's view-gradient threshold (planes 0, 1 = statistic)."""
        dp = _lib.densify_params(eps_split, eta, eps_abs, denom, eps_grad, budget, grad_gate)
        _lib.densify(params, params.shape[1], n, capacity, grad_S, grad_S.shape[1], dp, self.split_mask,
                     self.dest_index, self.lambda_min if want_lambda else None, self.n_split, self.dens_status,
                     self.dens_ws)

    # ---- f4 ----
    def densify_adc(self, params: torch.Tensor, grad_S: torch.Tensor, stats: torch.Tensor, normals: torch.Tensor,
                    n: int, capacity: int, eps_adc: float, tau_adc: float, clone_step: float = 0.0,
                    scale_factor: float = 0.8, denom: float = 1.0):
        """3DGS ADC baseline: clone / split by the mean view-space gradient norm."""
        if not hasattr(self, "adc_ws"):
            self.adc_ws = torch.empty(_lib.adc_workspace_size(self.cap), dtype=torch.uint8, device=self.device)
            self.adc_kind = torch.empty(self.cap, dtype=torch.uint8, device=self.device)
        ap = _lib.adc_params(eps_adc, tau_adc, clone_step, scale_factor, denom)
        _lib.densify_adc(params, n, capacity, grad_S, stats, normals, ap, self.adc_kind, self.dest_index, self.n_split,
                         self.dens_status, self.adc_ws)

    def forward_backward(self, params, n, cams, targets=None, grad_S=None, dL=None, accumulate=False):
        """a1..a6 for the V views of this call (no host sync)."""
        self.project(params, n, cams)
        self.bin_sort()
        self.render_fwd()
        if dL is None:
            self.l1_grad(targets)
        self.render_bwd(params, grad_S, dL=dL, accumulate=accumulate)

    # ---- host-side readers (tests / diagnostics; they synchronise) ----
    def binning_arrays(self):
        """(ids[I], ranges[V*tiles][2], I, overflow, tile_order[V*tiles]) copied to host."""
        b = self.binning
        base = self.sort_ws.data_ptr()
        def view(ptr_, nbytes, dtype):
            off = ptr_ - base
            return self.sort_ws[off:off + nbytes].view(dtype)
        I = int(view(b.n_instances, 8, torch.int64).item())
        ovf = int(view(b.overflow, 4, torch.int32).item())
        nv = int(view(b.n_visible, 8, torch.int64).item())
        tiles = b.tiles_x * b.tiles_y * b.V
        ids = view(b.ids, 4 * min(I, self.max_instances), torch.int32).cpu()
        ranges = view(b.ranges, 8 * tiles, torch.int32).view(tiles, 2).cpu()
        order = view(b.tile_order, 4 * tiles, torch.int32).cpu()   # view << 20 | tile
        return dict(ids=ids, ranges=ranges, n_instances=I, overflow=ovf, n_visible=nv, tile_order=order)


# ---------------------------------------------------------------------------------------------
# NEXT f1: the Algorithm-1 loop with the paper's schedule.
# Readings C17-C20: Adam per parameter group; densify steps take no gradient step;
# G and S windows restart after step t_start - T_split and after each densify (denominator T_split);
# split parents and offspring restart with zero Adam moments, the step count is global.
# ---------------------------------------------------------------------------------------------
@dataclasses.dataclass
class Adam:
    lr: tuple = (1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3)   # mean, log-scale, quaternion, opacity logit, rgb (3DGS)
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15


@dataclasses.dataclass
class Schedule:
    t_start: int = 500          # "density control for every 100 steps starting from the 500th step"
    t_split: int = 100
    eps_split: float = -1e-6
    eta: float = 0.5
    eps_grad: float | None = None   # compactest gate (App. A.2)
    budget: int | None = None       # increment budget (App. A.2)
    density: str = "sdc"            # "sdc" (Alg. 1) or "adc" (3DGS baseline, f4)
    grad_gate: float | None = None  # SDC: Alg. 1's "condition on G" as 3DGS's mean view-gradient threshold
                                    # (pixel units, C24); None: no condition (Z12)
    eps_adc: float | None = None    # ADC threshold on the mean ||dL/dPi(p)|| in pixel units; None: 3DGS's
                                    # 0.0002 in NDC units = 0.0004 / W (C22)
    tau_adc: float = 2e-3           # ADC clone/split boundary on ||Sigma||_2 = (0.01 x scene extent ~4.4)^2
    clone_step: float = 0.0         # ADC clone displacement along -G / T_split
    scale_factor: float = 0.8       # ADC split offspring scale
    min_opacity: float | None = None  # prune Gaussians below this opacity after each densify (3DGS: 0.005)
    t_stop: int | None = 15000      # last step that may densify (3DGS's densify_until_iter; the paper keeps
                                    # 3DGS's other hyper-parameters); None: Alg. 1 without a bound

    def densify_at(self, t: int) -> bool:
        if self.t_stop is not None and t > self.t_stop:
            return False
        return t >= self.t_start and (t - self.t_start) % self.t_split == 0

    def window_restarts_after(self, t: int) -> bool:
        return t == self.t_start - self.t_split or self.densify_at(t)


class Trainer:
    """Algorithm 1 on one GPU (or view-sharded over a process group: the 14 gradient planes are
    allreduced every step so the Adam update stays replicated, the 6 S planes only before densify).

    Device state, all [plane][capacity] fp32: params (14), grad_S (20: per-step gradients + the
    window's S), adam m/v (14 each), gacc (3: the window's position-gradient sum G); optionally the
    ADC statistic (2), SH rest coefficients with their gradients and Adam moments.  Host syncs: the
    tile-instance count after each bin_sort (`check_overflow`, grows the buffers when a scene's
    footprint outgrows them) and the new Gaussian count at each densify step."""

    def __init__(self, params0: torch.Tensor, n: int, capacity: int, V: int, width: int, height: int,
                 raster: Raster | None = None, adam: Adam | None = None, schedule: Schedule | None = None,
                 max_instances: int | None = None, group=None, seed: int = 0, normals_fn=None,
                 sh_degree: int | None = None, sh_rest0: torch.Tensor | None = None, sh_lr: float = 2.5e-3 / 20,
                 ssim_lambda: float | None = None):
        require_cuda()
        self.cap, self.n = int(capacity), int(n)
        if self.n > self.cap:
            raise ValueError("n > capacity")
        self.rz = Rasterizer(self.cap, V, width, height, raster, max_instances)
        d = self.rz.device
        self.params = torch.zeros(N_PLANES, self.cap, dtype=torch.float32, device=d)
        self.params[:, :self.n].copy_(params0[:, :self.n])
        self.grad_S = torch.zeros(N_ACC, self.cap, dtype=torch.float32, device=d)
        self.m = torch.zeros(N_PLANES, self.cap, dtype=torch.float32, device=d)
        self.v = torch.zeros(N_PLANES, self.cap, dtype=torch.float32, device=d)
        self.gacc = torch.zeros(3, self.cap, dtype=torch.float32, device=d)
        sch = schedule or Schedule()
        self.vstats = torch.zeros(2, self.cap, dtype=torch.float32, device=d) \
            if (sch.density == "adc" or sch.grad_gate is not None) else None
        self.normals = None
        self.normals_fn = normals_fn     # ADC: t -> [6][>= n] device normals; default: drawn on the device
        self.generator = torch.Generator(device=d)
        self.generator.manual_seed(seed)
        self.sh_degree = sh_degree
        self.sh_rest = self.grad_sh = self.m_sh = self.v_sh = None
        if sh_degree is not None:
            planes = 3 * ((sh_degree + 1) ** 2 - 1)
            mk = lambda: torch.zeros(max(planes, 1), self.cap, dtype=torch.float32, device=d)[:planes]
            self.sh_rest, self.grad_sh, self.m_sh, self.v_sh = mk(), mk(), mk(), mk()
            if sh_rest0 is not None and planes > 0:
                self.sh_rest[:, :self.n].copy_(sh_rest0[:planes, :self.n])
        self.ssim_lambda = ssim_lambda   # None: l1 loss; else (1 - lambda) l1 + lambda (1 - SSIM) (3DGS: 0.2)
        self.loss_ws = None
        if ssim_lambda is not None:
            self.loss_ws = torch.empty(_lib.loss_workspace_size(V, height, width), dtype=torch.uint8, device=d)
        self.adam = adam or Adam()
        self.ap_sh = _lib.adam_params((sh_lr,) * 5, self.adam.beta1, self.adam.beta2, self.adam.eps)
        self.ap = _lib.adam_params(self.adam.lr, self.adam.beta1, self.adam.beta2, self.adam.eps)
        self.sched = schedule or Schedule()
        self.group = group
        self.t = 0              # training steps done
        self.opt_steps = 0      # Adam steps done
        self.fresh = True       # the next gradient step opens an accumulation window
        self.history: list[dict] = []
        self.check_overflow = True   # grow the tile-instance buffers when needed (one 8-B read per step)

    def _world(self) -> int:
        import torch.distributed as dist
        return dist.get_world_size(self.group) if dist.is_available() and dist.is_initialized() else 1

    def _batch_views(self) -> int:
        """Views in one gradient step over all ranks.  The step's loss is their mean (C18), so the
        statistic k_gauss_bwd accumulates, ||dL_batch/dPi(p)||, is the per-view ||dL_view/dPi(p)|| of
        C22 / 3DGS divided by this count; the ADC threshold and the C24 gate are divided by it instead
        (the norm is positively homogeneous, so the decision is the same)."""
        return self.rz.V * self._world()

    def _allreduce_planes(self, first: int, count: int):
        if self._world() > 1:
            from .parallel import allreduce_planes
            allreduce_planes(self.grad_S, first, count, self.n, self.group)

    def _allreduce_stats(self):
        if self._world() > 1:
            from .parallel import allreduce_planes
            allreduce_planes(self.vstats, 0, 2, self.n, self.group)

    def step(self, cams: list[dict] | None = None, targets: torch.Tensor | None = None) -> dict:
        """Training step t = self.t + 1: a densify step (cams/targets ignored) or a gradient step on
        the batch (len(cams) == V views, targets [V][3][H][W] on the device)."""
        t = self.t + 1
        if self.sched.densify_at(t):
            info = self._densify(t)
        else:
            rz = self.rz
            sh = self.sh_degree is not None
            rz.project(self.params, self.n, cams, self.sh_rest, self.sh_degree)
            rz.bin_sort(check=self.check_overflow)
            count = 3 * rz._HW
            if self.ssim_lambda is None:
                rz.render_fwd_l1(targets, 1.0 / (count * rz.V * self._world()))
            else:
                rz.render_fwd()
                _lib.l1_ssim_grad(rz.image, targets, self.ssim_lambda, 1.0 / (rz.V * self._world()), rz.dL, rz.loss,
                                  self.loss_ws)
            rz.render_bwd_moments()
            mode = 0 if self.fresh else 2
            if sh:
                rz.sh_bwd(self.params, self.grad_S, self.sh_rest, self.sh_degree, self.grad_sh, mode)
            rz.gauss_bwd(self.params, self.grad_S, accumulate=mode | (4 if sh else 0), view_grad_stats=self.vstats)
            self._allreduce_planes(0, N_PLANES)
            if sh and self.grad_sh.shape[0] > 0 and self._world() > 1:
                from .parallel import allreduce_planes
                allreduce_planes(self.grad_sh, 0, self.grad_sh.shape[0], self.n, self.group)
            self.opt_steps += 1
            _lib.adam_step(self.params, self.n, self.grad_S, self.m, self.v, self.ap, self.opt_steps, self.gacc,
                           gacc_accumulate=not self.fresh)
            if sh and self.grad_sh.shape[0] > 0:
                _lib.adam_step_planes(self.sh_rest, self.n, self.grad_sh, self.m_sh, self.v_sh, self.ap_sh,
                                      self.opt_steps)
            self.fresh = False
            info = dict(t=t, kind="grad")
        if self.sched.window_restarts_after(t):
            self.fresh = True
        self.t = t
        return info

    def _densify(self, t: int) -> dict:
        rz, s = self.rz, self.sched
        n = self.n
        _lib.copy_planes(self.grad_S, self.gacc, n, 0, 3)           # G -> accumulator planes 0-2 (gate / clone)
        if s.density == "adc":
            self._allreduce_stats()
            if self.normals_fn is not None:
                self.normals = self.normals_fn(t)
            else:                                                      # z ~ N(0, I): an input of the method
                if self.normals is None:
                    self.normals = torch.empty(6, self.cap, dtype=torch.float32, device=rz.device)
                self.normals.normal_(generator=self.generator)
            eps_adc = (s.eps_adc if s.eps_adc is not None else 0.0004 / rz.W) / self._batch_views()
            rz.densify_adc(self.params, self.grad_S, self.vstats, self.normals, n, self.cap, eps_adc, s.tau_adc,
                           s.clone_step, s.scale_factor, float(s.t_split))
            reset_mask, reset_value = rz.adc_kind, 2                   # clone parents keep their Adam state
        else:
            self._allreduce_planes(14, 6)
            if s.grad_gate is not None:                                # statistic -> planes 0, 1 (gate 2)
                self._allreduce_stats()
                _lib.copy_planes(self.grad_S, self.vstats, n, 0, 2)
            gg = s.grad_gate / self._batch_views() if s.grad_gate is not None else None
            rz.densify(self.params, self.grad_S, n, self.cap, eps_split=s.eps_split, eta=s.eta,
                       denom=float(s.t_split), eps_grad=s.eps_grad, budget=s.budget, grad_gate=gg)
            reset_mask, reset_value = rz.split_mask, 1
        ns, st = int(rz.n_split.item()), int(rz.dens_status.item())
        if st != 0:
            raise _lib.SteepGSError("steepgs_densify", 3, f"capacity {self.cap} < {n} + {ns}")
        _lib.reset_moments(self.m, self.v, n, reset_mask, rz.n_split, reset_value)
        if self.sh_rest is not None and self.sh_rest.shape[0] > 0:
            _lib.copy_offspring(self.sh_rest, n, rz.dest_index)          # offspring inherit the SH rest
            _lib.reset_moments(self.m_sh, self.v_sh, n, reset_mask, rz.n_split, reset_value)
        self.n = n + ns
        n_pruned = self._prune() if s.min_opacity is not None else 0
        info = dict(t=t, kind="densify", n_before=n, n_split=ns, n_pruned=n_pruned)
        self.history.append(info)
        return info

    def _prune(self) -> int:
        """Opacity pruning after a densify (kept from 3DGS's density control): keep iff the
        opacity logit >= logit(min_opacity) (an exact fp32 comparison), compact every per-Gaussian
        buffer (params, Adam moments, SH rest and its moments) out of place, stable order."""
        import math
        n = self.n
        if not hasattr(self, "_prune_ws"):
            self._prune_ws = torch.empty(_lib.prune_workspace_size(self.cap), dtype=torch.uint8,
                                         device=self.params.device)
            self._new_index = torch.empty(self.cap, dtype=torch.int32, device=self.params.device)
            self._n_keep = torch.zeros(1, dtype=torch.int64, device=self.params.device)
        m = self.sched.min_opacity
        logit_min = float(torch.tensor(math.log(m / (1.0 - m)), dtype=torch.float32))
        _lib.prune_decide(self.params, n, logit_min, self._new_index, self._n_keep, self._prune_ws)
        keep = int(self._n_keep.item())
        if keep == n:
            return 0
        names = ["params", "m", "v"] + (["sh_rest", "m_sh", "v_sh"] if self.sh_rest is not None
                                        and self.sh_rest.shape[0] > 0 else [])
        for name in names:
            src = getattr(self, name)
            dst = torch.empty_like(src)
            _lib.compact_planes(src, dst, n, self._new_index)
            setattr(self, name, dst)
        self.n = keep
        return n - keep

    def loss(self) -> torch.Tensor:
        """Per-view losses of the last gradient step ([V], device)."""
        return self.rz.loss
