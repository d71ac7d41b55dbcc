"""Seeded synthetic inputs shared by the CPU oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no projection, compositing, gradient,
splitting matrix or eigen solve).  It only draws inputs: Gaussian parameter planes, cameras,
target images and loss-gradient images, with the shapes and distributions of the workloads in
SURVEY.md §8(d1) / BASELINE.json `configs`.  Every array is float32 (the product's storage
precision); the oracle widens the same values to float64 exactly.

Parameter planes ("params"), planar SoA, shape [14][n] float32:
  0-2  mean p (world units)
  3-5  log-scale log s
  6-9  quaternion (w, x, y, z), not necessarily normalised
  10   opacity logit  (o = sigmoid)
  11-13 rgb colour
Camera dict: R (3x3 world->camera rotation, row-major), t (3), fx, fy, cx, cy, width, height,
model (0 = pinhole EWA, 1 = affine), znear, guard.  Camera looks down +z, image y down.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

N_PLANES = 14
N_ACC = 20  # 14 gradient planes + 6 splitting-matrix planes (xx, xy, xz, yy, yz, zz)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    width: int
    height: int
    views: int
    kind: str  # "blobs" (C1) or "surface" (C2..C5)
    cite: str


# BASELINE.json "configs", in order.  `views` is the per-call view batch used by tests/bench.
CONFIGS = {
    "C1": Config("C1", 64, 64, 64, 1, "blobs", "BASELINE.json configs[0]: tiny, 64 Gaussians, 64x64"),
    "C2": Config("C2", 1_000_000, 980, 545, 16, "surface", "configs[1]: T&T-shaped, 1.0M, 980x545"),
    "C3": Config("C3", 3_000_000, 1237, 822, 8, "surface", "configs[2]: Mip-NeRF360-shaped, 3M, 1237x822"),
    "C4": Config("C4", 2_500_000, 1332, 876, 16, "surface", "configs[3]: Deep-Blending-shaped, 2.5M, 1332x876"),
    "C5": Config("C5", 6_000_000, 1920, 1080, 8, "surface", "configs[4]: 6M, 64 views 1920x1080 over 8 GPUs"),
}


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _frame_to_quat(m: np.ndarray) -> np.ndarray:
    """Rotation matrices [k,3,3] (columns = local axes) -> quaternions [k,4] (w,x,y,z).

    Input construction only (Shepperd's method); the method's own R(q) lives in the oracle
    and in the kernels."""
    k = m.shape[0]
    q = np.empty((k, 4))
    tr = m[:, 0, 0] + m[:, 1, 1] + m[:, 2, 2]
    cases = np.stack([tr, m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]], 1).argmax(1)
    for c in range(4):
        sel = cases == c
        if not sel.any():
            continue
        a = m[sel]
        if c == 0:
            s = np.sqrt(1.0 + tr[sel]) * 2
            q[sel] = np.stack([0.25 * s, (a[:, 2, 1] - a[:, 1, 2]) / s,
                               (a[:, 0, 2] - a[:, 2, 0]) / s, (a[:, 1, 0] - a[:, 0, 1]) / s], 1)
        elif c == 1:
            s = np.sqrt(1.0 + a[:, 0, 0] - a[:, 1, 1] - a[:, 2, 2]) * 2
            q[sel] = np.stack([(a[:, 2, 1] - a[:, 1, 2]) / s, 0.25 * s,
                               (a[:, 0, 1] + a[:, 1, 0]) / s, (a[:, 0, 2] + a[:, 2, 0]) / s], 1)
        elif c == 2:
            s = np.sqrt(1.0 + a[:, 1, 1] - a[:, 0, 0] - a[:, 2, 2]) * 2
            q[sel] = np.stack([(a[:, 0, 2] - a[:, 2, 0]) / s, (a[:, 0, 1] + a[:, 1, 0]) / s,
                               0.25 * s, (a[:, 1, 2] + a[:, 2, 1]) / s], 1)
        else:
            s = np.sqrt(1.0 + a[:, 2, 2] - a[:, 0, 0] - a[:, 1, 1]) * 2
            q[sel] = np.stack([(a[:, 1, 0] - a[:, 0, 1]) / s, (a[:, 0, 2] + a[:, 2, 0]) / s,
                               (a[:, 1, 2] + a[:, 2, 1]) / s, 0.25 * s], 1)
    return q


def _tangent_frames(normals: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    """Orthonormal frames [k,3,3] with columns (t1, t2, normal), random in-plane angle."""
    nrm = normals / np.linalg.norm(normals, axis=1, keepdims=True)
    helper = np.where(np.abs(nrm[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]), np.array([[1.0, 0.0, 0.0]]))
    t1 = np.cross(helper, nrm)
    t1 /= np.linalg.norm(t1, axis=1, keepdims=True)
    t2 = np.cross(nrm, t1)
    ang = rng.uniform(0, 2 * np.pi, size=(len(nrm), 1))
    a1 = np.cos(ang) * t1 + np.sin(ang) * t2
    a2 = -np.sin(ang) * t1 + np.cos(ang) * t2
    return np.stack([a1, a2, nrm], axis=2)


def _logit(o: np.ndarray) -> np.ndarray:
    return np.log(o) - np.log1p(-o)


def surface_scene(n: int, seed: int) -> np.ndarray:
    """Surface-like scene of SURVEY §8(d1): 35% background sphere r=6, 25% ground disk z=-1 r=5,
    40% on 20 object spheres; flat Gaussians tangent to the surface."""
    rng = _rng(seed)
    n_bg = int(round(0.35 * n))
    n_gd = int(round(0.25 * n))
    n_ob = n - n_bg - n_gd
    # background sphere
    v = rng.normal(size=(n_bg, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    p_bg, nrm_bg = 6.0 * v, v
    area_bg = 4 * np.pi * 36.0
    # ground disk at z = -1
    r = 5.0 * np.sqrt(rng.uniform(size=n_gd))
    th = rng.uniform(0, 2 * np.pi, size=n_gd)
    p_gd = np.stack([r * np.cos(th), r * np.sin(th), -np.ones(n_gd)], 1)
    nrm_gd = np.tile([0.0, 0.0, 1.0], (n_gd, 1))
    area_gd = np.pi * 25.0
    # object spheres
    centres = np.concatenate([rng.uniform(-1.5, 1.5, size=(20, 2)), rng.uniform(-0.8, 0.8, size=(20, 1))], 1)
    radii = rng.uniform(0.2, 0.8, size=20)
    which = rng.integers(0, 20, size=n_ob)
    v = rng.normal(size=(n_ob, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    p_ob = centres[which] + radii[which, None] * v
    nrm_ob = v
    area_ob = float(np.sum(4 * np.pi * radii**2))

    pos = np.concatenate([p_bg, p_gd, p_ob])
    nrm = np.concatenate([nrm_bg, nrm_gd, nrm_ob])
    st_base = np.concatenate([
        np.full(n_bg, 0.6 * math.sqrt(area_bg / max(n_bg, 1))),
        np.full(n_gd, 0.6 * math.sqrt(area_gd / max(n_gd, 1))),
        np.full(n_ob, 0.6 * math.sqrt(area_ob / max(n_ob, 1))),
    ])
    s1 = st_base * np.exp(0.5 * rng.normal(size=n))
    s2 = s1 * np.exp(0.3 * rng.normal(size=n))
    s3 = 0.1 * s1
    frames = _tangent_frames(nrm, rng)
    quat = _frame_to_quat(frames)
    perm = rng.permutation(n)  # interleave the three populations in index order
    params = np.empty((N_PLANES, n), dtype=np.float64)
    params[0:3] = pos[perm].T
    params[3:6] = np.log(np.stack([s1, s2, s3], 1)[perm]).T
    params[6:10] = quat[perm].T
    params[10] = _logit(rng.uniform(0.05, 0.95, size=n))
    params[11:14] = rng.uniform(0, 1, size=(3, n))
    return params.astype(np.float32)


def blob_scene(n: int, seed: int, scale: float = 0.22) -> np.ndarray:
    """C1 tiny scene: Gaussians in a unit box around the origin with a few-pixel footprint."""
    rng = _rng(seed)
    params = np.empty((N_PLANES, n), dtype=np.float64)
    params[0:3] = rng.uniform(-1.0, 1.0, size=(3, n))
    params[3:6] = np.log(scale) + 0.35 * rng.normal(size=(3, n))
    q = rng.normal(size=(4, n))
    q *= rng.uniform(0.7, 1.3, size=(1, n)) / np.linalg.norm(q, axis=0, keepdims=True)  # not unit
    params[6:10] = q
    params[10] = _logit(rng.uniform(0.05, 0.95, size=n))
    params[11:14] = rng.uniform(0, 1, size=(3, n))
    return params.astype(np.float32)


def look_at(eye, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)):
    eye = np.asarray(eye, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - eye
    f /= np.linalg.norm(f)
    right = np.cross(f, np.asarray(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    down = np.cross(f, right)
    R = np.stack([right, down, f])  # rows: camera x (right), y (down), z (forward)
    t = -R @ eye
    return R, t


def ring_cameras(views: int, width: int, height: int, seed: int, model: int = 0, radius: float = 4.0,
                 height_base: float = 0.3, focal: float = 0.9, znear: float = 0.2, guard: float = 1.3,
                 affine_depth: float = 4.0):
    """Ring of cameras looking at the origin.  For model=1 (affine) the same pose
    is used and the intrinsics are scaled by 1/affine_depth so image sizes stay comparable."""
    rng = _rng(seed)
    cams = []
    for v in range(views):
        ang = 2 * np.pi * v / views + rng.uniform(-0.05, 0.05)
        h = height_base + rng.uniform(-0.3, 0.3)
        R, t = look_at((radius * np.cos(ang), radius * np.sin(ang), h))
        fx = fy = focal * width
        if model == 1:
            fx = fy = focal * width / affine_depth
        cams.append(dict(R=R.astype(np.float32), t=t.astype(np.float32), fx=np.float32(fx),
                         fy=np.float32(fy), cx=np.float32(width / 2), cy=np.float32(height / 2),
                         width=int(width), height=int(height), model=int(model),
                         znear=np.float32(znear), guard=np.float32(guard)))
    return cams


def target_images(views: int, width: int, height: int, seed: int) -> np.ndarray:
    """Procedural smooth colour fields in [0,1], [V][3][H][W] float32 (no renderer involved)."""
    rng = _rng(seed)
    yy, xx = np.meshgrid(np.arange(height) / max(height, 1), np.arange(width) / max(width, 1), indexing="ij")
    out = np.empty((views, 3, height, width), dtype=np.float32)
    for v in range(views):
        for c in range(3):
            img = np.full((height, width), 0.5)
            for _ in range(6):
                kx, ky = rng.uniform(-12, 12, size=2)
                ph = rng.uniform(0, 2 * np.pi)
                img += rng.uniform(0.05, 0.2) * np.sin(2 * np.pi * (kx * xx + ky * yy) / 4 + ph)
            img += 0.03 * rng.normal(size=img.shape)
            out[v, c] = np.clip(img, 0.0, 1.0)
    return out


def dl_dimage(views: int, width: int, height: int, seed: int) -> np.ndarray:
    """A loss-agnostic dL/dimage input: +-1/(3HW) with random signs and a few exact zeros."""
    rng = _rng(seed)
    s = rng.choice(np.array([-1.0, 0.0, 1.0]), p=[0.48, 0.04, 0.48], size=(views, 3, height, width))
    return (s / (3.0 * width * height)).astype(np.float32)


def scene_for(cfg: Config, seed: int | None = None) -> np.ndarray:
    idx = int(cfg.name[1:])
    seed = 1000 + idx if seed is None else seed
    if cfg.kind == "blobs":
        return blob_scene(cfg.n, seed)
    return surface_scene(cfg.n, seed)


def cameras_for(cfg: Config, views: int | None = None, seed: int | None = None, model: int = 0):
    idx = int(cfg.name[1:])
    seed = 1001 + idx if seed is None else seed
    return ring_cameras(cfg.views if views is None else views, cfg.width, cfg.height, seed, model=model)


def targets_for(cfg: Config, views: int | None = None, seed: int | None = None) -> np.ndarray:
    idx = int(cfg.name[1:])
    seed = 1002 + idx if seed is None else seed
    return target_images(cfg.views if views is None else views, cfg.width, cfg.height, seed)


def splitting_matrices(n: int, seed: int, neg_frac: float = 0.3, scale: float = 1e-3) -> np.ndarray:
    """Random symmetric 3x3 matrices as 6 planes [6][n] (xx,xy,xz,yy,yz,zz), float32, with
    roughly `neg_frac` of them indefinite (an input for densify-only tests)."""
    rng = _rng(seed)
    a = rng.normal(size=(n, 3, 3)) * scale
    a = 0.5 * (a + a.transpose(0, 2, 1))
    shift = np.where(rng.uniform(size=n) < neg_frac, 0.0, 3.0 * scale)
    a += shift[:, None, None] * np.eye(3)
    planes = np.stack([a[:, 0, 0], a[:, 0, 1], a[:, 0, 2], a[:, 1, 1], a[:, 1, 2], a[:, 2, 2]])
    return planes.astype(np.float32)


def sh_coefficients(n: int, degree: int, seed: int, scale: float = 0.1) -> np.ndarray:
    """Seeded SH rest coefficients [3 ((degree + 1)^2 - 1)][n] float32 (f3 workloads): N(0, scale^2)."""
    K = (degree + 1) ** 2
    return (_rng(seed).normal(size=(3 * (K - 1), n)) * scale).astype(np.float32)
