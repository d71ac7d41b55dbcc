"""GPU edge cases through the C ABI: instance-capacity overflow, degenerate / NaN parameters, negative
affine depths, the maximum view batch, huge footprints, and argument validation."""
import numpy as np
import pytest

import synth
from helpers import affine_cam, params_from

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEFAULT = dict(alpha_min=1.0 / 255.0, alpha_max=0.99, t_min=1e-4, dilation=0.3, bg=(0.0, 0.0, 0.0), tile=16)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_instance_overflow_is_flagged_and_memory_safe():
    from gpu_run import run_forward
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=2)
    rz, _ = run_forward(p, cams, DEFAULT, max_instances=16)
    b = rz.binning_arrays()
    assert b["overflow"] == 1 and b["n_instances"] > 16
    assert b["ids"].numel() == 16
    assert int(((b["ranges"][:, 1] - b["ranges"][:, 0]) >= 0).all()) == 1
    assert torch.isfinite(rz.image).all()


def test_degenerate_and_nan_parameters_are_culled(orc):
    from gpu_run import decisions, run_forward
    n = 12
    p = params_from(np.random.default_rng(0).uniform(-0.5, 0.5, size=(n, 3)), [0.2, 0.2, 0.2])
    p[6:10, 0] = 0.0                  # zero quaternion
    p[0, 1] = np.nan                  # NaN mean
    p[3:6, 2] = -80.0                 # vanishing scales: covariance = dilation only
    p[10, 3] = -40.0                  # opacity ~ 0 < alpha_min
    p[3:6, 4] = np.inf                # infinite scale
    cams = synth.ring_cameras(1, 64, 48, 3)
    rz, _ = run_forward(p, cams, DEFAULT)
    g = decisions(rz, n)
    d = orc.decide(p, cams[0], DEFAULT)
    assert np.array_equal(g["tiles_touched"][0] > 0, d["visible"].astype(bool))
    assert np.array_equal(g["tiles_touched"][0][d["visible"] == 1], d["tiles_touched"][d["visible"] == 1])
    assert d["visible"][[0, 1, 3]].sum() == 0
    assert torch.isfinite(rz.image).all()


def test_affine_negative_depth_keys_bitexact(orc):
    """Affine cameras do not cull on z; depth keys of negative z use the sign-flip transform (C7)."""
    from gpu_run import decisions, run_forward
    rng = np.random.default_rng(4)
    n = 200
    p = params_from(np.concatenate([rng.uniform(-3, 3, size=(n, 2)), rng.uniform(-2, 2, size=(n, 1))], 1),
                    np.exp(np.log(0.3) + 0.3 * rng.normal(size=(n, 3))), rng.normal(size=(n, 4)),
                    rng.uniform(0.2, 0.9, size=n), rng.uniform(0, 1, size=(n, 3)))
    cam = affine_cam(48, 40, fx=6.0, cx=24.0, cy=20.0, t=(0.0, 0.0, 0.5))
    rz, _ = run_forward(p, [cam], DEFAULT)
    g = decisions(rz, n)
    d = orc.decide(p, cam, DEFAULT)
    vis = d["visible"].astype(bool)
    assert (np.asarray(p[2], np.float64)[vis] + 0.5 < 0).any()    # some negative depths are visible
    assert np.array_equal(g["key"][0][vis], d["key"][vis])
    # the instance order through the sort: keys on both sides of the sign flip (all four radix passes)
    from test_gpu_parity import expected_binning
    ids, counts = expected_binning([d], 48, 40)
    b = rz.binning_arrays()
    assert b["overflow"] == 0 and b["n_instances"] == ids.size
    assert np.array_equal(b["ids"].numpy().astype(np.int64), ids)
    assert np.array_equal((b["ranges"][:, 1] - b["ranges"][:, 0]).numpy(), counts)
    o = orc.render(p, cam, DEFAULT)
    img = rz.image.cpu().numpy()[0]
    ok = (np.abs(img - o["image"]) <= 1e-4 * np.abs(o["image"]) + 1e-6) | (o["amb_px"][None] != 0)
    assert ok.all()


def test_max_view_batch():
    from gpu_run import run_forward
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=64)
    rz, _ = run_forward(p, cams, DEFAULT)
    img = rz.image.cpu().numpy()
    ref, _ = run_forward(p, cams[37:38], DEFAULT)
    assert np.array_equal(img[37], ref.image.cpu().numpy()[0])    # view batching changes nothing


def test_huge_footprint_covers_every_tile(orc):
    from gpu_run import run_forward
    p = params_from([[0.0, 0.0, 0.0]], [[3.0, 3.0, 3.0]], opac=[0.6], rgb=[[0.3, 0.6, 0.9]])
    cams = synth.ring_cameras(1, 200, 120, 1)
    rz, _ = run_forward(p, cams, DEFAULT)
    b = rz.binning_arrays()
    assert b["n_instances"] == ((200 + 15) // 16) * ((120 + 15) // 16)
    o = orc.render(p, cams[0], DEFAULT)
    img = rz.image.cpu().numpy()[0]
    assert np.allclose(img, o["image"], rtol=1e-4, atol=1e-6)


def test_argument_validation():
    from paper_2505_05587_b200 import _lib
    from paper_2505_05587_b200.pipeline import Raster, Rasterizer
    rz = Rasterizer(64, 1, 64, 64)
    p = torch.zeros(14, 64, device="cuda")
    cams = synth.cameras_for(synth.CONFIGS["C1"], views=1)
    bad = Raster()
    rz.rp = _lib.raster_params(tile=8)
    with pytest.raises(_lib.SteepGSError) as e:
        rz.project(p, 64, cams)
    assert e.value.status == 1
    rz.rp = bad.c()
    with pytest.raises(_lib.SteepGSError):
        _lib.project(p, 10, 64, _lib.cameras(cams), 1, rz.rp, rz.splats, rz.depth_key, rz.tile_rect,
                     rz.tiles_touched)                                       # ld < n
    small = torch.empty(1024, dtype=torch.uint8, device="cuda")
    rz.project(p, 64, cams)
    with pytest.raises(_lib.SteepGSError) as e:
        _lib.bin_sort(rz.depth_key, rz.tile_rect, rz.tiles_touched, 64, rz.cams_arr, 1, rz.rp, small, 4096)
    assert e.value.status == 2
    with pytest.raises(_lib.SteepGSError):
        Rasterizer(64, 65, 64, 64)                                           # > 64 views
    # a binning without the forward -> backward per-instance masks is rejected before any launch
    rz.bin_sort()
    b = _lib.Binning.from_buffer_copy(rz.binning)
    b.inst_mask = None
    with pytest.raises(_lib.SteepGSError) as e:
        _lib.render_fwd(rz.splats, 64, b, rz.cams_arr, 1, rz.rp, rz.image, rz.final_T, rz.n_contrib)
    assert e.value.status == 1


def test_instance_overflow_auto_grow():
    """bin_sort(check=True) grows the instance buffers and re-sorts, so the render is the one of a
    generously sized binning."""
    from gpu_run import run_forward, to_dev
    from paper_2505_05587_b200.pipeline import Raster, Rasterizer
    cfg = synth.CONFIGS["C1"]
    p = synth.scene_for(cfg)
    cams = synth.cameras_for(cfg, views=2)
    ref, _ = run_forward(p, cams, DEFAULT)
    rz = Rasterizer(p.shape[1], 2, 64, 64, Raster(), max_instances=16)
    rz.project(to_dev(p), p.shape[1], cams)
    rz.bin_sort(check=True)
    rz.render_fwd()
    b = rz.binning_arrays()
    assert b["overflow"] == 0 and rz.max_instances >= b["n_instances"] > 16
    assert torch.equal(rz.image, ref.image)


def test_backward_rejects_stale_binning():
    """STEEPGS_ERR_STALE_STATE: render_bwd refuses a binning that was not rendered
    forward since its bin_sort, or whose forward used other splats / cameras / raster params;
    nothing is launched and the moments stay zero."""
    from gpu_run import to_dev
    from paper_2505_05587_b200 import _lib
    from paper_2505_05587_b200.pipeline import Raster, Rasterizer
    cfg = synth.CONFIGS["C1"]
    p = to_dev(synth.scene_for(cfg))
    cams = synth.cameras_for(cfg, views=1)
    dl = to_dev(synth.dl_dimage(1, 64, 64, 3))
    rz = Rasterizer(64, 1, 64, 64)
    rz.project(p, 64, cams)
    rz.bin_sort()

    def bwd(rp=None, cams_arr=None, splats=None):
        _lib.render_bwd_moments(rz.splats if splats is None else splats, 64, rz.binning,
                                rz.cams_arr if cams_arr is None else cams_arr, 1, rz.rp if rp is None else rp,
                                rz.final_T, rz.n_contrib, dl, rz.moments)

    for case in ("no forward", "re-sorted", "other raster", "other camera", "other splats"):
        if case == "re-sorted":
            rz.render_fwd()
            rz.bin_sort()
        elif case != "no forward":
            rz.render_fwd()
        kw = {}
        if case == "other raster":
            kw["rp"] = Raster(alpha_min=0.01).c()
        elif case == "other camera":
            kw["cams_arr"] = _lib.cameras(synth.cameras_for(cfg, views=1, seed=99))
        elif case == "other splats":
            kw["splats"] = rz.splats[64:]
        with pytest.raises(_lib.SteepGSError) as e:
            bwd(**kw)
        assert e.value.status == 4, case
    rz.render_fwd()
    bwd()                                                                   # the matching forward: accepted
    torch.cuda.synchronize()
    assert float(rz.moments.abs().sum()) > 0


def test_tile_order_many_tiles():
    """binning.tile_order when V * tiles exceeds the order kernel's register-cached path (24,576
    tiles: here C5's 8160 tiles x 4 views): a permutation of (view << 20 | tile) with list lengths
    non-increasing in half-octave buckets."""
    from gpu_run import run_forward
    cfg = synth.CONFIGS["C5"]
    p = synth.scene_for(cfg)[:, :200_000]
    cams = synth.cameras_for(cfg, views=4)
    rz, _ = run_forward(np.ascontiguousarray(p), cams, DEFAULT)
    b = rz.binning_arrays()
    t = b["tile_order"].numpy().astype(np.int64)
    counts = (b["ranges"][:, 1] - b["ranges"][:, 0]).numpy().astype(np.int64)
    tpv = counts.size // 4
    assert counts.size > 24576
    flat = (t >> 20) * tpv + (t & 0xFFFFF)
    assert ((t & 0xFFFFF) < tpv).all() and np.array_equal(np.sort(flat), np.arange(counts.size))
    L = counts[flat]
    nz = L > 0
    c = np.where(nz, 31 - np.floor(np.log2(np.maximum(L, 1))).astype(np.int64), 32)
    nb = np.where(nz & (c < 31), (L >> np.maximum(30 - c, 0)) & 1, 0)
    key = np.where(nz, 2 * c + 1 - nb, 64)
    assert (np.diff(key) >= 0).all() and nz.sum() > 0
    assert torch.isfinite(rz.image).all()
