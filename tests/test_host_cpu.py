"""CPU-only checks of the boundary and host logic: the C-ABI library loads and exports every symbol
include/steepgs.h declares (no compute calls without a GPU), struct layouts match, the oracle and
the product share no code, and the multi-rank (gloo, world_size 2) view-sharded reduction."""
import ctypes
import os
import re
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "steepgs.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(steepgs_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libsteepgs():
    from paper_2505_05587_b200 import build as B
    B.build()
    return ctypes.CDLL(B.LIB)


def test_library_exports_every_declared_symbol(libsteepgs):
    syms = header_symbols()
    assert len(syms) >= 14
    missing = [s for s in syms if not hasattr(libsteepgs, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_2505_05587_b200", "libsteepgs.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (steepgs_\w+)", out))
    assert set(syms) <= exported


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2505_05587_b200", "libsteepgs.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_only_entry_points(libsteepgs):
    from paper_2505_05587_b200 import _lib
    assert ctypes.sizeof(_lib.Camera) == 84 and ctypes.sizeof(_lib.RasterParams) == 32
    # the ctypes mirrors must match the C layouts of include/steepgs.h (checked with the C compiler)
    src = ('#include <stdio.h>\n#include "steepgs.h"\nint main(void){printf("%zu %zu %zu %zu %zu %zu\\n",'
           'sizeof(steepgs_camera), sizeof(steepgs_raster_params), sizeof(steepgs_densify_params),'
           'sizeof(steepgs_binning), sizeof(steepgs_splat), sizeof(steepgs_adam_params));return 0;}')
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "s.c"), "w").write(src)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", os.path.join(d, "s"), os.path.join(d, "s.c")])
        sizes = [int(x) for x in subprocess.check_output([os.path.join(d, "s")]).split()]
    assert sizes == [ctypes.sizeof(_lib.Camera), ctypes.sizeof(_lib.RasterParams), ctypes.sizeof(_lib.DensifyParams),
                     ctypes.sizeof(_lib.Binning), _lib.SPLAT_BYTES, ctypes.sizeof(_lib.AdamParams)]
    # field offsets of the binning struct too (the render calls read fields the forward / backward share)
    fields = [f for f, _ in _lib.Binning._fields_]
    src2 = ('#include <stdio.h>\n#include <stddef.h>\n#include "steepgs.h"\nint main(void){'
            + "".join(f'printf("%zu ", offsetof(steepgs_binning, {f}));' for f in fields) + "return 0;}")
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "o.c"), "w").write(src2)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", os.path.join(d, "o"), os.path.join(d, "o.c")])
        offs = [int(x) for x in subprocess.check_output([os.path.join(d, "o")]).split()]
    assert offs == [getattr(_lib.Binning, f).offset for f in fields]
    assert _lib.version().startswith("steepgs-b200")
    assert _lib.bin_sort_workspace_size(1000, 2, 64, 48, 10000) > 0
    assert _lib.densify_workspace_size(5000) >= 8
    libsteepgs.steepgs_status_string.restype = ctypes.c_char_p
    assert libsteepgs.steepgs_status_string(3) == b"capacity exceeded"
    with pytest.raises(_lib.SteepGSError):
        _lib.bin_sort_workspace_size(-1, 2, 64, 48, 10)


def test_no_cpu_fallback_without_device():
    """On a box without a compute-capability-10.x device the product refuses to run."""
    import torch
    if torch.cuda.is_available() and torch.cuda.get_device_capability()[0] == 10:
        pytest.skip("a B200 is present")
    from paper_2505_05587_b200.pipeline import Rasterizer
    with pytest.raises(RuntimeError):
        Rasterizer(16, 1, 16, 16)


def test_oracle_and_product_share_no_code():
    prod = [os.path.join(ROOT, "paper_2505_05587_b200", f) for f in os.listdir(os.path.join(ROOT, "paper_2505_05587_b200"))
            if f.endswith(".py")]
    prod += [os.path.join(ROOT, "paper_2505_05587_b200", "csrc", f)
             for f in os.listdir(os.path.join(ROOT, "paper_2505_05587_b200", "csrc"))]
    prod.append(os.path.join(ROOT, "include", "steepgs.h"))
    for f in prod:
        txt = open(f).read()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
        assert "oracle.h" not in txt and "liboracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".h", ".py")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r'#include\s*[<"][^>"]*steepgs\.h', txt), f
            assert not re.search(r"^\s*(import|from)\s+paper_2505_05587_b200", txt, re.M), f
    # the shared input generator holds no method arithmetic (no projection / compositing / eigen)
    syn = open(os.path.join(ROOT, "synth", "__init__.py")).read()
    for word in ("conic", "alpha_blend", "eigvalsh", "sigmoid(", "import oracle", "paper_2505_05587_b200"):
        assert word not in syn


def test_shard_views_partition():
    from paper_2505_05587_b200.parallel import shard_views
    for V in (1, 7, 64):
        for R in (1, 2, 3, 8):
            got = sorted(v for r in range(R) for v in shard_views(V, r, R))
            assert got == list(range(V))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import oracle, synth
from paper_2505_05587_b200.parallel import shard_views, allreduce_accumulators
rank, world = int(sys.argv[1]), int(sys.argv[2])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=world)
cfg = synth.CONFIGS["C1"]
p = synth.scene_for(cfg); cams = synth.cameras_for(cfg, views=5)
dl = synth.dl_dimage(5, 64, 64, 9)
cap = p.shape[1] + 8
acc = torch.zeros(20, cap, dtype=torch.float64)
for v in shard_views(5, rank, world):
    acc[:, :p.shape[1]] += torch.from_numpy(oracle.render(p, cams[v], dl_dimage=dl[v])["grad"])
allreduce_accumulators(acc, n=p.shape[1])
full = sum(oracle.render(p, cams[v], dl_dimage=dl[v])["grad"] for v in range(5))
assert np.allclose(acc[:, :p.shape[1]].numpy(), full, rtol=1e-12, atol=1e-18), "allreduce mismatch"
assert float(acc[:, p.shape[1]:].abs().max()) == 0.0
dist.destroy_process_group()
print("ok", rank)
'''


def test_gloo_two_rank_view_sharded_allreduce(orc):
    port = _free_port()
    code = WORKER.format(root=ROOT, port=port)
    env = dict(os.environ, OMP_NUM_THREADS="1")
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r), "2"], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True, env=env) for r in range(2)]
    outs = [p.communicate(timeout=180) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
        assert o.startswith("ok")


def test_bench_reference_arm_runs_on_cpu():
    """`bench.py --impl reference` (the CPU oracle arm) prints one JSON line with the contract keys."""
    import json
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "ms/view" and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0


def test_schedule_densify_until_and_exclusive_gates():
    """Schedule.t_stop (3DGS's densify_until_iter): no densify step and no window restart after it;
    densify_params rejects the compactest gate together with the C24 gate."""
    from paper_2505_05587_b200 import _lib
    from paper_2505_05587_b200.pipeline import Schedule
    s = Schedule(t_start=5, t_split=3, t_stop=20)
    assert [t for t in range(1, 40) if s.densify_at(t)] == [5, 8, 11, 14, 17, 20]
    assert [t for t in range(1, 40) if s.window_restarts_after(t)] == [2, 5, 8, 11, 14, 17, 20]
    assert Schedule().t_stop == 15000 and not Schedule(t_start=500, t_split=100).densify_at(15100)
    assert Schedule(t_start=500, t_split=100, t_stop=None).densify_at(15100)
    with pytest.raises(ValueError):
        _lib.densify_params(eps_grad=1e-3, grad_gate=1e-4)


def test_bench_gpus_flag_never_times_fewer_ranks():
    """`python bench.py --gpus 2` without torchrun launches 2 ranks itself, and fails loudly (non-zero,
    nothing printed on stdout) when the node has fewer devices; a WORLD_SIZE that disagrees with
    --gpus is an error too."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, env={k: v for k, v in os.environ.items()
                                                                         if k not in ("WORLD_SIZE", "RANK")})
    import torch
    if torch.cuda.device_count() < 2:
        assert r.returncode == 3 and "CUDA device" in r.stderr and r.stdout.strip() == ""
    env = dict(os.environ, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--steps", "0", "--warmup", "0"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr and r.stdout.strip() == ""


def test_fused_reduce_owner_ranges():
    """steepgs_scatter_chunk (host-only C-ABI call): the R owner ranges [q chunk, (q + 1) chunk) ∩ [0, n)
    of the fused reduce-scatter cover [0, n) once, start on 32-column boundaries, and only the last
    owner can be short or empty (tests/test_fused_collective.py runs the kernels)."""
    from paper_2505_05587_b200 import _lib
    for n in (0, 1, 31, 32, 3001, 1_000_000, 6_000_001):
        for R in range(1, 9):
            c = _lib.scatter_chunk(n, R)
            assert c % 32 == 0 and c * R >= n and (n == 0 or c - 32 < -(-n // R))
            covered = sum(max(0, min(n, (q + 1) * c) - q * c) for q in range(R))
            assert covered == n
    with pytest.raises(_lib.SteepGSError):
        _lib.scatter_chunk(10, 9)                    # more ranks than one NVSwitch domain's peer set
