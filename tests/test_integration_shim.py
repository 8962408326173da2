"""The reference-side binding (integration/bitsdf_b200.py):
the file a maintainer drops into the reference as bitsdf/_b200.py.

CPU: every ctypes struct of the shim (and of the package's own mirror) has the
header's size and field offsets (a C program compiled against
include/dbtsdf.h prints them); the shim loads libdbtsdf.so and binds every
symbol it declares; with /root/reference present (build container) the shim,
placed inside a copy of the reference package, resolves the reference's own
FrameStats / errors / motion_compensate and converts the reference's
KernelBank / VoxelGrid objects exactly as the package does.
GPU: the shim runs end to end on VoxelGrid-shaped stand-ins (plain numpy
arrays, as the reference's dataclass holds them) and reproduces the
reference's golden grids, FrameStats counts, integrate_point outcomes and
meshes.
"""

import ctypes
import importlib
import json
import shutil
import subprocess
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

import cases
from paper_2509_20081_b200 import _native, build_kernel_bank

ROOT = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "integration"))
shim = importlib.import_module("bitsdf_b200")


@pytest.fixture(scope="module")
def layout(tmp_path_factory):
    exe = tmp_path_factory.mktemp("abi") / "abi_layout"
    subprocess.run(["gcc", "-std=c99", "-O0", str(ROOT / "tests" / "native" / "abi_layout.c"), "-o", str(exe)],
                   check=True)
    return json.loads(subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout)


@pytest.mark.parametrize("pair", [("dbt_params", shim.Params), ("dbt_stats", shim.Stats),
                                  ("dbt_mc_tables", shim.McTables), ("dbt_params", _native.Params),
                                  ("dbt_stats", _native.Stats), ("dbt_deskew", shim.Deskew),
                                  ("dbt_deskew", _native.Deskew)], ids=lambda p: f"{p[1].__module__}.{p[0]}")
def test_ctypes_structs_match_header(layout, pair):
    cname, cls = pair
    assert ctypes.sizeof(cls) == layout[cname]
    for f, _ in cls._fields_:
        off, size = layout[f"{cname}.{f}"]
        assert getattr(cls, f).offset == off, f
        assert getattr(cls, f).size == size, f
    assert len(cls._fields_) == sum(1 for k in layout if k.startswith(cname + "."))


def test_shim_binds_every_symbol_it_uses():
    L = shim.lib(str(_native.LIB_PATH))
    src = (ROOT / "integration" / "bitsdf_b200.py").read_text()
    used = set(__import__("re").findall(r"lib\(\)\.(dbt_\w+)", src))
    assert used
    for name in used:
        assert hasattr(L, name) and getattr(L, name).argtypes is not None or name == "dbt_last_error", name


def test_shim_bank_tables_match_package():
    bank = build_kernel_bank(shadow_radius=2)
    dk, xyz, cnt = shim.bank_tables(bank)
    assert dk.dtype == np.uint32 and dk.shape == (21, 21, 21)
    assert xyz.dtype == np.int32 and xyz.shape == (int(cnt.sum()), 3)
    assert np.array_equal(np.concatenate(bank.shadow_offsets), xyz)


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference not present (GPU box)")
def test_shim_inside_reference_package(tmp_path):
    """Drop the shim into a copy of the reference package as bitsdf/_b200.py:
    its relative imports resolve to the reference's own types, and it accepts
    the reference's VoxelGrid / KernelBank objects."""
    pkg = tmp_path / "bitsdf"
    shutil.copytree(REF_SRC / "bitsdf", pkg)
    shutil.copy(ROOT / "integration" / "bitsdf_b200.py", pkg / "_b200.py")
    code = f"""
import sys, numpy as np
sys.path.insert(0, {str(tmp_path)!r})
sys.path.insert(1, {str(ROOT)!r})
import bitsdf, bitsdf._b200 as b
from bitsdf import errors, integrator, grid as G, kernels as K
assert b.FrameStats is integrator.FrameStats and b._errors is errors
assert b.motion_compensate is integrator.motion_compensate
rb = K.build_kernel_bank(shadow_radius=3)
from paper_2509_20081_b200 import build_kernel_bank
ob = build_kernel_bank(shadow_radius=3)
for x, y in zip(b.bank_tables(rb), b.bank_tables(ob)):
    assert x.dtype == y.dtype and np.array_equal(x, y)
g = G.new_grid((30, 31, 32), 0.1)
m, s, h = b._fields(g)
assert m is g.mask and s is g.sign and h is g.hits
from bitsdf import _mc_tables as T
t = b.mc_tables()
assert list(t.edge_table) == [int(v) for v in T.EDGE_TABLE]
print("ok")
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.stdout.strip().endswith("ok"), out.stderr


# ------------------------------------------------------------------ GPU
def _standin(c):
    """A VoxelGrid-shaped object: what the reference's dataclass holds."""
    shp = tuple(c.dims)
    g = SimpleNamespace(dims=shp, voxel_size=c.voxel_size, origin=np.asarray(c.origin, np.float64),
                        mask=np.full(shp, 0xFFFFFFFF, np.uint32), sign=np.ones(shp, np.uint8),
                        hits=np.zeros(shp, np.uint8), h_max=255, t_occ=2)
    if c.init is not None:
        g.mask[...], g.sign[...], g.hits[...] = c.init
    return g


def _params(d):
    return SimpleNamespace(h_max=d.get("h_max", 255), t_occ=d.get("t_occ", 2), compensation="none",
                           downsample=d.get("downsample", 1),
                           first_return_per_voxel=d.get("first_return_per_voxel", False))


SHIM_CASES = ["frame500_default", "frame500_first_return", "frame500_downsample3", "yaw_frames_f32",
              "nonfresh_hemisphere_h7_t3", "arbitrary_state", "edge_returns", "empty_scan", "cfg2_scans0-2"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", SHIM_CASES)
def test_shim_integrate_frame_matches_reference(name, golden):
    shim.lib(str(_native.LIB_PATH))
    c = next(x for x in cases.small_cases() + cases.config_cases(include_slow=False) if x.name == name)
    g = _standin(c)
    bank = build_kernel_bank(**c.bank)
    prm = _params(c.params)
    ref = golden["cases"][name]
    for (pts, pose), want in zip(c.frames, ref["stats"]):
        scan = SimpleNamespace(points=np.asarray(pts, np.float64).reshape(-1, 3), pose=pose, timestamps=None,
                               prev_pose=None)
        st = shim.integrate_frame(g, bank, scan, prm)
        assert [st.points_in, st.points_discarded] == want[:2]
    assert cases.sha(g.mask) == ref["mask"]
    assert cases.sha(g.sign) == ref["sign"]
    assert cases.sha(g.hits) == ref["hits"]


@pytest.mark.gpu
def test_shim_integrate_point_matches_reference(golden):
    shim.lib(str(_native.LIB_PATH))
    c = next(x for x in cases.small_cases() if x.name == "c1_points10k")
    g = _standin(c)
    bank = build_kernel_bank(**c.bank)
    prm = _params(c.params)
    shim.keep_on_device(g)  # one upload; 10 000 calls without grid transfers
    applied = sum(shim.integrate_point(g, bank, p, s, prm) == "applied" for p, s in zip(*c.hits))
    shim.sync_to_host(g)
    ref = golden["cases"][c.name]
    assert applied == ref["applied"]
    assert (cases.sha(g.mask), cases.sha(g.sign), cases.sha(g.hits)) == (ref["mask"], ref["sign"], ref["hits"])


@pytest.mark.gpu
def test_shim_extract_mesh_matches_reference(golden):
    shim.lib(str(_native.LIB_PATH))
    tables = dict(np.load(ROOT / "tests" / "golden" / "mc_tables.npz"))
    c = next(x for x in cases.small_cases() if x.name == "frame500_default")
    g = _standin(c)
    bank = build_kernel_bank(**c.bank)
    for pts, pose in c.frames:
        shim.integrate_frame(g, bank, SimpleNamespace(points=np.asarray(pts, np.float64), pose=pose,
                                                      timestamps=None, prev_pose=None), _params(c.params))
    for iso, ref in golden["cases"][c.name]["mesh"].items():
        v, f = shim.extract_mesh(g, float(iso), tables)
        assert cases.sha(np.ascontiguousarray(v, np.float64)) == ref["vertices"]
        assert cases.sha(np.ascontiguousarray(f, np.int64)) == ref["triangles"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["deskew_se3_linspace", "deskew_yaw_ts_ds2"])
def test_shim_deskew_matches_reference(name, golden):
    """compensation "se3" / "yaw" through the shim: deskewed on the device."""
    shim.lib(str(_native.LIB_PATH))
    c = next(x for x in cases.deskew_cases() if x.name == name)
    g = _standin(SimpleNamespace(dims=c.dims, voxel_size=c.voxel_size, origin=c.origin, init=None))
    bank = build_kernel_bank(**c.bank)
    prm = _params(c.params)
    prm.compensation = c.params["compensation"]
    ref = golden["deskew"][name]
    for (pts, pose, prev, ts), want in zip(c.frames, ref["stats"]):
        scan = SimpleNamespace(points=np.asarray(pts, np.float64).reshape(-1, 3), pose=pose, timestamps=ts,
                               prev_pose=prev)
        st = shim.integrate_frame(g, bank, scan, prm)
        assert [st.points_in, st.points_discarded] == want[:2]
    assert shim._DESKEW_OK
    assert (cases.sha(g.mask), cases.sha(g.sign), cases.sha(g.hits)) == (ref["mask"], ref["sign"], ref["hits"])
