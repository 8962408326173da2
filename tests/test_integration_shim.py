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
import os
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


REF_INSTALLED = ROOT / "baseline" / "_ref"  # pip --target install of the reference (git-ignored, travels)


def _ref_path():
    """The reference package on this machine: the build container's source
    tree, else the installed copy that travels to the GPU box."""
    if REF_SRC.exists():
        return REF_SRC
    return REF_INSTALLED if (REF_INSTALLED / "bitsdf").exists() else None


@pytest.mark.skipif(_ref_path() is None, reason="reference package not present")
def test_plugin_rebinds_reference_names():
    """integration/pytest_b200.py (the plugin that runs the reference's own
    suites against the drop-in): after install() every bitsdf module's
    integrate_frame / integrate_point / extract_mesh is the plugin's, the
    shim sits at bitsdf._b200, and the CPU originals stay reachable."""
    code = f"""
import sys
sys.path.insert(0, {str(_ref_path())!r}); sys.path.insert(0, {str(ROOT / "integration")!r})
import os
os.environ["BITSDF_B200_LIB"] = {str(_native.LIB_PATH)!r}
import bitsdf.integrator as ri, bitsdf.mesher as rm
cpu = (ri.integrate_frame, ri.integrate_point, rm.extract_mesh)
import pytest_b200 as P
shim = P.install()
import bitsdf, bitsdf.cli as cli
assert bitsdf._b200 is shim and sys.modules["bitsdf._b200"] is shim
for mod in (bitsdf, ri, cli):
    assert mod.integrate_frame.__module__ == "pytest_b200", mod
assert ri.integrate_point.__module__ == "pytest_b200"
assert rm.extract_mesh.__module__ == "pytest_b200" and cli.extract_mesh is rm.extract_mesh
assert tuple(bitsdf._b200_cpu[k] for k in ("integrate_frame", "integrate_point", "extract_mesh")) == cpu
assert shim.FrameStats is ri.FrameStats
print("ok")
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.stdout.strip().endswith("ok"), out.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not (REF_INSTALLED / "bitsdf").exists(), reason="baseline/_ref (installed reference) not present")
def test_live_reference_crosscheck(tmp_path):
    """The reference itself, imported on the GPU box from baseline/_ref, as a
    live oracle: a short trajectory through the plugin with
    BITSDF_B200_CROSSCHECK=1 — every integrate_frame / integrate_point /
    extract_mesh call is repeated by the reference's CPU code on a copy of the
    grid and compared array for array, FrameStats included (exact
    voxels_written)."""
    t = tmp_path / "test_live.py"
    t.write_text("""
import numpy as np
from bitsdf.grid import new_grid
from bitsdf.integrator import IntegrationParams, ScanFrame, integrate_frame, integrate_point
from bitsdf.kernels import build_kernel_bank
from bitsdf.mesher import extract_mesh

def test_trajectory():
    rng = np.random.default_rng(11)
    grid = new_grid((72, 64, 56), 0.1)
    bank = build_kernel_bank(shadow_radius=2)
    for k, prm in enumerate([IntegrationParams(t_occ=1), IntegrationParams(t_occ=2, first_return_per_voxel=True),
                             IntegrationParams(t_occ=2, downsample=3), IntegrationParams(t_occ=1)]):
        pose = np.eye(4); pose[:3, 3] = (3.0 + 0.3 * k, 3.2, 2.8)
        d = rng.normal(size=(3000, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
        pts = d * rng.uniform(0.05, 4.5, size=(3000, 1))
        dt = np.float32 if k % 2 else np.float64
        st = integrate_frame(grid, bank, ScanFrame(points=pts.astype(dt), pose=pose), prm)
        assert st.points_in > 0
    assert integrate_point(grid, bank, (2.0, 2.0, 2.0), (3.0, 3.0, 3.0), IntegrationParams(t_occ=1)) == "applied"
    assert len(extract_mesh(grid).triangles) > 0
""")
    env = dict(os.environ, PYTHONPATH=f"{REF_INSTALLED}:{ROOT / 'integration'}", BITSDF_B200_LIB=str(_native.LIB_PATH),
               BITSDF_B200_CROSSCHECK="1", DBT_EXACT_VOXELS_WRITTEN="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-p", "pytest_b200", "--rootdir", str(tmp_path), "-c",
                          "/dev/null", "-p", "no:cacheprovider", "-q", str(t)], capture_output=True, text=True, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "crosschecked 6" in out.stdout, out.stdout[-1500:]


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
