"""Motion compensation on the device (§8(f)3; reference integrator.py:91-123,
223-230): compensation "se3" / "yaw" deskews every point in the
preprocessing kernel (csrc/deskew.cuh) instead of through scipy on the host.

The reference's result depends on the C library's sin/cos (scipy's Cython
Rotation calls them per point), which are not correctly rounded, so the
device restates glibc's algorithm (csrc/libm_emu.cuh) and reads the library's
own sin/cos table at run time. Checked here:

CPU (the same headers built for the host with -ffp-contract=off):
* the sin/cos restatement equals this process's libm on every branch;
* the per-point deskew reproduces the reference's own motion_compensate
  output (hashes in tests/golden/golden.json "deskew", written by
  make_golden.py --only-deskew from the reference) and the package's host
  port on random sweeps;
* the oracle fed with the host port's deskewed points reproduces the
  reference's final grids.

GPU (-m gpu): dbt_deskew_points equals the reference's points; integrate_frame
/ integrate_frames with compensation reproduce the reference's grids and
point counts bit for bit.
"""

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

import cases
import oracle
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, new_grid
from paper_2509_20081_b200 import _native
from paper_2509_20081_b200.integrator import deskew_params, motion_compensate

ROOT = Path(__file__).resolve().parent.parent
DESKEW = cases.deskew_cases()


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@pytest.fixture(scope="module")
def host(tmp_path_factory):
    d = tmp_path_factory.mktemp("deskew")
    libs = {}
    for name in ("libm_host", "deskew_host"):
        out = d / f"{name}.so"
        subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                        str(ROOT / "tests" / "native" / f"{name}.cpp"), "-o", str(out), "-ldl"], check=True)
        libs[name] = ctypes.CDLL(str(out))
    libs["libm_host"].libm_compare.restype = ctypes.c_long
    libs["deskew_host"].deskew_host.restype = ctypes.c_long
    if not libs["libm_host"].libm_tab_found():
        pytest.skip("the C library's sin/cos table is not found (not glibc's dbl-64 sin/cos)")
    return libs


def _host_deskew(host, d, pts, ts):
    pts = np.ascontiguousarray(pts, np.float64)
    out = np.empty_like(pts)
    tsp = None if ts is None else np.ascontiguousarray(ts, np.float64)
    rare = host["deskew_host"].deskew_host(ctypes.byref(d), _ptr(pts), None if tsp is None else _ptr(tsp),
                                           pts.shape[0], _ptr(out))
    assert rare == 0
    return out


def _downsampled(c, frame):
    pts, pose, prev, ts = frame
    k = slice(None, None, c.params.get("downsample", 1))
    return ScanFrame(points=np.asarray(pts)[k], pose=pose, timestamps=None if ts is None else ts[k], prev_pose=prev)


def test_libm_restatement_matches_c_library(host):
    L = host["libm_host"]
    assert L.libm_check() == 0
    rng = np.random.default_rng(0)
    for lo, hi in [(0, 0.126), (0, 0.86), (0.85, 2.43), (2.4, 4.0), (4.0, 1e4), (-3.3, 3.3)]:
        x = rng.uniform(lo, hi, 400_000)
        s, c = np.empty_like(x), np.empty_like(x)
        assert L.libm_compare(_ptr(x), x.size, _ptr(s), _ptr(c)) == 0, (lo, hi)
    x = np.concatenate([np.ldexp(rng.uniform(0.5, 1, 20000), rng.integers(-40, 0, 20000)), [0.0, -0.0, 1e-300]])
    s, c = np.empty_like(x), np.empty_like(x)
    assert L.libm_compare(_ptr(x), x.size, _ptr(s), _ptr(c)) == 0


@pytest.mark.parametrize("c", DESKEW, ids=lambda c: c.name)
def test_host_deskew_reproduces_reference_points(c, host, golden):
    """The restatement against the reference's own motion_compensate output."""
    ref = golden["deskew"][c.name]
    assert c.input_hash() == ref["input"], "case generator drift"
    for k, fr in enumerate(c.frames):
        sc = _downsampled(c, fr)
        got = _host_deskew(host, deskew_params(sc, c.params["compensation"]), sc.points, sc.timestamps)
        assert cases.sha(got) == ref["points"][k], f"frame {k}"
        assert cases.sha(motion_compensate(sc, c.params["compensation"]).points) == ref["points"][k]


@pytest.mark.parametrize("mode", ["se3", "yaw"])
def test_host_deskew_matches_host_port_random(mode, host):
    from scipy.spatial.transform import Rotation as R

    from paper_2509_20081_b200.transforms import make_pose

    rng = np.random.default_rng(17 if mode == "se3" else 18)
    for trial in range(24):
        T0 = make_pose(R.random(random_state=trial) if trial % 3 == 0 else
                       R.from_euler("zyx", [rng.uniform(-3.1, 3.1), rng.normal() * 0.05, rng.normal() * 0.05]),
                       rng.normal(size=3) * 5)
        d = R.from_rotvec(rng.normal(size=3) * rng.uniform(0, 0.5)) if trial % 3 else R.from_euler("z", 3.0)
        T1 = make_pose(d * R.from_matrix(T0[:3, :3]), T0[:3, 3] + rng.normal(size=3))
        n = int(rng.integers(1, 2500))
        pts = (rng.normal(size=(n, 3)) * 10).astype(np.float32 if trial % 4 == 0 else np.float64)
        ts = None if trial % 5 == 0 else np.sort(rng.uniform(-0.1, 1.1, n))
        sc = ScanFrame(points=pts, pose=T1, prev_pose=T0, timestamps=ts)
        want = motion_compensate(sc, mode).points
        got = _host_deskew(host, deskew_params(sc, mode), sc.points, ts)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), trial


@pytest.mark.parametrize("c", [c for c in DESKEW if not c.name.startswith("deskew_cfg")], ids=lambda c: c.name)
def test_oracle_on_deskewed_points_reproduces_reference_grid(c, golden):
    ref = golden["deskew"][c.name]
    bank = build_kernel_bank(**c.bank)
    og = oracle.OracleGrid(c.dims, c.voxel_size, c.origin)
    ob = oracle.OracleBank.from_bank(bank)
    for k, fr in enumerate(c.frames):
        sc = _downsampled(c, fr)
        st = oracle.integrate_frame(og, ob, motion_compensate(sc, c.params["compensation"]).points, fr[1], threads=4)
        assert [st.points_in, st.points_discarded] == ref["stats"][k][:2]
    assert (cases.sha(og.mask), cases.sha(og.sign), cases.sha(og.hits)) == (ref["mask"], ref["sign"], ref["hits"])


# ---------------------------------------------------------------- GPU

gpu = pytest.mark.gpu


@gpu
def test_device_deskew_available():
    from paper_2509_20081_b200.integrator import device_deskew_available

    assert device_deskew_available()


@gpu
@pytest.mark.parametrize("c", DESKEW, ids=lambda c: c.name)
def test_device_deskew_points_match_reference(c, golden):
    ref = golden["deskew"][c.name]
    L = _native.lib()
    ds = c.params.get("downsample", 1)
    for k, (pts, pose, prev, ts) in enumerate(c.frames):
        sc = ScanFrame(points=pts, pose=pose, prev_pose=prev, timestamps=ts)
        d = deskew_params(sc, c.params["compensation"])
        payload, dtype = sc.device_payload()
        m = (payload.shape[0] + ds - 1) // ds
        out = np.empty((m, 3))
        tsp = None if ts is None else np.ascontiguousarray(ts, np.float64)
        _native.check(L.dbt_deskew_points(0, _ptr(payload), dtype, payload.shape[0],
                                          None if tsp is None else _ptr(tsp), ds, ctypes.byref(d), _ptr(out)))
        assert cases.sha(out) == ref["points"][k], f"frame {k}"


@gpu
@pytest.mark.parametrize("batched", [False, True])
@pytest.mark.parametrize("c", DESKEW, ids=lambda c: c.name)
def test_device_deskew_integration_matches_reference(c, batched, golden):
    from paper_2509_20081_b200 import integrate_frames

    ref = golden["deskew"][c.name]
    bank = build_kernel_bank(**c.bank)
    g = new_grid(c.dims, c.voxel_size, c.origin)
    params = IntegrationParams(**c.params)
    frames = [ScanFrame(points=p, pose=pose, prev_pose=prev, timestamps=ts) for p, pose, prev, ts in c.frames]
    sts = integrate_frames(g, bank, frames, params) if batched else [integrate_frame(g, bank, f, params)
                                                                       for f in frames]
    assert [[s.points_in, s.points_discarded] for s in sts] == [r[:2] for r in ref["stats"]]
    m, s, h = g.download_range(0, c.dims[0])
    assert cases.sha(m) == ref["mask"], "mask differs from the reference"
    assert cases.sha(s) == ref["sign"], "sign differs from the reference"
    assert cases.sha(h) == ref["hits"], "hits differ from the reference"


@gpu
def test_device_deskew_exact_voxels_written(golden):
    """The serial voxels_written of the reference on a compensated scan."""
    c = next(c for c in DESKEW if c.name == "deskew_se3_linspace")
    ref = golden["deskew"][c.name]
    bank = build_kernel_bank(**c.bank)
    g = new_grid(c.dims, c.voxel_size, c.origin)
    params = IntegrationParams(exact_voxels_written=True, **c.params)
    for k, (p, pose, prev, ts) in enumerate(c.frames):
        st = integrate_frame(g, bank, ScanFrame(points=p, pose=pose, prev_pose=prev, timestamps=ts), params)
        assert [st.points_in, st.points_discarded, st.voxels_written] == ref["stats"][k]
