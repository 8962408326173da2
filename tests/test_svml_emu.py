"""The device binning's arctan2/arcsin restatement (csrc/svml_emu.cuh) against
numpy itself, on the CPU: the same header is compiled for the host
(-ffp-contract=off) and must reproduce numpy's float64 arctan2/arcsin bit for
bit — numpy is the reference's dependency for these two calls
(kernels.py:51-55). Also pins the committed VRCP14/VRSQRT14 seed table to the
hardware instructions when the host has AVX-512."""

import ctypes
import math
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
SEEDS = ROOT / "paper_2509_20081_b200" / "csrc" / "svml_seeds.bin"


def _simd_dispatch():
    import numpy._core._multiarray_umath as m

    return bool(m.__cpu_features__.get("AVX512_SKX"))


pytestmark = pytest.mark.skipif(not _simd_dispatch(),
                                reason="numpy uses SVML only on AVX512_SKX hosts (build container and GPU box both are)")


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    out = tmp_path_factory.mktemp("svml") / "libsvmlhost.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                    str(ROOT / "tests" / "native" / "svml_host.cpp"), "-o", str(out)], check=True)
    L = ctypes.CDLL(str(out))
    tab = np.fromfile(SEEDS, dtype=np.uint16)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731

    def atan2(y, x):
        y = np.ascontiguousarray(y, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(y)
        rare = np.zeros(len(y), np.int32)
        L.svml_atan2_arr(P(y), P(x), ctypes.c_long(len(y)), P(tab), P(out), P(rare))
        return out, rare

    def asin(x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty_like(x)
        L.svml_asin_arr(P(x), ctypes.c_long(len(x)), P(tab), P(out))
        return out

    return atan2, asin


def _same(a, b):
    return a.view(np.uint64) == b.view(np.uint64)


def test_atan2_random_and_structured(emu):
    atan2, _ = emu
    rng = np.random.default_rng(0)
    n = 400_000
    d = rng.uniform(0.1, 100, n)
    sets = {
        "normal": (rng.normal(size=n), rng.normal(size=n)),
        "wide": (rng.normal(size=n) * 10.0 ** rng.uniform(-8, 8, n), rng.normal(size=n) * 10.0 ** rng.uniform(-8, 8, n)),
        "diagonals": (d * rng.choice([-1, 1], n), d * (1 + rng.integers(-4, 5, n) * 2.0 ** -52) * rng.choice([-1, 1], n)),
        "zeros": (np.where(rng.random(n) < .5, 0.0, rng.normal(size=n)) * rng.choice([-1., 1.], n),
                  np.where(rng.random(n) < .5, 0.0, rng.normal(size=n)) * rng.choice([-1., 1.], n)),
    }
    for name, (y, x) in sets.items():
        got, rare = atan2(y, x)
        assert int(rare.sum()) == 0, name
        assert np.all(_same(got, np.arctan2(y, x))), name


def test_asin_full_range(emu):
    _, asin = emu
    rng = np.random.default_rng(1)
    q = np.concatenate([rng.uniform(-1, 1, 400_000), 1 - rng.uniform(0, 1e-6, 50_000), rng.normal(size=50_000) * 1e-5,
                        [0.0, -0.0, 0.5, -0.5, 1.0, -1.0, math.sqrt(0.5), -math.sqrt(0.5), np.nextafter(0.5, 0),
                         np.nextafter(1.0, 0)]])
    q = np.clip(q, -1.0, 1.0)
    assert np.all(_same(asin(q), np.arcsin(q)))


def test_spin_fans_bins_match(emu):
    """Noise-free azimuth x elevation fans (every 45-degree multiple hit
    exactly): the restated binning equals numpy's bins everywhere, which
    libm / CUDA atan2 do not."""
    from oracle import prep

    atan2, asin = emu
    for n_az, n_el in ((200, 100), (250, 200), (2048, 128), (1800, 16)):
        az = np.linspace(0.0, 2 * np.pi, n_az, endpoint=False)
        el = np.radians(np.linspace(-80, 80, n_el))
        aa, ee = np.meshgrid(az, el, indexing="ij")
        dirs = np.stack([np.cos(ee) * np.cos(aa), np.cos(ee) * np.sin(aa), np.sin(ee)], -1).reshape(-1, 3)
        for t in ((0.0, 0.0, 0.0), (3.2, 7.1, 1.5), (100.0, 100.0, 1.8)):
            p = dirs * 7.3 + np.array(t)
            rays = p - np.array(t)
            n = np.linalg.norm(rays, axis=1)
            a, _ = atan2(rays[:, 1], rays[:, 0])
            a = np.where(a < 0.0, a + 2 * math.pi, a)
            b_a = np.clip((a / (2 * math.pi) * 40).astype(np.int64), 0, 39)
            e = asin(np.clip(rays[:, 2] / n, -1.0, 1.0))
            b_e = np.clip(((e + np.pi / 2) / np.pi * 40).astype(np.int64), 0, 39)
            ra, re = prep.bin_index_array(rays, 40, 40)
            assert np.array_equal(b_a, ra) and np.array_equal(b_e, re)


def test_seed_table_matches_hardware(tmp_path):
    """The committed seed table equals the VRCP14PD/VRSQRT14PD outputs of
    this CPU (regenerated with tools/gen_svml_seeds.c)."""
    import os

    flags = open("/proc/cpuinfo").read() if os.path.exists("/proc/cpuinfo") else ""
    if "avx512f" not in flags:
        pytest.skip("no AVX-512 on this host")
    exe = tmp_path / "gen"
    subprocess.run(["gcc", "-O2", "-mavx512f", str(ROOT / "tools" / "gen_svml_seeds.c"), "-o", str(exe)], check=True)
    out = tmp_path / "seeds.bin"
    subprocess.run([str(exe), str(out)], check=True)
    assert out.read_bytes() == SEEDS.read_bytes()
