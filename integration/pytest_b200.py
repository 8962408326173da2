"""pytest plugin: run the reference's OWN test suites against the B200 drop-in.

SURVEY.md §4 / VERDICT r1 "missing #5": the reference's hot-path suites
(pkg/tests/test_integrator.py, test_oracle.py, test_acceptance.py,
test_mesher.py) call ``bitsdf.integrator.integrate_frame`` /
``integrate_point`` and ``bitsdf.mesher.extract_mesh``. This plugin installs
``integration/bitsdf_b200.py`` inside the imported reference package as
``bitsdf._b200`` (exactly where INTEGRATION.md §2 tells a maintainer to put
it) and rebinds those three names in every ``bitsdf`` module before the test
modules are collected, so the reference's unmodified tests exercise the CUDA
engine through the C ABI.

usage (GPU box; the reference package on the path, e.g. installed with
``pip install --no-deps --target baseline/_ref <reference>/pkg``)::

    PYTHONPATH=baseline/_ref:integration BITSDF_B200_LIB=$PWD/paper_2509_20081_b200/libdbtsdf.so \
        python -m pytest -p pytest_b200 <reference>/pkg/tests/test_integrator.py ...

``BITSDF_B200_CROSSCHECK=1`` additionally runs the reference's CPU function
on a copy of the same grid for EVERY call the suites make and asserts that
mask, sign, hits and the FrameStats counts are identical (voxels_written too
when ``DBT_EXACT_VOXELS_WRITTEN=1``), and that meshes are equal array for
array: a live reference comparison, not a golden file.

The plugin holds no reference code: it only moves names around.
"""

from __future__ import annotations

import copy
import importlib
import importlib.util
import os
import sys
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
CALLS = {"integrate_frame": 0, "integrate_point": 0, "extract_mesh": 0, "crosschecked": 0}


def _load_shim(bitsdf):
    spec = importlib.util.spec_from_file_location("bitsdf._b200", _HERE / "bitsdf_b200.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules["bitsdf._b200"] = mod
    spec.loader.exec_module(mod)  # its relative imports resolve to the reference's modules
    bitsdf._b200 = mod
    return mod


def _grid_copy(grid):
    g = copy.copy(grid)
    g.mask, g.sign, g.hits = grid.mask.copy(), grid.sign.copy(), grid.hits.copy()
    for k in ("_dbt_grid", "_dbt_resident"):
        g.__dict__.pop(k, None)
    return g


def _same_grid(a, b, what):
    for f in ("mask", "sign", "hits"):
        x, y = getattr(a, f), getattr(b, f)
        if not np.array_equal(x, y):
            bad = np.argwhere(x != y)
            raise AssertionError(f"{what}: {f} differs from the reference at {len(bad)} voxels, first {bad[0].tolist()}")


def install():
    import bitsdf
    from bitsdf import integrator as ri
    from bitsdf import mesher as rm

    shim = _load_shim(bitsdf)
    shim.lib(os.environ.get("BITSDF_B200_LIB"))
    cross = os.environ.get("BITSDF_B200_CROSSCHECK") == "1"
    exact = os.environ.get("DBT_EXACT_VOXELS_WRITTEN") == "1"
    cpu_frame, cpu_point, cpu_mesh = ri.integrate_frame, ri.integrate_point, rm.extract_mesh

    def integrate_frame(grid, bank, scan, params, threads=1):
        CALLS["integrate_frame"] += 1
        ref = _grid_copy(grid) if cross else None
        st = shim.integrate_frame(grid, bank, scan, params, threads=threads)
        if cross:
            rs = cpu_frame(ref, bank, scan, params, threads=threads)
            _same_grid(grid, ref, "integrate_frame")
            assert (st.points_in, st.points_discarded) == (rs.points_in, rs.points_discarded), (st, rs)
            if exact:
                assert st.voxels_written == rs.voxels_written, (st, rs)
            CALLS["crosschecked"] += 1
        return st

    def integrate_point(grid, bank, p_map, sensor_pos, params):
        CALLS["integrate_point"] += 1
        ref = _grid_copy(grid) if cross else None
        out = shim.integrate_point(grid, bank, p_map, sensor_pos, params)
        if cross:
            assert cpu_point(ref, bank, p_map, sensor_pos, params) == out
            _same_grid(grid, ref, "integrate_point")
            CALLS["crosschecked"] += 1
        return out

    def extract_mesh(grid, iso=0.0):
        CALLS["extract_mesh"] += 1
        if min(grid.dims) < 2:  # mesher.py:46-47
            return rm.empty_mesh()
        v, f = shim.extract_mesh(grid, iso)
        mesh = rm.TriangleMesh(vertices=v, triangles=f) if len(v) else rm.empty_mesh()
        if cross:
            r = cpu_mesh(grid, iso)
            assert np.array_equal(mesh.vertices, r.vertices) and np.array_equal(mesh.triangles, r.triangles), \
                "extract_mesh differs from the reference"
            CALLS["crosschecked"] += 1
        return mesh

    new = {id(cpu_frame): integrate_frame, id(cpu_point): integrate_point, id(cpu_mesh): extract_mesh}
    for sub in ("cli", "oracle", "metrics", "io"):
        try:
            importlib.import_module(f"bitsdf.{sub}")
        except Exception:  # an optional dependency of a module outside the hot path
            pass
    for name, mod in list(sys.modules.items()):
        if name == "bitsdf" or name.startswith("bitsdf."):
            for attr, val in list(vars(mod).items()):
                if id(val) in new and mod is not shim:
                    setattr(mod, attr, new[id(val)])
    bitsdf._b200_cpu = {"integrate_frame": cpu_frame, "integrate_point": cpu_point, "extract_mesh": cpu_mesh}
    return shim


def pytest_configure(config):
    install()


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(
        "bitsdf B200 drop-in: " + ", ".join(f"{k} {v}" for k, v in CALLS.items()) +
        f" (crosscheck {'on' if os.environ.get('BITSDF_B200_CROSSCHECK') == '1' else 'off'}, "
        f"exact voxels_written {'on' if os.environ.get('DBT_EXACT_VOXELS_WRITTEN') == '1' else 'off'})")
