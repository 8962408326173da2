"""Marching cubes (reference mesher.py:43-127).

CPU: the oracle restatement (oracle/mc_oracle.py) reproduces the reference's
own meshes on the golden grids (hashes in tests/golden/golden.json, tables
in tests/golden/mc_tables.npz, both written by make_golden.py --only-mesh),
and the reference's mesh properties (closed surfaces, unobserved frontier).

GPU: the device mesher (csrc/mesh.cu through dbt_mesh_extract) against the
same golden hashes and against the oracle on hand-built and random grids:
vertices bit-exact float64, triangles exact int64, same order.
"""

from pathlib import Path

import numpy as np
import pytest

import cases
from oracle import mc_oracle

TABLES = Path(__file__).resolve().parent / "golden" / "mc_tables.npz"
MESH_CASES = ("frame500_default", "arbitrary_state", "nonfresh_cone_h200_t2", "k9_bins8", "cfg2_scans0-2")
FULL = 0xFFFFFFFF


def tables():
    return dict(np.load(TABLES))


def run_mask(k):
    return 0 if k <= 0 else (FULL >> (32 - min(k, 32)))


def ball_state(n=20, vs=0.05, radius=0.25):
    """Signed field of a ball centred in an n^3 grid, every voxel observed."""
    c = (np.indices((n, n, n)).transpose(1, 2, 3, 0) + 0.5) * vs
    r = np.linalg.norm(c - n * vs / 2, axis=-1)
    cells = np.clip(np.ceil(np.abs(r - radius) / vs).astype(np.int64), 0, 32)
    mask = np.array([run_mask(k) for k in range(33)], dtype=np.uint32)[cells]
    inside = r < radius
    sign = np.where(inside, 0, 1).astype(np.uint8)
    hits = np.where(inside, 5, 1).astype(np.uint8)
    return mask, sign, hits


def one_voxel_state(n=7, observed=True):
    mask = np.full((n, n, n), run_mask(3) if observed else FULL, np.uint32)
    sign = np.ones((n, n, n), np.uint8)
    hits = np.full((n, n, n), 1 if observed else 0, np.uint8)
    c = n // 2
    mask[c, c, c], sign[c, c, c], hits[c, c, c] = 0, 0, 2
    return mask, sign, hits


def edge_counts(tri):
    e = np.sort(np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [2, 0]]]), axis=1)
    _, cnt = np.unique(e, axis=0, return_counts=True)
    return cnt


def final_oracle_state(name):
    from test_oracle_golden import run_oracle

    c = next(c for c in cases.small_cases() + cases.config_cases(include_slow=False) if c.name == name)
    g, _, _ = run_oracle(c, threads=8)
    return c, g


def mesh_hashes(v, f):
    return (cases.sha(np.ascontiguousarray(v, dtype=np.float64)), cases.sha(np.ascontiguousarray(f, dtype=np.int64)),
            v.shape[0], f.shape[0])


def gold_tuple(entry):
    return entry["vertices"], entry["triangles"], entry["n_vertices"], entry["n_triangles"]


# --------------------------------------------------------------------- CPU
class TestOracleMesh:
    @pytest.mark.parametrize("name", MESH_CASES)
    def test_matches_reference(self, name, golden):
        c, g = final_oracle_state(name)
        ref = golden["cases"][name]
        assert cases.sha(g.mask) == ref["mask"]
        for iso in (0.0, 0.1):
            v, f = mc_oracle.mesh(g.mask, g.sign, g.hits, c.voxel_size, c.origin, iso, tables())
            assert mesh_hashes(v, f) == gold_tuple(ref["mesh"][repr(iso)])
            assert cases.sha(mc_oracle.normals(v, f)) == ref["mesh"][repr(iso)]["normals"]

    def test_single_voxel_closed_surface(self):
        v, f = mc_oracle.mesh(*one_voxel_state(), 0.1, (0, 0, 0), 0.0, tables())
        cnt = edge_counts(f)
        assert v.shape[0] - cnt.size + f.shape[0] == 2  # Euler characteristic of a sphere
        assert set(cnt.tolist()) == {2}

    def test_ball_watertight(self):
        v, f = mc_oracle.mesh(*ball_state(), 0.05, (0, 0, 0), 0.0, tables())
        assert f.shape[0] > 0 and set(edge_counts(f).tolist()) == {2}
        assert np.all(np.abs(np.linalg.norm(v - 0.5, axis=1) - 0.25) <= 0.05)

    def test_unobserved_frontier_empty(self):
        v, f = mc_oracle.mesh(*one_voxel_state(observed=False), 0.1, (0, 0, 0), 0.0, tables())
        assert v.shape == (0, 3) and f.shape == (0, 3)

    def test_tables_struct_matches_header(self):
        import ctypes

        from paper_2509_20081_b200.mesher import McTables, load_mc_tables

        assert ctypes.sizeof(McTables) == 4 * (256 + 4096 + 24 + 36 + 12)
        t = load_mc_tables(str(TABLES))
        ref = tables()
        assert list(t.edge_table) == ref["EDGE_TABLE"].tolist()
        assert list(t.tri_table) == ref["TRI_TABLE"].ravel().tolist()
        assert list(t.edge_axis) == ref["EDGE_AXIS"].tolist()

    def test_missing_table_rejected(self):
        from paper_2509_20081_b200.errors import ConfigurationError
        from paper_2509_20081_b200.mesher import load_mc_tables

        t = tables()
        del t["TRI_TABLE"]
        with pytest.raises(ConfigurationError):
            load_mc_tables(t)
        t = tables()
        t["EDGE_AXIS"] = t["EDGE_AXIS"][:11]
        with pytest.raises(ConfigurationError):
            load_mc_tables(t)


# --------------------------------------------------------------------- GPU
def device_grid(state, vs=0.1, origin=(0.0, 0.0, 0.0)):
    from paper_2509_20081_b200 import new_grid

    m, s, h = state
    g = new_grid(m.shape, vs, origin)
    g.mask[...], g.sign[...], g.hits[...] = m, s, h
    g.release_host()
    return g


def device_mesh(g, iso=0.0):
    from paper_2509_20081_b200.mesher import extract_mesh

    return extract_mesh(g, iso, tables=tables())


def assert_same(mesh, v, f):
    assert mesh.vertices.dtype == np.float64 and mesh.triangles.dtype == np.int64
    assert mesh.vertices.shape == v.shape and mesh.triangles.shape == f.shape
    assert np.array_equal(mesh.vertices.view(np.uint64), np.ascontiguousarray(v).view(np.uint64))
    assert np.array_equal(mesh.triangles, f)


@pytest.mark.gpu
class TestDeviceMesh:
    @pytest.mark.parametrize("name", MESH_CASES)
    def test_matches_reference(self, name, golden):
        from test_gpu_parity import engine_run

        c = next(c for c in cases.small_cases() + cases.config_cases(include_slow=False) if c.name == name)
        g, _, _ = engine_run(c)
        ref = golden["cases"][name]
        for iso in (0.0, 0.1):
            m = device_mesh(g, iso)
            assert mesh_hashes(m.vertices, m.triangles) == gold_tuple(ref["mesh"][repr(iso)])

    def test_after_batched_frames(self, golden):
        """integrate_frames leaves shadow visits pending in the records; the
        mesher folds them first."""
        from test_gpu_parity import engine_run

        c = next(c for c in cases.small_cases() if c.name == "nonfresh_cone_h200_t2")
        g, _, _ = engine_run(c, batch=True)
        m = device_mesh(g, 0.0)
        assert mesh_hashes(m.vertices, m.triangles) == gold_tuple(golden["cases"][c.name]["mesh"]["0.0"])

    @pytest.mark.parametrize("iso", [0.0, -0.0, 0.05, 0.1, -0.1, 0.3, -3.2, 3.3, 0.123])
    def test_random_state_vs_oracle(self, iso):
        rng = np.random.default_rng(5)
        dims = (23, 17, 29)
        k = rng.integers(0, 33, size=dims)
        mask = np.array([run_mask(i) for i in range(33)], dtype=np.uint32)[k]
        mask[rng.random(dims) < 0.1] = FULL
        sel = rng.random(dims) < 0.05  # arbitrary (non-run) masks
        mask[sel] = rng.integers(0, 2**32, size=int(sel.sum()), dtype=np.uint64).astype(np.uint32)
        sign = rng.integers(0, 3, size=dims).astype(np.uint8)
        hits = rng.integers(0, 3, size=dims).astype(np.uint8)
        org = (-1.25, 0.5, 3.0)
        g = device_grid((mask, sign, hits), 0.1, org)
        v, f = mc_oracle.mesh(mask, sign, hits, 0.1, org, iso, tables())
        assert f.shape[0] > 0 or iso in (-3.2, 3.3)
        assert_same(device_mesh(g, iso), v, f)

    def test_ball_vs_oracle(self):
        st = ball_state()
        g = device_grid(st, 0.05)
        m = device_mesh(g)
        v, f = mc_oracle.mesh(*st, 0.05, (0, 0, 0), 0.0, tables())
        assert_same(m, v, f)
        assert set(edge_counts(m.triangles).tolist()) == {2}

    def test_single_voxel(self):
        st = one_voxel_state()
        m = device_mesh(device_grid(st))
        v, f = mc_oracle.mesh(*st, 0.1, (0, 0, 0), 0.0, tables())
        assert_same(m, v, f)
        cnt = edge_counts(m.triangles)
        assert m.vertices.shape[0] - cnt.size + m.triangles.shape[0] == 2

    def test_unobserved_and_fresh_are_empty(self):
        from paper_2509_20081_b200 import new_grid

        assert device_mesh(device_grid(one_voxel_state(observed=False))).is_empty
        m = device_mesh(new_grid((10, 10, 10), 0.1))
        assert m.vertices.shape == (0, 3) and m.triangles.shape == (0, 3) and m.triangles.dtype == np.int64

    @pytest.mark.parametrize("dims", [(1, 5, 5), (5, 1, 5), (5, 5, 1), (2, 2, 2), (2, 3, 9)])
    def test_thin_grids(self, dims):
        rng = np.random.default_rng(9)
        k = rng.integers(0, 4, size=dims)
        st = (np.array([run_mask(i) for i in range(33)], dtype=np.uint32)[k], rng.integers(0, 2, size=dims)
              .astype(np.uint8), np.ones(dims, np.uint8))
        v, f = mc_oracle.mesh(*st, 0.1, (0, 0, 0), 0.1, tables())
        assert_same(device_mesh(device_grid(st), 0.1), v, f)

    def test_deterministic_and_device_buffers(self):
        from paper_2509_20081_b200.mesher import extract_mesh_device

        g = device_grid(ball_state(), 0.05)
        a, b = device_mesh(g), device_mesh(g)
        assert np.array_equal(a.vertices, b.vertices) and np.array_equal(a.triangles, b.triangles)
        with extract_mesh_device(g, 0.0, tables()) as dm:
            pv, pf = dm.device_pointers()
            assert pv and pf and dm.n_vertices == a.vertices.shape[0] and dm.n_triangles == a.triangles.shape[0]

    def test_sharded_grid_rejected(self):
        from paper_2509_20081_b200.errors import ConfigurationError
        from paper_2509_20081_b200.grid import VoxelGrid

        g = VoxelGrid((16, 8, 8), 0.1, (0, 0, 0), slab=(0, 8))
        with pytest.raises(ConfigurationError):
            device_mesh(g)

    @pytest.mark.parametrize("name", ("arbitrary_state", "cfg2_scans0-2"))
    def test_normals_match_reference(self, name, golden):
        from test_gpu_parity import engine_run

        from paper_2509_20081_b200.mesher import vertex_normals

        c = next(c for c in cases.small_cases() + cases.config_cases(include_slow=False) if c.name == name)
        g, _, _ = engine_run(c)
        for iso in (0.0, 0.1):
            m = vertex_normals(device_mesh(g, iso))
            assert cases.sha(m.normals) == golden["cases"][name]["mesh"][repr(iso)]["normals"]

    def test_normals_device_handle(self):
        from paper_2509_20081_b200.mesher import extract_mesh_device

        st = ball_state()
        v, f = mc_oracle.mesh(*st, 0.05, (0, 0, 0), 0.0, tables())
        with extract_mesh_device(device_grid(st, 0.05), 0.0, tables()) as dm:
            n = dm.normals()
        want = mc_oracle.normals(v, f)
        assert np.array_equal(n.view(np.uint64), want.view(np.uint64))
        radial = v - 0.5
        radial /= np.linalg.norm(radial, axis=1, keepdims=True)
        assert np.mean(np.abs(np.sum(n * radial, axis=1))) > 0.9

    def test_normals_hand_meshes(self):
        from paper_2509_20081_b200.errors import ConfigurationError
        from paper_2509_20081_b200.mesher import TriangleMesh, vertex_normals

        rng = np.random.default_rng(3)
        v = rng.normal(size=(40, 3))
        f = rng.integers(0, 40, size=(120, 3))
        f[:5] = [[0, 0, 1], [2, 3, 2], [4, 4, 4], [5, 6, 7], [5, 6, 7]]  # degenerate + duplicate faces
        v[39] = [5, 5, 5]
        f[f == 39] = 38                                                   # vertex 39 isolated
        f[7] = [-2, -3, 3]                                                # numpy-style negative indices
        got = vertex_normals(TriangleMesh(v, f)).normals
        assert np.array_equal(got.view(np.uint64), mc_oracle.normals(v, f).view(np.uint64))
        assert np.all(got[39] == 0.0)
        one = vertex_normals(TriangleMesh(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]), np.array([[0, 1, 2]])))
        assert np.allclose(np.abs(one.normals[:, 2]), 1.0) and np.allclose(one.normals[:, :2], 0.0)
        e = vertex_normals(TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64)))
        assert e.normals.shape == (0, 3)
        lone = vertex_normals(TriangleMesh(np.ones((2, 3)), np.zeros((0, 3), dtype=np.int64)))
        assert np.array_equal(lone.normals, np.zeros((2, 3)))
        with pytest.raises(ConfigurationError):
            vertex_normals(TriangleMesh(v, np.array([[0, 1, 40]])))

    def test_bad_tables_rejected(self):
        from paper_2509_20081_b200.errors import ConfigurationError
        from paper_2509_20081_b200.mesher import extract_mesh

        g = device_grid(ball_state(), 0.05)
        for key, val in (("EDGE_AXIS", 3), ("TRI_TABLE", 12), ("EDGE_BASE", 2)):
            t = tables()
            t[key] = t[key].copy()
            t[key].ravel()[5] = val
            with pytest.raises(ConfigurationError):
                extract_mesh(g, 0.0, tables=t)


def test_packaged_tables_equal_the_reference_tables():
    """The tables shipped in the package are the ones the reference meshes
    were pinned with (tests/golden/mc_tables.npz, written from the
    reference's _mc_tables by make_golden.py --only-mesh)."""
    from paper_2509_20081_b200.mesher import _PKG_TABLES

    a, b = np.load(_PKG_TABLES), np.load(TABLES)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
