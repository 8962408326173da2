"""GPU parity: the libdbtsdf engine, called through the drop-in API / C ABI,
against the reference's golden outputs and the oracle.

Bar: bit-exact final mask/sign/hits (integer state) and exact
points_in/points_discarded; voxels_written is the concurrent change count
(DESIGN.md §voxels_written), checked for its bounds.
"""

import numpy as np
import pytest

import cases
import oracle
from oracle import prep
from paper_2509_20081_b200 import (
    IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, integrate_frames, integrate_point,
    integrate_points, new_grid)
from paper_2509_20081_b200 import grid as G
from paper_2509_20081_b200 import kernels as Kmod
from paper_2509_20081_b200 import _native
from paper_2509_20081_b200.errors import ConfigurationError, CorruptionError

pytestmark = pytest.mark.gpu

SMALL = cases.small_cases()
CONFIG = cases.config_cases(include_slow=True)


def engine_run(c: cases.Case, batch=False, point_loop=True):
    bank = build_kernel_bank(**c.bank)
    g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 42)
    if c.init is not None:
        g.mask[...] = c.init[0]
        g.sign[...] = c.init[1]
        g.hits[...] = c.init[2]
        g.release_host()  # device authoritative again; the upload happens here
    params = IntegrationParams(**c.params)
    stats = []
    if c.frames:
        frames = [ScanFrame(points=p, pose=pose) for p, pose in c.frames]
        if batch and len(frames) > 1:
            sts = integrate_frames(g, bank, frames, params)
        else:
            sts = [integrate_frame(g, bank, f, params) for f in frames]
        stats = [[s.points_in, s.points_discarded, s.voxels_written] for s in sts]
    applied = None
    if c.hits is not None:
        if point_loop:
            applied = sum(integrate_point(g, bank, p, s, params) == "applied" for p, s in zip(*c.hits))
        else:
            applied = int(integrate_points(g, bank, c.hits[0], c.hits[1], params).sum())
    return g, stats, applied


def check(c, gold, g, stats, applied, batch=False):
    ref = gold["cases"][c.name]
    assert ref["input"] == c.input_hash(), "generator drift: inputs differ from the reference run"
    m, s, h = g.download_range(0, c.dims[0])
    assert cases.sha(m) == ref["mask"], "mask differs from the reference"
    assert cases.sha(s) == ref["sign"], "sign differs from the reference"
    assert cases.sha(h) == ref["hits"], "hits differ from the reference"
    assert applied == ref["applied"]
    K3 = c.bank.get("size", 21) ** 3
    assert len(stats) == len(ref["stats"])
    for got, want in zip(stats, ref["stats"]):
        assert got[:2] == want[:2]
    if batch:  # one launch: the change count is launch-wide, reported on the first scan
        stats = [[sum(x[0] for x in stats), sum(x[1] for x in stats), sum(x[2] for x in stats)]]
        want_w = sum(x[2] for x in ref["stats"])
        wants = [[0, 0, want_w]]
    else:
        wants = ref["stats"]
    for got, want in zip(stats, wants):
        if want[2] == 0:
            assert got[2] == 0
        else:
            assert 0 < got[2] <= (got[0] - got[1]) * K3


@pytest.mark.parametrize("c", SMALL, ids=[c.name for c in SMALL])
def test_engine_matches_reference_small(c, golden):
    check(c, golden, *engine_run(c))


@pytest.mark.parametrize("c", CONFIG, ids=[c.name for c in CONFIG])
def test_engine_matches_reference_configs(c, golden):
    check(c, golden, *engine_run(c))


@pytest.mark.parametrize("name", ["yaw_frames_f32", "nonfresh_cone_h200_t2", "cfg2_scans0-2", "cfg3_scans0-1"])
def test_batched_launch_matches_reference(name, golden):
    """Config-5 path: several scans in one launch sequence."""
    c = next(x for x in SMALL + CONFIG if x.name == name)
    check(c, golden, *engine_run(c, batch=True), batch=True)


def test_batched_integrate_points_matches_reference(golden):
    c = next(x for x in SMALL if x.name == "c1_points10k")
    check(c, golden, *engine_run(c, point_loop=False))


@pytest.mark.parametrize("name", list(cases.bin_dir_sets()))
def test_device_bins_match_reference(name, golden):
    dirs = cases.bin_dir_sets()[name]
    ref = golden["bins"][name]
    b_a, b_e = Kmod.bin_index_array(dirs, 40, 40)
    assert cases.sha(b_a) == ref["b_a"]
    assert cases.sha(b_e) == ref["b_e"]


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_device_bins_match_numpy_on_config_rays(cfg):
    """Every map-frame ray of a config scan bins identically on the device and
    in numpy (the reference's arctan2/arcsin)."""
    import workloads

    w = workloads.get(cfg)
    for k in range(min(3, w.n_scans)):
        pts = w.scan(k).astype(np.float64)
        pose = w.poses[k]
        rays = prep.transform(pts, pose) - pose[:3, 3]
        rays = rays[np.linalg.norm(rays, axis=1) > 0]
        ra, re = prep.bin_index_array(rays, 40, 40)
        da, de = Kmod.bin_index_array(rays, 40, 40)
        assert int((ra != da).sum()) == 0 and int((re != de).sum()) == 0


@pytest.mark.parametrize("n_az,n_el", [(200, 100), (250, 200), (2048, 128), (1800, 16)])
def test_device_bins_match_numpy_on_noise_free_fans(n_az, n_el):
    """Exact azimuth x elevation fans (45-degree multiples hit exactly, the
    structured knife edges where CUDA's own atan2 differs from numpy's) from
    several sensor positions: device bins == numpy bins for every ray."""
    az = np.linspace(0.0, 2 * np.pi, n_az, endpoint=False)
    el = np.radians(np.linspace(-80, 80, n_el))
    aa, ee = np.meshgrid(az, el, indexing="ij")
    dirs = np.stack([np.cos(ee) * np.cos(aa), np.cos(ee) * np.sin(aa), np.sin(ee)], -1).reshape(-1, 3)
    for t in ((0.0, 0.0, 0.0), (3.2, 7.1, 1.5), (100.0, 100.0, 1.8)):
        rays = (dirs * 7.3 + np.array(t)) - np.array(t)
        ra, re = prep.bin_index_array(rays, 40, 40)
        da, de = Kmod.bin_index_array(rays, 40, 40)
        assert np.array_equal(ra, da) and np.array_equal(re, de)


def test_slab_grids_reassemble_reference():
    """Multi-GPU decomposition on one device: three x-slab grids integrate the
    same scan; their union is the reference grid."""
    import workloads

    c = next(x for x in CONFIG if x.name == "cfg1_scan0")
    bank = build_kernel_bank(**c.bank)
    pts, pose = c.frames[0]
    nx = c.dims[0]
    parts = []
    for x0, x1 in ((0, 70), (70, 71), (71, nx)):
        g = G.VoxelGrid(c.dims, c.voxel_size, c.origin, slab=(x0, x1))
        st = integrate_frame(g, bank, ScanFrame(points=pts, pose=pose), IntegrationParams())
        assert (st.points_in, st.points_discarded) == (28800, 0)
        parts.append(g.download_range(x0, x1))
    full = [np.concatenate([p[i] for p in parts]) for i in range(3)]
    ref = oracle.OracleGrid(c.dims, c.voxel_size, c.origin)
    oracle.integrate_frame(ref, oracle.OracleBank.from_bank(bank), pts, pose, threads=8)
    assert np.array_equal(full[0], ref.mask) and np.array_equal(full[1], ref.sign)
    assert np.array_equal(full[2], ref.hits)


@pytest.fixture(scope="module")
def bank():
    return build_kernel_bank(shadow_radius=3)


class TestReferenceBehaviours:
    """The reference's own integrator tests (test_integrator.py) re-expressed
    against the drop-in API."""

    def fresh(self, n=41):
        return new_grid((n, n, n), 0.1)

    def test_center_stamp_distances(self, bank):
        g = self.fresh()
        p = np.array([2.05, 2.05, 2.05])
        assert integrate_point(g, bank, p, p - [1, 0, 0], IntegrationParams()) == "applied"
        pc = G.popcount_array(g.mask)
        assert (pc[20, 20, 20], pc[23, 20, 20], pc[20, 25, 20]) == (0, 3, 5)
        assert np.array_equal(G.popcount_array(g), pc)  # device readout == host popcount

    def test_and_idempotence(self, bank):
        p = np.array([2.05, 2.05, 2.05])
        g = self.fresh()
        integrate_point(g, bank, p, p - [1, 0, 0], IntegrationParams())
        m1, h1 = g.mask.copy(), g.hits.copy()
        integrate_point(g, bank, p, p - [1, 0, 0], IntegrationParams())
        assert np.array_equal(g.mask, m1) and np.array_equal(g.hits, h1 * 2)

    def test_discards(self, bank):
        g = self.fresh()
        before = g.mask.copy()
        p = np.array([0.55, 2.05, 2.05])
        assert integrate_point(g, bank, p, p - [1, 0, 0], IntegrationParams()) == "discarded"
        p = np.array([2.05, 2.05, 2.05])
        assert integrate_point(g, bank, p, p - [0.001, 0, 0], IntegrationParams()) == "discarded"
        assert np.array_equal(g.mask, before)

    def test_sign_requires_threshold(self, bank):
        g = self.fresh()
        p = np.array([2.05, 2.05, 2.05])
        integrate_point(g, bank, p, p - [1, 0, 0], IntegrationParams(t_occ=2))
        assert g.sign[20, 20, 20] != G.SIGN_OCCUPIED
        integrate_point(g, bank, p, p - [1, 0, 0], IntegrationParams(t_occ=2))
        assert g.sign[20, 20, 20] == G.SIGN_OCCUPIED

    def test_empty_scan(self, bank):
        g = self.fresh()
        st = integrate_frame(g, bank, ScanFrame(points=np.zeros((0, 3)), pose=np.eye(4)), IntegrationParams())
        assert (st.points_in, st.points_discarded, st.voxels_written) == (0, 0, 0)
        assert np.all(g.mask == G.FULL_MASK)

    def test_order_and_permutation_independence(self, bank):
        rng = np.random.default_rng(11)
        pts = rng.uniform(1.2, 2.9, size=(2000, 3))
        grids = []
        for perm in (np.arange(2000), rng.permutation(2000), rng.permutation(2000)):
            g = self.fresh()
            integrate_frame(g, bank, ScanFrame(points=pts[perm], pose=np.eye(4)), IntegrationParams())
            grids.append((g.mask.copy(), g.sign.copy(), g.hits.copy()))
        for a in grids[1:]:
            for x, y in zip(grids[0], a):
                assert np.array_equal(x, y)

    def test_monotone_across_frames(self, bank):
        rng = np.random.default_rng(13)
        g = self.fresh()
        prev = G.popcount_array(g.mask)
        prev_sign = g.sign.copy()
        for _ in range(5):
            integrate_frame(g, bank, ScanFrame(points=rng.uniform(1.2, 2.9, (100, 3)), pose=np.eye(4)),
                            IntegrationParams())
            cur = G.popcount_array(g.mask)
            assert np.all(cur <= prev)
            assert not np.any((prev_sign == G.SIGN_OCCUPIED) & (g.sign != G.SIGN_OCCUPIED))
            prev, prev_sign = cur, g.sign.copy()

    def test_downsample_first_return_transform(self, bank):
        rng = np.random.default_rng(15)
        st = integrate_frame(self.fresh(), bank, ScanFrame(points=rng.uniform(1.2, 2.9, (100, 3)), pose=np.eye(4)),
                             IntegrationParams(downsample=4))
        assert st.points_in == 25
        g = self.fresh()
        p = np.array([[2.05, 2.05, 2.05], [2.06, 2.06, 2.06]])
        st = integrate_frame(g, bank, ScanFrame(points=p, pose=np.eye(4)),
                             IntegrationParams(first_return_per_voxel=True, t_occ=1))
        assert g.hits[20, 20, 20] == 1 and st.points_applied == 1
        from scipy.spatial.transform import Rotation

        from paper_2509_20081_b200.transforms import make_pose

        g = self.fresh()
        integrate_frame(g, bank, ScanFrame(points=np.array([[1.05, 2.05, 2.05]]),
                                           pose=make_pose(Rotation.identity(), (1.0, 0, 0))), IntegrationParams())
        assert G.popcount_array(g.mask)[20, 20, 20] == 0

    def test_compensated_frames_match_oracle(self, bank):
        """se3 deskew runs on the host exactly as the reference; the deskewed
        float64 points then go through the device path."""
        from scipy.spatial.transform import Rotation

        from paper_2509_20081_b200.integrator import motion_compensate
        from paper_2509_20081_b200.transforms import make_pose

        rng = np.random.default_rng(5)
        pts = rng.uniform(-0.8, 0.8, size=(500, 3))
        prev = make_pose(Rotation.from_euler("z", 0.05), (2.0, 2.0, 2.0))
        cur = make_pose(Rotation.from_euler("z", 0.15), (2.1, 2.05, 2.0))
        scan = ScanFrame(points=pts, pose=cur, prev_pose=prev)
        g = self.fresh()
        integrate_frame(g, bank, scan, IntegrationParams(compensation="se3", downsample=2))
        og = oracle.OracleGrid((41, 41, 41), 0.1, (0, 0, 0))
        k = ScanFrame(points=pts[::2], pose=cur, prev_pose=prev)
        oracle.integrate_frame(og, oracle.OracleBank.from_bank(bank), motion_compensate(k, "se3").points, cur)
        assert np.array_equal(g.mask, og.mask) and np.array_equal(g.hits, og.hits)
        assert np.array_equal(g.sign, og.sign)


class TestStampCertificate:
    """Skipping a centre whose own stamp is already applied (cache byte 0)
    must never change the grid."""

    def _oracle_after(self, bank, frames, init=None, dims=(48, 48, 48)):
        og = oracle.OracleGrid(dims, 0.1, (0, 0, 0))
        if init is not None:
            og.mask[...], og.sign[...], og.hits[...] = init
        for bk, pts in frames:
            oracle.integrate_frame(og, oracle.OracleBank.from_bank(bk), pts, np.eye(4))
        return og

    def test_repeat_scans_skip_and_match(self):
        bank = build_kernel_bank(shadow_radius=2)
        rng = np.random.default_rng(3)
        pts = rng.uniform(1.15, 3.6, size=(400, 3))
        g = new_grid((48, 48, 48), 0.1)
        s1 = integrate_frame(g, bank, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams())
        s2 = integrate_frame(g, bank, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams())
        assert s1.unique_centers + s1.centers_skipped == s1.points_applied == 400
        assert s1.unique_centers > 300
        assert s2.unique_centers == 0 and s2.centers_skipped == 400  # every stamp already applied
        og = self._oracle_after(bank, [(bank, pts), (bank, pts)])
        assert np.array_equal(g.mask, og.mask) and np.array_equal(g.hits, og.hits) and np.array_equal(g.sign, og.sign)

    def test_bank_change_voids_certificate(self):
        small = build_kernel_bank(size=9, shadow_radius=1)
        big = build_kernel_bank(size=21, shadow_radius=1)
        rng = np.random.default_rng(4)
        pts = rng.uniform(1.15, 3.6, size=(300, 3))
        g = new_grid((48, 48, 48), 0.1)
        s1 = integrate_frame(g, small, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams())
        st = integrate_frame(g, big, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams())
        # every distinct centre is swept again: the small kernel's stamps certify nothing
        assert st.unique_centers == s1.unique_centers > 250
        og = self._oracle_after(big, [(small, pts), (big, pts)])
        assert np.array_equal(g.mask, og.mask)

    def test_uploaded_zero_is_not_a_certificate(self):
        bank = build_kernel_bank(shadow_radius=1)
        g = new_grid((48, 48, 48), 0.1)
        g.mask[24, 24, 24] = 0  # distance 0 written by the host, no stamp applied
        init = (g.mask.copy(), g.sign.copy(), g.hits.copy())
        p = np.array([[2.45, 2.45, 2.45]])  # centre voxel (24, 24, 24)
        st = integrate_frame(g, bank, ScanFrame(points=p, pose=np.eye(4)), IntegrationParams())
        assert st.centers_skipped == 0
        og = self._oracle_after(bank, [(bank, p)], init=init)
        assert np.array_equal(g.mask, og.mask)


SNAP = [c for c in SMALL if c.name in ("frame500_default", "arbitrary_state", "nonfresh_cone_h200_t2", "k9_bins8")]


class TestSnapshot:
    """DBTSDF01 snapshots from the device layout (io.py:449-486): the bytes are
    the reference's own save_grid bytes for the same final grid."""

    @pytest.mark.parametrize("c", SNAP, ids=[c.name for c in SNAP])
    def test_save_matches_reference_bytes(self, c, golden, tmp_path, monkeypatch):
        import hashlib

        from paper_2509_20081_b200 import snapshot
        from paper_2509_20081_b200 import load_grid, save_grid

        g, _, _ = engine_run(c)
        params = IntegrationParams(**c.params)
        g.h_max, g.t_occ = params.h_max, params.t_occ
        p = tmp_path / "g.dbtsdf"
        save_grid(g, p)
        raw = p.read_bytes()
        ref = golden["cases"][c.name]["snapshot"]
        assert len(raw) == ref["bytes"] and hashlib.sha256(raw).hexdigest()[:32] == ref["sha"]
        # streamed in 1-plane chunks: same bytes
        monkeypatch.setattr(snapshot, "_CHUNK_BYTES", 1)
        p2 = tmp_path / "g2.dbtsdf"
        save_grid(g, p2)
        assert p2.read_bytes() == raw
        # load (chunked) -> identical grid, h_max/t_occ restored, byte-identical re-save
        g2 = load_grid(p2)
        assert (g2.h_max, g2.t_occ) == (params.h_max, params.t_occ)
        m, s_, h = g.download_range(0, c.dims[0])
        m2, s2, h2 = g2.download_range(0, c.dims[0])
        assert np.array_equal(m, m2) and np.array_equal(s_, s2) and np.array_equal(h, h2)
        p3 = tmp_path / "g3.dbtsdf"
        save_grid(g2, p3)
        assert p3.read_bytes() == raw

    def test_loaded_grid_integrates_like_reference(self, tmp_path):
        """A grid loaded from a snapshot carries no stamp certificates: the
        next scan must still match the oracle exactly."""
        from paper_2509_20081_b200 import load_grid, save_grid

        bank = build_kernel_bank(shadow_radius=2)
        rng = np.random.default_rng(5)
        pts1, pts2 = rng.uniform(1.15, 3.6, size=(300, 3)), rng.uniform(1.15, 3.6, size=(300, 3))
        g = new_grid((48, 48, 48), 0.1)
        integrate_frame(g, bank, ScanFrame(points=pts1, pose=np.eye(4)), IntegrationParams())
        save_grid(g, tmp_path / "a.dbtsdf")
        g2 = load_grid(tmp_path / "a.dbtsdf")
        integrate_frame(g2, bank, ScanFrame(points=pts1, pose=np.eye(4)), IntegrationParams())
        integrate_frame(g2, bank, ScanFrame(points=pts2, pose=np.eye(4)), IntegrationParams())
        og = oracle.OracleGrid((48, 48, 48), 0.1, (0, 0, 0))
        ob = oracle.OracleBank.from_bank(bank)
        for pts in (pts1, pts1, pts2):
            oracle.integrate_frame(og, ob, pts, np.eye(4))
        assert np.array_equal(g2.mask, og.mask) and np.array_equal(g2.sign, og.sign) and np.array_equal(g2.hits, og.hits)


class TestPendingShadowVisits:
    """Shadow visits are counted in the record's spare bytes and folded before
    reads (engine.cuh): overflow fold, parameter changes, partial reads."""

    def test_count_crossing_fold_threshold(self):
        bank = build_kernel_bank(shadow_radius=1)
        p = np.array([[2.45, 2.45, 2.45]])
        pm = np.repeat(p, 40_000, axis=0)            # 40k visits of the same cells in one launch
        sens = pm - np.array([1.0, 0.0, 0.0])
        for h_max, t in ((255, 2), (7, 3)):
            g = new_grid((48, 48, 48), 0.1)
            params = IntegrationParams(h_max=h_max, t_occ=t)
            integrate_points(g, bank, pm, sens, params)
            integrate_points(g, bank, pm[:3], sens[:3], params)  # more visits after the in-kernel fold
            og = oracle.OracleGrid((48, 48, 48), 0.1, (0, 0, 0))
            ob = oracle.OracleBank.from_bank(bank)
            oracle.integrate_points_map(og, ob, pm, sens, h_max=h_max, t_occ=t)
            oracle.integrate_points_map(og, ob, pm[:3], sens[:3], h_max=h_max, t_occ=t)
            assert np.array_equal(g.hits, og.hits) and np.array_equal(g.sign, og.sign)
            assert np.array_equal(g.mask, og.mask)

    def test_parameter_change_folds_pending_visits_first(self):
        bank = build_kernel_bank(shadow_radius=2)
        rng = np.random.default_rng(12)
        frames = [rng.uniform(1.15, 3.6, size=(400, 3)) for _ in range(4)]
        plist = [(7, 3), (7, 3), (200, 2), (2, 1)]
        g = new_grid((48, 48, 48), 0.1)
        og = oracle.OracleGrid((48, 48, 48), 0.1, (0, 0, 0))
        ob = oracle.OracleBank.from_bank(bank)
        for pts, (hm, t) in zip(frames, plist):
            integrate_frame(g, bank, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams(h_max=hm, t_occ=t))
            oracle.integrate_frame(og, ob, pts, np.eye(4), h_max=hm, t_occ=t)
        assert np.array_equal(g.hits, og.hits) and np.array_equal(g.sign, og.sign)

    def test_every_read_path_sees_folded_records(self):
        bank = build_kernel_bank(shadow_radius=1)
        rng = np.random.default_rng(13)
        pts = rng.uniform(1.15, 3.6, size=(500, 3))
        og = oracle.OracleGrid((48, 48, 48), 0.1, (0, 0, 0))
        oracle.integrate_frame(og, oracle.OracleBank.from_bank(bank), pts, np.eye(4))
        occ = og.sign == 0
        readers = [
            lambda g: np.array_equal(g.download_range(5, 30)[2], og.hits[5:30]),
            lambda g: G.grid_counts(g)[1] == int(occ.sum()),
            lambda g: np.array_equal(G.observed_array(g), ~((og.mask == G.FULL_MASK) & (og.hits == 0))),
            lambda g: np.array_equal(G.to_records(g)["hits"], og.hits.ravel(order="F")),
        ]
        for read in readers:
            g = new_grid((48, 48, 48), 0.1)
            integrate_frame(g, bank, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams())
            assert read(g)


class TestPinnedScans:
    """Scans in pinned host memory are read zero-copy by preprocessing, one
    device pointer per scan for batches (dbt_integrate_scans): same grid as
    the pageable path and the reference."""

    def test_pinned_batch_and_single_match_golden(self, golden):
        import ctypes

        c = next(c for c in CONFIG if c.name == "cfg2_scans0-2")
        L = _native.lib()
        bufs, pinned = [], []
        for p, _ in c.frames:
            p = np.ascontiguousarray(p, dtype=np.float32)
            buf = ctypes.c_void_p()
            _native.check(L.dbt_host_alloc(p.nbytes, ctypes.byref(buf)))
            arr = np.ctypeslib.as_array((ctypes.c_float * p.size).from_address(buf.value)).reshape(p.shape)
            arr[...] = p
            bufs.append(buf)
            pinned.append(arr)
        try:
            bank = build_kernel_bank(**c.bank)
            for batch in (True, False):
                g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 42)
                frames = [ScanFrame(points=a, pose=pose) for a, (_, pose) in zip(pinned, c.frames)]
                if batch:
                    sts = integrate_frames(g, bank, frames, IntegrationParams())
                else:
                    sts = [integrate_frame(g, bank, f, IntegrationParams()) for f in frames]
                stats = [[x.points_in, x.points_discarded, x.voxels_written] for x in sts]
                check(c, golden, g, stats, None, batch=batch)
        finally:
            for b in bufs:
                L.dbt_host_free(b)


class TestOrderIndependence:
    """The reference stamps in sorted centre order (integrator.py:266-284);
    the engine's updates commute, so any point order, any batching and any
    repetition gives the same grid."""

    def test_permuted_and_repeated_scan(self, golden):
        c = next(c for c in CONFIG if c.name == "cfg2_scans0-2")
        bank = build_kernel_bank(**c.bank)
        rng = np.random.default_rng(99)
        grids = []
        for variant in ("orig", "permuted", "split"):
            g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 42)
            for pts, pose in c.frames:
                if variant == "permuted":
                    pts = pts[rng.permutation(len(pts))]
                if variant == "split":  # the scan as 3 launches of uneven size
                    for part in np.split(pts, [5000, 41000]):
                        integrate_frame(g, bank, ScanFrame(points=part, pose=pose), IntegrationParams())
                else:
                    integrate_frame(g, bank, ScanFrame(points=pts, pose=pose), IntegrationParams())
            grids.append(g.download_range(0, c.dims[0]))
        ref = golden["cases"][c.name]
        for m, s_, h in grids:
            assert cases.sha(m) == ref["mask"] and cases.sha(s_) == ref["sign"] and cases.sha(h) == ref["hits"]


class TestLongSequenceSnapshots:
    """Reference acceptance C3 (test_acceptance.py:73-102: byte-identical
    snapshots for threads 1 vs 8 over a 200-frame sequence) for this engine:
    a 40-scan config-2 trajectory integrated scan by scan, in batches of 8 and
    in batches of 5 gives byte-identical DBTSDF01 snapshots."""

    def test_batching_invariance_bytes(self, tmp_path):
        import workloads

        from paper_2509_20081_b200 import save_grid

        w = workloads.get(2)
        frames = [ScanFrame(points=w.scan(k), pose=w.poses[k]) for k in range(40)]
        bank = build_kernel_bank(shadow_radius=w.shadow_radius)
        blobs = []
        for batch in (1, 8, 5):
            g = new_grid(w.dims, w.voxel_size, w.origin)
            g.release_host()
            for i in range(0, len(frames), batch):
                if batch == 1:
                    integrate_frame(g, bank, frames[i], IntegrationParams())
                else:
                    integrate_frames(g, bank, frames[i:i + batch], IntegrationParams())
            p = tmp_path / f"b{batch}.dbtsdf"
            save_grid(g, p)
            blobs.append(p.read_bytes())
        assert blobs[0] == blobs[1] == blobs[2]


class TestInterleavedSharding:
    """Interleaved x-blocks (dbt_grid_create_interleaved): each part stamps
    only its blocks; the parts reassemble to the reference grid. Both sweeps
    (culling for the standard kernel, generic for an asymmetric one)."""

    @staticmethod
    def _assemble(parts, dims):
        m = np.empty(dims, np.uint32)
        s_ = np.empty(dims, np.uint8)
        h = np.empty(dims, np.uint8)
        for g in parts:
            m[g.owned_x], s_[g.owned_x], h[g.owned_x] = g.mask, g.sign, g.hits
        return m, s_, h

    def test_parts_reassemble_to_reference(self, golden):
        from paper_2509_20081_b200.grid import VoxelGrid

        c = next(c for c in CONFIG if c.name == "cfg2_scans0-2")
        bank = build_kernel_bank(**c.bank)
        for w, P in ((16, 3), (64, 2), (7, 4)):
            parts = [VoxelGrid(c.dims, c.voxel_size, c.origin, interleave=(w, P, r)) for r in range(P)]
            assert sum(len(g.owned_x) for g in parts) == c.dims[0]
            for g in parts:
                g.release_host()
                for pts, pose in c.frames:
                    integrate_frame(g, bank, ScanFrame(points=pts, pose=pose), IntegrationParams())
            m, s_, h = self._assemble(parts, c.dims)
            ref = golden["cases"][c.name]
            assert cases.sha(m) == ref["mask"] and cases.sha(s_) == ref["sign"] and cases.sha(h) == ref["hits"]

    def test_generic_sweep_interleaved(self):
        import dataclasses

        from paper_2509_20081_b200.grid import VoxelGrid

        base = build_kernel_bank(shadow_radius=2)
        dk = base.distance_kernel.copy()
        dk[12:, 14:, :] &= np.uint32(0x3F)
        bank = dataclasses.replace(base, distance_kernel=dk, _device={})
        rng = np.random.default_rng(21)
        frames = [(rng.uniform(1.15, 3.6, size=(400, 3)), cases.yaw_pose(0.3 * k, (0.02 * k, 0, 0))) for k in range(2)]
        dims = (48, 48, 48)
        parts = [VoxelGrid(dims, 0.1, (0, 0, 0), interleave=(5, 3, r)) for r in range(3)]
        for g in parts:
            for pts, pose in frames:
                integrate_frame(g, bank, ScanFrame(points=pts, pose=pose), IntegrationParams())
        m, s_, h = self._assemble(parts, dims)
        og = oracle.OracleGrid(dims, 0.1, (0, 0, 0))
        ob = oracle.OracleBank.from_bank(bank)
        for pts, pose in frames:
            oracle.integrate_frame(og, ob, pts, pose)
        assert np.array_equal(m, og.mask) and np.array_equal(s_, og.sign) and np.array_equal(h, og.hits)


class TestSweepPaths:
    """The symmetric-kernel sweep (base-pair table) and the generic sweep
    (distinct-row table) must both reproduce the reference stamping."""

    def _run(self, bank, frames, dims=(48, 48, 48), first_return=False):
        g = new_grid(dims, 0.1)
        og = oracle.OracleGrid(dims, 0.1, (0, 0, 0))
        ob = oracle.OracleBank.from_bank(bank)
        for pts, pose in frames:
            st = integrate_frame(g, bank, ScanFrame(points=pts, pose=pose),
                                 IntegrationParams(first_return_per_voxel=first_return))
            ost = oracle.integrate_frame(og, ob, pts, pose, first_return=first_return)
            assert st.points_applied == ost.points_applied  # first-return winners / applied returns
        assert np.array_equal(g.mask, og.mask) and np.array_equal(g.sign, og.sign) and np.array_equal(g.hits, og.hits)

    @pytest.mark.parametrize("first_return", [False, True])
    def test_asymmetric_kernel_takes_generic_sweep(self, first_return):
        import dataclasses
        base = build_kernel_bank(shadow_radius=2)
        dk = base.distance_kernel.copy()
        # break the x/y symmetry: one octant gets shorter runs, one row longer
        dk[12:, 14:, :] &= np.uint32(0x3F)
        dk[3, 17, :] = np.uint32(0xFFFFF)
        bank = dataclasses.replace(base, distance_kernel=dk, _device={})
        rng = np.random.default_rng(8)
        frames = [(rng.uniform(1.15, 3.6, size=(400, 3)), cases.yaw_pose(0.4 * k, (0.02 * k, 0, 0))) for k in range(3)]
        self._run(bank, frames, first_return=first_return)

    @pytest.mark.parametrize("size", [3, 5, 9, 15, 21, 25, 27])
    def test_symmetric_kernel_sizes(self, size):
        bank = build_kernel_bank(size=size, shadow_radius=1)
        rng = np.random.default_rng(size)
        frames = [(rng.uniform(1.4, 3.4, size=(300, 3)), cases.yaw_pose(0.3 * k, (0.0, 0.01 * k, 0))) for k in range(2)]
        self._run(bank, frames)


class TestGridSemantics:
    def test_host_mirror_in_place_and_injected_fault(self):
        bank = build_kernel_bank(shadow_radius=3)
        g = new_grid((64, 64, 64), 0.1)
        m = g.mask  # reference semantics: arrays mutated in place
        rng = np.random.default_rng(1)
        pm, sens = cases._random_hits(rng, 50, (64, 64, 64), 0.1)
        integrate_points(g, bank, pm, sens, IntegrationParams())
        assert m is g.mask and np.any(m != G.FULL_MASK)
        pop = G.decode_distance(g.mask[32, 32, 32])
        g.mask[32, 32, 32] = G.run_mask(pop + 1 if pop < 32 else 0)  # corrupt through the mirror
        og = oracle.OracleGrid((64, 64, 64), 0.1, (0, 0, 0))
        oracle.integrate_points_map(og, oracle.OracleBank.from_bank(bank), pm, sens)
        diff = np.argwhere(G.popcount_array(g) != np.bitwise_count(og.mask))
        assert diff.tolist() == [[32, 32, 32]]

    def test_any_host_state_round_trips(self):
        """The device record is the reference's record: any mask (also non-run),
        sign byte and hit count survives upload/download unchanged."""
        rng = np.random.default_rng(9)
        g = new_grid((8, 9, 13), 0.1)
        m = rng.integers(0, 2**32, size=g.dims, dtype=np.uint64).astype(np.uint32)
        sg = rng.integers(0, 256, size=g.dims).astype(np.uint8)
        h = rng.integers(0, 256, size=g.dims).astype(np.uint8)
        g.mask[...], g.sign[...], g.hits[...] = m, sg, h
        g.release_host()
        mm, ss, hh = g.download_range(0, 8)
        assert np.array_equal(mm, m) and np.array_equal(ss, sg) and np.array_equal(hh, h)

    def test_readout_matches_reference_formulas(self):
        import workloads

        w = workloads.get(1)
        bank = build_kernel_bank(shadow_radius=w.shadow_radius)
        g = new_grid(w.dims, w.voxel_size, w.origin)
        integrate_frame(g, bank, ScanFrame(points=w.scan(0), pose=w.poses[0]), IntegrationParams(t_occ=1))
        field, obs = G.signed_distance_field(g)
        m, s, h = g.download_range(0, w.dims[0])
        # grid.py:161-175 on the downloaded arrays
        dist = np.bitwise_count(m).astype(np.int32).astype(np.float64) * g.voxel_size
        sigma = np.where(s == G.SIGN_OCCUPIED, -1.0, 1.0)
        ref_field = sigma * dist
        ref_obs = ~((m == G.FULL_MASK) & (h == 0))
        assert np.array_equal(obs, ref_obs) and np.array_equal(G.observed_array(g), ref_obs)
        assert np.array_equal(field.view(np.uint64), ref_field.view(np.uint64))  # incl. -0.0
        n_obs, n_occ = G.grid_counts(g)
        assert n_obs == int(ref_obs.sum()) and n_occ == int((s == 0).sum())
        idx = np.argwhere(ref_obs)[:: max(1, int(ref_obs.sum()) // 50)]
        for ix, iy, iz in idx[:50]:
            assert G.signed_distance(g, ix, iy, iz) == ref_field[ix, iy, iz]
        assert G.signed_distance(g, 0, 0, 0) is None
        with pytest.raises(IndexError):
            G.signed_distance(g, w.dims[0], 0, 0)

    def test_records_layout_and_round_trip(self):
        g = new_grid((3, 2, 2), 0.1)
        g.mask[1, 0, 0] = G.run_mask(5)
        g.mask[0, 1, 0] = G.run_mask(7)
        g.mask[0, 0, 1] = G.run_mask(9)
        rec = G.to_records(g)
        assert rec["mask"][1] == G.run_mask(5) and rec["mask"][3] == G.run_mask(7) and rec["mask"][6] == G.run_mask(9)
        assert np.all(rec["reserved"] == 0)
        rng = np.random.default_rng(7)
        g = new_grid((40, 33, 70), 0.25, origin=(1, 2, 3))
        g.mask[...] = np.array([G.run_mask(k) for k in rng.integers(0, 33, g.num_voxels)],
                               dtype=np.uint32).reshape(g.dims)
        g.hits[...] = rng.integers(0, 255, g.dims)
        g.sign[...] = rng.integers(0, 2, g.dims)
        rec = G.to_records(g)
        assert np.array_equal(rec["mask"], g.mask.ravel(order="F"))
        assert np.array_equal(rec["hits"], g.hits.ravel(order="F"))
        assert np.array_equal(rec["sign"], g.sign.ravel(order="F"))
        g2 = G.from_records(rec, g.dims, g.voxel_size, g.origin)
        assert G.grids_equal(g, g2)
        with pytest.raises(CorruptionError):
            G.from_records(rec[:-1], g.dims, g.voxel_size, g.origin)

    def test_gather_and_errors(self):
        g = new_grid((16, 16, 16), 0.1)
        m, s, h = G.gather(g, [(0, 0, 0), (15, 15, 15)])
        assert m.tolist() == [G.FULL_MASK] * 2 and s.tolist() == [1, 1] and h.tolist() == [0, 0]
        with pytest.raises(ConfigurationError):
            G.gather(g, [(16, 0, 0)])
        with pytest.raises(ConfigurationError):
            G.VoxelGrid((16, 16, 16), 0.1, (0, 0, 0), slab=(5, 3))

    def test_launch_counter_counts_engine_kernels(self):
        bank = build_kernel_bank(shadow_radius=1)
        g = new_grid((41, 41, 41), 0.1)
        n0 = _native.lib().dbt_launch_count()
        integrate_frame(g, bank, ScanFrame(points=np.full((10, 3), 2.05), pose=np.eye(4)), IntegrationParams())
        assert _native.lib().dbt_launch_count() - n0 >= 2  # prep (+ fused shadow), sweep


class TestExactVoxelsWritten:
    """DBT_FLAG_EXACT_WRITTEN: FrameStats.voxels_written equal to the
    reference's serial count (integrator.py:268-285), every FrameStats field
    exact, on every golden case with frames."""

    @staticmethod
    def run(c, **extra):
        bank = build_kernel_bank(**c.bank)
        g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 42)
        if c.init is not None:
            g.mask[...], g.sign[...], g.hits[...] = c.init
            g.release_host()
        params = IntegrationParams(**c.params, exact_voxels_written=True, **extra)
        frames = [ScanFrame(points=p, pose=pose) for p, pose in c.frames]
        sts = integrate_frames(g, bank, frames, params)
        return g, [[s.points_in, s.points_discarded, s.voxels_written] for s in sts]

    @pytest.mark.parametrize("c", [c for c in SMALL + CONFIG if c.frames], ids=lambda c: c.name)
    def test_stats_match_reference(self, c, golden):
        g, stats = self.run(c)
        ref = golden["cases"][c.name]
        assert stats == ref["stats"]
        m, s, h = g.download_range(0, c.dims[0])
        assert cases.sha(m) == ref["mask"] and cases.sha(s) == ref["sign"] and cases.sha(h) == ref["hits"]

    def test_repeated_scan_writes_nothing(self):
        c = next(c for c in SMALL if c.name == "frame500_default")
        bank = build_kernel_bank(**c.bank)
        g = new_grid(c.dims, c.voxel_size, c.origin)
        prm = IntegrationParams(exact_voxels_written=True)
        f = ScanFrame(points=c.frames[0][0], pose=c.frames[0][1])
        first = integrate_frame(g, bank, f, prm)
        again = integrate_frame(g, bank, f, prm)
        assert first.voxels_written > 0 and again.voxels_written == 0

    def test_env_default(self, monkeypatch):
        monkeypatch.setenv("DBT_EXACT_VOXELS_WRITTEN", "1")
        assert IntegrationParams().exact_voxels_written
        monkeypatch.delenv("DBT_EXACT_VOXELS_WRITTEN")
        assert not IntegrationParams().exact_voxels_written

    def test_sharded_grid_rejected(self):
        from paper_2509_20081_b200.grid import VoxelGrid

        c = next(c for c in SMALL if c.name == "frame500_default")
        g = VoxelGrid(c.dims, c.voxel_size, c.origin, slab=(0, 20))
        with pytest.raises(ConfigurationError):
            integrate_frame(g, build_kernel_bank(**c.bank), ScanFrame(points=c.frames[0][0], pose=c.frames[0][1]),
                            IntegrationParams(exact_voxels_written=True))


class TestReplicaMerge:
    """Data-parallel replicas (sharded.ReplicatedGrid): each replica
    integrates a subset of the scans; dbt_replica_pack -> MIN/MIN/SUM across
    replicas (torch ops standing in for the NCCL all-reduces) ->
    dbt_replica_apply must give every replica the reference's final grid."""

    @staticmethod
    def merge(grids):
        import ctypes

        import torch

        L = _native.lib()
        n = int(np.prod(grids[0].dims))
        packs = []
        for g in grids:
            mk = torch.empty(n, dtype=torch.uint8, device="cuda")
            sg = torch.empty(n, dtype=torch.uint8, device="cuda")
            dl = torch.empty(n, dtype=torch.float16, device="cuda")
            _native.check(L.dbt_replica_pack(g.handle, ctypes.c_void_p(mk.data_ptr()), ctypes.c_void_p(sg.data_ptr()),
                                             ctypes.c_void_p(dl.data_ptr()), None))
            packs.append((mk, sg, dl))
        torch.cuda.synchronize()
        mk = torch.stack([p[0] for p in packs]).amin(0).contiguous()
        sg = torch.stack([p[1] for p in packs]).amin(0).contiguous()
        dl = torch.stack([p[2] for p in packs]).sum(0).contiguous()  # float16, like NCCL
        torch.cuda.synchronize()  # apply runs on the grids' own streams
        return mk, sg, dl

    @staticmethod
    def apply(grids, red, params):
        import ctypes

        import torch

        L = _native.lib()
        mk, sg, dl = red
        for g in grids:
            _native.check(L.dbt_replica_apply(g.handle, ctypes.c_void_p(mk.data_ptr()), ctypes.c_void_p(sg.data_ptr()),
                                              ctypes.c_void_p(dl.data_ptr()), params.h_max, params.t_occ, None))
            g.synchronize()
        torch.cuda.synchronize()

    @staticmethod
    def merge_apply_sparse(grids, params):
        """The sparse protocol (dbt_replica_dirty/select/pack_bricks/
        apply_bricks) with torch reductions standing in for NCCL."""
        import ctypes

        import torch

        L = _native.lib()
        nb, reach = ctypes.c_int64(), ctypes.c_int32()
        flags, reaches = [], []
        for g in grids:
            _native.check(L.dbt_replica_bricks(g.handle, ctypes.byref(nb), ctypes.byref(reach)))
            f = torch.empty(int(nb.value), dtype=torch.uint8, device="cuda")
            _native.check(L.dbt_replica_dirty(g.handle, ctypes.c_void_p(f.data_ptr()), None))
            g.synchronize()
            flags.append(f)
            reaches.append(reach.value)
        fl = torch.stack(flags).amax(0).contiguous()
        torch.cuda.synchronize()
        packs, nsel = [], []
        for g in grids:
            n = ctypes.c_int64()
            _native.check(L.dbt_replica_select(g.handle, ctypes.c_void_p(fl.data_ptr()), max(reaches),
                                               ctypes.byref(n), None))
            nsel.append(n.value)
            ms = torch.empty(2 * 4096 * n.value, dtype=torch.uint8, device="cuda")
            dl = torch.empty(4096 * n.value, dtype=torch.float16, device="cuda")
            _native.check(L.dbt_replica_pack_bricks(g.handle, ctypes.c_void_p(ms.data_ptr()),
                                                    ctypes.c_void_p(dl.data_ptr()), None))
            g.synchronize()
            packs.append((ms, dl))
        assert len(set(nsel)) == 1
        ms = torch.stack([p[0] for p in packs]).amin(0).contiguous()
        dl = torch.stack([p[1] for p in packs]).sum(0).contiguous()
        torch.cuda.synchronize()
        for g in grids:
            _native.check(L.dbt_replica_apply_bricks(g.handle, ctypes.c_void_p(ms.data_ptr()),
                                                     ctypes.c_void_p(dl.data_ptr()), params.h_max, params.t_occ, None))
            g.synchronize()
        torch.cuda.synchronize()
        return nsel[0]

    def run(self, c, n_rep, intervals=1, sparse=False):
        bank = build_kernel_bank(**c.bank)
        grids = []
        for _ in range(n_rep):
            g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 42)
            if c.init is not None:
                g.mask[...], g.sign[...], g.hits[...] = c.init
                g.release_host()
            _native.check(_native.lib().dbt_replica_mark(g.handle))
            grids.append(g)
        params = IntegrationParams(**c.params)
        frames = [ScanFrame(points=p, pose=pose) for p, pose in c.frames]
        chunks = np.array_split(np.arange(len(frames)), intervals)
        for chunk in chunks:
            for j, k in enumerate(chunk):
                integrate_frame(grids[j % n_rep], bank, frames[k], params)
            if sparse:
                self.merge_apply_sparse(grids, params)
            else:
                self.apply(grids, self.merge(grids), params)
        return grids

    @pytest.mark.parametrize("name,n_rep,intervals", [
        ("cfg2_scans0-2", 2, 1), ("cfg2_scans0-2", 3, 1), ("yaw_frames_f32", 3, 2), ("yaw_frames_f32", 4, 1),
        ("nonfresh_hemisphere_h7_t3", 2, 1), ("nonfresh_cone_h200_t2", 3, 1), ("nonfresh_hemisphere_h255_t1", 2, 2),
        ("arbitrary_state", 2, 1)])
    def test_merged_replicas_match_reference(self, name, n_rep, intervals, golden):
        c = next(c for c in SMALL + CONFIG if c.name == name)
        ref = golden["cases"][name]
        for g in self.run(c, n_rep, intervals):
            m, s, h = g.download_range(0, c.dims[0])
            assert cases.sha(m) == ref["mask"], "mask differs from the reference"
            assert cases.sha(s) == ref["sign"], "sign differs from the reference"
            assert cases.sha(h) == ref["hits"], "hits differ from the reference"

    @pytest.mark.parametrize("name,n_rep,intervals", [
        ("cfg2_scans0-2", 2, 1), ("cfg2_scans0-2", 3, 2), ("yaw_frames_f32", 3, 2),
        ("nonfresh_hemisphere_h7_t3", 2, 1), ("nonfresh_cone_h200_t2", 3, 1), ("nonfresh_hemisphere_h255_t1", 2, 2),
        ("arbitrary_state", 2, 1), ("edge_returns", 2, 1)])
    def test_sparse_merge_matches_reference(self, name, n_rep, intervals, golden):
        c = next(c for c in SMALL + CONFIG if c.name == name)
        ref = golden["cases"][name]
        for g in self.run(c, n_rep, intervals, sparse=True):
            m, s, h = g.download_range(0, c.dims[0])
            assert cases.sha(m) == ref["mask"], "mask differs from the reference"
            assert cases.sha(s) == ref["sign"], "sign differs from the reference"
            assert cases.sha(h) == ref["hits"], "hits differ from the reference"

    def test_sparse_merge_moves_only_touched_bricks(self):
        """One return in a corner of a 256^3 grid: the merge selects the
        3^3 bricks around its brick (R = 10 -> one brick of dilation), not
        the 4096 bricks of the grid; a merge with no work selects none."""
        bank = build_kernel_bank()
        g = new_grid((256, 256, 256), 0.1)
        _native.check(_native.lib().dbt_replica_mark(g.handle))
        assert self.merge_apply_sparse([g], IntegrationParams()) == 0
        pts = np.array([[2.45, 2.45, 2.45]])  # voxel (24, 24, 24): brick (1, 1, 1)
        integrate_frame(g, bank, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams())
        assert self.merge_apply_sparse([g], IntegrationParams()) == 27
        assert self.merge_apply_sparse([g], IntegrationParams()) == 0

    def test_merge_without_work_is_identity(self, golden):
        c = next(c for c in SMALL if c.name == "arbitrary_state")
        g = new_grid(c.dims, c.voxel_size, c.origin)
        g.mask[...], g.sign[...], g.hits[...] = c.init
        g.release_host()
        _native.check(_native.lib().dbt_replica_mark(g.handle))
        self.apply([g], self.merge([g]), IntegrationParams(h_max=250, t_occ=4))
        m, s, h = g.download_range(0, c.dims[0])
        assert np.array_equal(m, c.init[0]) and np.array_equal(s, c.init[1]) and np.array_equal(h, c.init[2])

    def test_pack_needs_mark(self):
        import ctypes

        g = new_grid((16, 16, 16), 0.1)
        with pytest.raises(ConfigurationError):
            _native.check(_native.lib().dbt_replica_pack(g.handle, ctypes.c_void_p(0), ctypes.c_void_p(0),
                                                         ctypes.c_void_p(0), None))


@pytest.mark.parametrize("shadow_radius", [1, 2])
def test_bin_fallback_counted_per_scan(shadow_radius):
    """A ray component below 2^-1020 takes SVML's scalar helper, which is not
    restated: the engine bins that ray with CUDA's atan2 and counts it in the
    scan's bin_fallbacks. r_s = 1 (|S| = 4) bins in shadow_bin_kernel, r_s = 2
    (|S| = 17) in prep; a two-scan launch attributes the count to its scan.
    The azimuth of (2, 1e-308) is bin 0 either way, so the grid still equals
    the oracle's."""
    bank = build_kernel_bank(shadow_radius=shadow_radius)
    dims, vs, org = (64, 64, 64), 0.1, (-3.2, -3.2, -3.2)
    pts_a = np.array([[2.0, 0.5, 0.3], [1.0, -1.0, 0.5]])
    pts_b = np.array([[2.0, 1e-308, 0.3], [-1.5, 0.7, -0.2]])
    eye = np.eye(4)
    g = new_grid(dims, vs, org)
    sts = integrate_frames(g, bank, [ScanFrame(points=pts_a, pose=eye), ScanFrame(points=pts_b, pose=eye)],
                           IntegrationParams())
    assert [s.bin_fallbacks for s in sts] == [0, 1]
    assert [s.points_in - s.points_discarded for s in sts] == [2, 2]
    st = integrate_frame(new_grid(dims, vs, org), bank, ScanFrame(points=pts_b, pose=eye), IntegrationParams())
    assert st.bin_fallbacks == 1
    og = oracle.OracleGrid(dims, vs, org)
    ob = oracle.OracleBank.from_bank(bank)
    oracle.integrate_frame(og, ob, pts_a, eye)
    oracle.integrate_frame(og, ob, pts_b, eye)
    m, s, h = g.download_range(0, dims[0])
    assert np.array_equal(m, og.mask) and np.array_equal(s, og.sign) and np.array_equal(h, og.hits)


class TestAsyncFrames:
    """integrate_frame_async (dbt_integrate_frame_async / dbt_frame_wait):
    pipelined calls give the same grid and FrameStats as synchronous ones."""

    @pytest.mark.parametrize("name", ["cfg2_scans0-2", "yaw_frames_f32", "nonfresh_cone_h200_t2",
                                      "frame500_first_return", "frame500_downsample3"])
    def test_async_matches_reference(self, name, golden):
        from paper_2509_20081_b200 import integrate_frame_async

        c = next(c for c in SMALL + CONFIG if c.name == name)
        ref = golden["cases"][name]
        bank = build_kernel_bank(**c.bank)
        g = new_grid(c.dims, c.voxel_size, c.origin)
        if c.init is not None:
            g.mask[...], g.sign[...], g.hits[...] = c.init
        params = IntegrationParams(**c.params)
        futs = [integrate_frame_async(g, bank, ScanFrame(points=p, pose=pose), params) for p, pose in c.frames]
        sts = [f.result() for f in futs]
        assert [[s.points_in, s.points_discarded] for s in sts] == [r[:2] for r in ref["stats"]]
        m, s, h = g.download_range(0, c.dims[0])
        assert (cases.sha(m), cases.sha(s), cases.sha(h)) == (ref["mask"], ref["sign"], ref["hits"])

    def test_trajectory_pipelined_equals_sync(self):
        """40 config-2 scans, at most 2 outstanding, against synchronous
        calls: identical grids and per-scan counts."""
        import workloads
        from paper_2509_20081_b200 import integrate_frame_async

        w = workloads.get(2)
        bank = build_kernel_bank(shadow_radius=w.shadow_radius)
        scans = [w.scan(k) for k in range(40)]
        a, b = new_grid(w.dims, w.voxel_size, w.origin), new_grid(w.dims, w.voxel_size, w.origin)
        sync = [integrate_frame(a, bank, ScanFrame(points=s, pose=w.poses[k]), IntegrationParams())
                for k, s in enumerate(scans)]
        pend, got = [], []
        for k, s in enumerate(scans):
            pend.append(integrate_frame_async(b, bank, ScanFrame(points=s, pose=w.poses[k]), IntegrationParams()))
            if len(pend) > 2:
                got.append(pend.pop(0).result())
        got += [f.result() for f in pend]
        assert [(x.points_in, x.points_discarded) for x in got] == [(x.points_in, x.points_discarded) for x in sync]
        for x0, x1 in ((0, 211), (211, w.dims[0])):
            ma, sa, ha = a.download_range(x0, x1)
            mb, sb, hb = b.download_range(x0, x1)
            assert np.array_equal(ma, mb) and np.array_equal(sa, sb) and np.array_equal(ha, hb)

    def test_pageable_staging_equals_direct_copy(self, monkeypatch):
        """Plain numpy scans of >= 64 KB go through the slot's pinned staging
        (host copy pool); $DBT_NO_HOST_STAGE=1 hands the pageable pointer to
        cudaMemcpyAsync instead. Same grids, same counts."""
        import workloads
        from paper_2509_20081_b200 import integrate_frame_async

        w = workloads.get(2)
        bank = build_kernel_bank(shadow_radius=w.shadow_radius)
        scans = [w.scan(k) for k in range(6)]
        assert min(s.nbytes for s in scans) >= (64 << 10)
        grids, stats = [], []
        for direct in (False, True):
            if direct:
                monkeypatch.setenv("DBT_NO_HOST_STAGE", "1")
            g = new_grid(w.dims, w.voxel_size, w.origin)
            futs = [integrate_frame_async(g, bank, ScanFrame(points=s, pose=w.poses[k]), IntegrationParams())
                    for k, s in enumerate(scans[:3])]  # at most 4 calls outstanding
            futs.append(integrate_frame_async(g, bank, ScanFrame(points=scans[3], pose=w.poses[3]), IntegrationParams()))
            stats.append([(f.result().points_in, f.result().points_discarded) for f in futs])
            grids.append(g)
        assert stats[0] == stats[1]
        for x0, x1 in ((0, 211), (211, w.dims[0])):
            a = grids[0].download_range(x0, x1)
            b = grids[1].download_range(x0, x1)
            assert all(np.array_equal(x, y) for x, y in zip(a, b))

    def test_async_exact_voxels_written(self, golden):
        from paper_2509_20081_b200 import integrate_frame_async

        c = next(c for c in SMALL + CONFIG if c.name == "cfg2_scans0-2")
        ref = golden["cases"][c.name]
        bank = build_kernel_bank(**c.bank)
        g = new_grid(c.dims, c.voxel_size, c.origin)
        params = IntegrationParams(exact_voxels_written=True, **c.params)
        futs = [integrate_frame_async(g, bank, ScanFrame(points=p, pose=pose), params) for p, pose in c.frames]
        assert [[f.result().points_in, f.result().points_discarded, f.result().voxels_written] for f in futs] == \
            ref["stats"]

    def test_expired_ticket_and_result_idempotent(self):
        from paper_2509_20081_b200 import integrate_frame_async

        bank = build_kernel_bank()
        g = new_grid((48, 48, 48), 0.1)
        pts = np.random.default_rng(0).uniform(1.2, 3.6, size=(300, 3))
        futs = [integrate_frame_async(g, bank, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams())
                for _ in range(6)]
        with pytest.raises(ConfigurationError):
            futs[0].result()  # 5 calls issued since: its slot was reused
        r = futs[5].result()
        assert r.points_in == 300 and futs[5].result() is r
