"""Host-side logic of the drop-in API (CPU only, no device calls): kernel
bank tables vs the reference's (golden hashes), scalar binning known answers
(reference test_kernels.py:18-37), parameter / pose validation
(test_integrator.py:32-90), grid helpers (test_grid.py) and error mapping."""

import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import cases
from paper_2509_20081_b200 import errors
from paper_2509_20081_b200.errors import ConfigurationError, CorruptionError, ResourceError
from paper_2509_20081_b200.grid import (
    FULL_MASK, VOXEL_DTYPE, decode_distance, is_run_mask, new_grid, popcount_array, run_mask)
from paper_2509_20081_b200.integrator import IntegrationParams, ScanFrame, motion_compensate
from paper_2509_20081_b200.kernels import (
    bin_direction, bin_index, build_kernel_bank, build_shadow_mask, default_shadow_radius, make_distance_mask)
from paper_2509_20081_b200.transforms import interpolate_pose_yaw, make_pose


@pytest.mark.parametrize("spec", cases.bank_specs(), ids=cases.bank_key)
def test_bank_matches_reference(spec, golden):
    assert cases.bank_hashes(build_kernel_bank(**spec)) == golden["banks"][cases.bank_key(spec)]


class TestBinIndex:
    def test_known_answers(self):
        assert bin_index((1, 0, 0), 40, 40) == (0, 20)
        assert bin_index((0, 0, 1), 40, 40) == (0, 39)
        assert bin_index((0, -1, 0), 40, 40) == (30, 20)

    def test_zero_vector_rejected(self):
        with pytest.raises(ConfigurationError):
            bin_index((0, 0, 0), 40, 40)

    def test_round_trip_all_bins(self):
        for b_a in range(40):
            for b_e in range(40):
                assert bin_index(bin_direction(b_a, b_e, 40, 40), 40, 40) == (b_a, b_e)

    def test_bin_centre_angles(self):
        v = bin_direction(0, 20, 40, 40)
        assert math.degrees(math.atan2(v[1], v[0])) == pytest.approx(4.5)
        assert math.degrees(math.asin(v[2])) == pytest.approx(2.25)

    def test_out_of_range(self):
        with pytest.raises(ConfigurationError):
            bin_direction(40, 0, 40, 40)


class TestKernels:
    def test_distance_masks(self):
        assert make_distance_mask((0, 0, 0)) == 0
        assert make_distance_mask((1, 0, 0)) == 0x1
        assert make_distance_mask((1, 2, 0)) == 0x7
        base = make_distance_mask((1, 2, 3))
        for off in [(3, 2, 1), (-1, 2, -3), (2, -3, 1), (-3, -2, -1)]:
            assert make_distance_mask(off) == base

    def test_shadow_sets(self):
        got = {tuple(o) for o in build_shadow_mask((1, 0, 0), 1, "hemisphere")}
        assert got == {(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)}
        for model in ("hemisphere", "cone"):
            assert [tuple(o) for o in build_shadow_mask((0, 0, 1), 0, model)] == [(0, 0, 0)]
        hemi = {tuple(o) for o in build_shadow_mask((1, 0, 0), 2, "hemisphere")}
        cone = {tuple(o) for o in build_shadow_mask((1, 0, 0), 2, "cone", 45.0)}
        assert cone <= hemi and (0, 0, 0) in cone
        with pytest.raises(ConfigurationError):
            build_shadow_mask((1, 0, 0), 11, "hemisphere")

    def test_bank_shape_and_errors(self):
        bank = build_kernel_bank(shadow_radius=3)
        assert bank.distance_kernel.shape == (21, 21, 21)
        assert len(bank.shadow_offsets) == 1600
        assert np.bitwise_count(bank.distance_kernel).max() == 18
        with pytest.raises(ConfigurationError):
            build_kernel_bank(size=20)
        with pytest.raises(ConfigurationError):
            build_kernel_bank(shadow_model="pyramid")

    def test_shadow_radius_heuristic(self):
        assert default_shadow_radius(0.05) == 1
        assert default_shadow_radius(0.1) == 1
        assert default_shadow_radius(0.02) == 2  # banker's rounding of 2.5
        assert default_shadow_radius(0.01) == 5
        assert default_shadow_radius(0.001) == 10


class TestParamsAndFrames:
    def test_params(self):
        with pytest.raises(ConfigurationError):
            IntegrationParams(h_max=3, t_occ=5)
        with pytest.raises(ConfigurationError):
            IntegrationParams(t_occ=0)
        with pytest.raises(ConfigurationError):
            IntegrationParams(compensation="pitch")
        with pytest.raises(ConfigurationError):
            IntegrationParams(downsample=0)
        p = IntegrationParams(h_max=9, t_occ=3, downsample=2, first_return_per_voxel=True).native()
        assert (p.h_max, p.t_occ, p.downsample, p.first_return) == (9, 3, 2, 1)

    def test_scanframe(self):
        bad = np.eye(4)
        bad[0, 0] = 2.0
        with pytest.raises(ConfigurationError):
            ScanFrame(points=np.zeros((1, 3)), pose=bad)
        with pytest.raises(ConfigurationError):
            ScanFrame(points=np.zeros((3, 3)), pose=np.eye(4), timestamps=[0.0, 1.0])
        f32 = np.arange(12, dtype=np.float32).reshape(4, 3)
        s = ScanFrame(points=f32, pose=np.eye(4))
        assert s.points.dtype == np.float64 and np.array_equal(s.points, f32.astype(np.float64))
        arr, code = s.device_payload()
        assert arr.dtype == np.float32 and code == 0
        s.points = np.ones((2, 3))
        assert s.device_payload()[0].dtype == np.float64 and s.n_points == 2

    def test_motion_compensation(self):
        scan = ScanFrame(points=np.random.default_rng(0).normal(size=(10, 3)), pose=np.eye(4))
        assert motion_compensate(scan, "none") is scan
        pose = make_pose(Rotation.from_euler("z", 0.3), (1, 2, 3))
        pts = np.random.default_rng(1).normal(size=(20, 3))
        s = ScanFrame(points=pts, pose=pose, prev_pose=pose.copy())
        for mode in ("yaw", "se3"):
            assert np.allclose(motion_compensate(s, mode).points, pts, atol=1e-12)
        prev = make_pose(Rotation.identity(), (0, 0, 0))
        cur = make_pose(Rotation.identity(), (1, 0, 0))
        pts = np.array([[2.0, 0.0, 0.0], [5.0, 1.0, -1.0]])
        s = ScanFrame(points=pts, pose=cur, prev_pose=prev, timestamps=[0.5, 0.5])
        for mode in ("yaw", "se3"):
            assert np.allclose(motion_compensate(s, mode).points, pts - [0.5, 0.0, 0.0])
        out = motion_compensate(ScanFrame(points=np.zeros((3, 3)), pose=cur, prev_pose=prev), "se3")
        assert np.allclose(out.points[:, 0], [-1.0, -0.5, 0.0])
        with pytest.raises(ConfigurationError):
            motion_compensate(ScanFrame(points=np.zeros((2, 3)), pose=np.eye(4)), "se3")

    def test_check_rotation_decisions_match_numpy_formulation(self):
        """The float fast path decides exactly like np.allclose/np.isclose
        (transforms.py:30-37) on random near-rotations, reflections and
        non-finite input."""
        from paper_2509_20081_b200.transforms import _check_rotation_numpy, check_rotation

        rng = np.random.default_rng(0)

        def decide(f):
            try:
                f()
                return "ok"
            except ConfigurationError as e:
                return str(e)

        mats = []
        for k in range(3000):
            R = Rotation.random(random_state=k).as_matrix()
            R = R + rng.normal(size=(3, 3)) * 10.0 ** rng.uniform(-16, -3) * (rng.random() < 0.7)
            mats.append(-R if rng.random() < 0.1 else R)
        mats += [np.full((3, 3), np.nan), np.diag([np.inf, 1, 1]), np.eye(3) * (1 + 1e-5)]
        for R in mats:
            T = np.eye(4)
            T[:3, :3] = R
            assert decide(lambda: check_rotation(T)) == decide(lambda: _check_rotation_numpy(R, 1e-9))

    def test_yaw_interpolation(self):
        a = make_pose(Rotation.from_euler("z", 0.1), (0, 0, 0))
        b = make_pose(Rotation.from_euler("z", 0.5), (2, 0, 0))
        m = interpolate_pose_yaw(a, b, 0.5)
        assert np.allclose(m[:3, 3], [1, 0, 0])
        assert Rotation.from_matrix(m[:3, :3]).as_euler("zyx")[0] == pytest.approx(0.3)


class TestGridHelpers:
    def test_new_grid_validation_is_host_side(self):
        with pytest.raises(ConfigurationError):
            new_grid((0, 4, 4), 0.1)
        with pytest.raises(ConfigurationError):
            new_grid((4, 4, 4), 0.0)
        with pytest.raises(ResourceError):
            new_grid((100, 100, 100), 0.1, memory_cap=1_000_000)

    def test_decode(self):
        assert decode_distance(0) == 0 and decode_distance(FULL_MASK) == 32 and decode_distance(7) == 3
        assert not is_run_mask(0b101)
        with pytest.raises(CorruptionError):
            decode_distance(0b101)
        for k1 in range(33):
            for k2 in range(33):
                assert decode_distance(run_mask(k1) & run_mask(k2)) == min(k1, k2)
        with pytest.raises(ConfigurationError):
            run_mask(33)

    def test_popcount_host_array_and_record_dtype(self):
        m = np.array([0, 1, 3, FULL_MASK], dtype=np.uint32)
        assert popcount_array(m).tolist() == [0, 1, 2, 32]
        assert VOXEL_DTYPE.itemsize == 8

    def test_error_codes_follow_cli_exit_codes(self):
        # cli.py:34-40
        assert errors.CODE_TO_ERROR[2] is ConfigurationError
        assert errors.CODE_TO_ERROR[3] is errors.FormatError
        assert errors.CODE_TO_ERROR[4] is CorruptionError
        assert errors.CODE_TO_ERROR[5] is errors.EvaluationError
        assert errors.CODE_TO_ERROR[6] is ResourceError


class TestSnapshotHeader:
    """DBTSDF01 validation happens on the host before any device work
    (io.py:462-477; reference test_io.py snapshot cases)."""

    def _write(self, p, body):
        p.write_bytes(body)
        return p

    def test_header_layout(self):
        from paper_2509_20081_b200 import snapshot

        assert snapshot.SNAPSHOT_MAGIC == b"DBTSDF01" and snapshot._HEADER.size == 52

    def test_wrong_magic(self, tmp_path):
        from paper_2509_20081_b200 import load_grid

        with pytest.raises(CorruptionError):
            load_grid(self._write(tmp_path / "bad.dbtsdf", b"NOTADUMP" + b"\x00" * 64))

    def test_truncated_header(self, tmp_path):
        from paper_2509_20081_b200 import load_grid

        with pytest.raises(CorruptionError):
            load_grid(self._write(tmp_path / "t.dbtsdf", b"DBTSDF01" + b"\x00" * 20))

    def test_zero_dims_and_short_payload(self, tmp_path):
        from paper_2509_20081_b200 import load_grid, snapshot

        head = snapshot._HEADER.pack(0, 2, 2, 0.1, 0.0, 0.0, 0.0, 255, 2)
        with pytest.raises(CorruptionError):
            load_grid(self._write(tmp_path / "z.dbtsdf", b"DBTSDF01" + head + b"\x00" * 64))
        head = snapshot._HEADER.pack(4, 4, 4, 0.1, 0.0, 0.0, 0.0, 255, 2)
        with pytest.raises(CorruptionError):
            load_grid(self._write(tmp_path / "s.dbtsdf", b"DBTSDF01" + head + b"\x00" * (64 * 8 - 16)))
