"""Pin the oracle against outputs of the reference itself (tests/golden).

CPU only. For every parity case the seeded inputs are regenerated (their
hash must match the one recorded when the reference ran), the oracle
integrates them and the sha256 of the final mask/sign/hits plus every
FrameStats field (points_in, points_discarded, voxels_written) must equal the
reference's. Also pins the oracle's bank tables and binning.
"""

import numpy as np
import pytest

import cases
import oracle
from oracle import prep

SMALL = cases.small_cases()
CONFIG = cases.config_cases(include_slow=True)


def run_oracle(c: cases.Case, c_prep=False, threads=4):
    ob = oracle.OracleBank.build(**c.bank)
    g = oracle.OracleGrid(c.dims, c.voxel_size, c.origin)
    if c.init is not None:
        g.mask[...] = c.init[0]
        g.sign[...] = c.init[1]
        g.hits[...] = c.init[2]
    p = dict(h_max=255, t_occ=2, downsample=1, first_return_per_voxel=False)
    p.update(c.params)
    stats = []
    for pts, pose in c.frames:
        st = oracle.integrate_frame(g, ob, pts, pose, h_max=p["h_max"], t_occ=p["t_occ"], downsample=p["downsample"],
                                    first_return=p["first_return_per_voxel"], threads=threads, c_prep=c_prep)
        stats.append([st.points_in, st.points_discarded, st.voxels_written])
    applied = None
    if c.hits is not None:
        applied = int(oracle.integrate_points_map(g, ob, c.hits[0], c.hits[1], p["h_max"], p["t_occ"]).sum())
    return g, stats, applied


def check(c, gold, g, stats, applied):
    ref = gold["cases"][c.name]
    assert ref["input"] == c.input_hash(), "generator drift: inputs differ from the reference run"
    assert stats == ref["stats"]
    assert applied == ref["applied"]
    assert cases.sha(g.mask) == ref["mask"]
    assert cases.sha(g.sign) == ref["sign"]
    assert cases.sha(g.hits) == ref["hits"]


@pytest.mark.parametrize("c", SMALL, ids=[c.name for c in SMALL])
def test_oracle_matches_reference_small(c, golden):
    check(c, golden, *run_oracle(c))


@pytest.mark.parametrize("c", CONFIG, ids=[c.name for c in CONFIG])
def test_oracle_matches_reference_configs(c, golden):
    check(c, golden, *run_oracle(c, threads=8))


@pytest.mark.parametrize("name", ["cfg1_scan0", "cfg2_scans0-2"])
def test_c_preprocessing_matches_reference(name, golden):
    """The all-C oracle (libm transcendentals) used for the timed CPU baseline
    agrees with the reference on the config inputs (no knife-edge returns)."""
    c = next(x for x in CONFIG if x.name == name)
    check(c, golden, *run_oracle(c, c_prep=True, threads=8))


@pytest.mark.parametrize("spec", cases.bank_specs(), ids=cases.bank_key)
def test_oracle_bank_tables(spec, golden):
    ob = oracle.OracleBank.build(**spec)
    ref = golden["banks"][cases.bank_key(spec)]
    assert cases.sha(ob.distance_kernel) == ref["distance_kernel"]
    counts = np.diff(ob.shadow_start)
    assert cases.sha(counts.astype(np.int64)) == ref["shadow_counts"]
    assert cases.sha(ob.shadow_xyz.astype(np.int64)) == ref["shadow_offsets"]


@pytest.mark.parametrize("name", list(cases.bin_dir_sets()))
def test_oracle_bins(name, golden):
    dirs = cases.bin_dir_sets()[name]
    ref = golden["bins"][name]
    assert cases.sha(dirs) == ref["input"]
    b_a, b_e = prep.bin_index_array(dirs, 40, 40)
    assert cases.sha(b_a.astype(np.int64)) == ref["b_a"]
    assert cases.sha(b_e.astype(np.int64)) == ref["b_e"]
    # the libm restatement agrees away from knife edges (these sets have none)
    L = oracle.lib()
    d = np.ascontiguousarray(dirs)
    ca = np.empty(len(d), np.int64)
    ce = np.empty(len(d), np.int64)
    L.orc_bin_index_array(d.ctypes.data_as(oracle._dp), len(d), 40, 40, ca.ctypes.data_as(oracle._i64p),
                          ce.ctypes.data_as(oracle._i64p))
    assert np.array_equal(ca, b_a) and np.array_equal(ce, b_e)


def test_slab_stamping_equals_whole_grid():
    """Oracle slab stamping (used by the multi-rank tests) reassembles to the
    whole-grid result."""
    c = SMALL[0]
    full, _, _ = run_oracle(c, threads=1)
    ob = oracle.OracleBank.build(**c.bank)
    pts, pose = c.frames[0]
    parts = []
    for x0, x1 in ((0, 13), (13, 30), (30, 41)):
        g = oracle.OracleGrid(c.dims, c.voxel_size, c.origin, slab=(x0, x1))
        oracle.integrate_frame(g, ob, pts, pose)
        parts.append(g)
    assert np.array_equal(np.concatenate([p.mask for p in parts]), full.mask)
    assert np.array_equal(np.concatenate([p.hits for p in parts]), full.hits)
    assert np.array_equal(np.concatenate([p.sign for p in parts]), full.sign)
