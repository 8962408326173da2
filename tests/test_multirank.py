"""Multi-rank slab sharding on CPU: world_size 2 over gloo.

Exercises the same host logic the NCCL path uses (paper_2509_20081_b200/
sharded.py): slab partition, the broadcast protocol (header, per-scan
counts/poses, raw float32 payload), per-rank preprocessing against the global
dims, slab-restricted stamping (here the oracle's slab stamping stands in for
the device engine, which the GPU tests cover per slab) and the stats
all-reduce. The gathered slabs must reproduce the reference's golden grid and
FrameStats for config 1 and the 3-scan config-2 case.
"""

import os
import socket
import sys

import numpy as np
import pytest

import cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case_name, out_path, interleave=0):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import cases as C
    import oracle
    from paper_2509_20081_b200 import sharded
    from paper_2509_20081_b200.integrator import FrameStats

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = next(x for x in C.config_cases(include_slow=False) if x.name == case_name)
    from paper_2509_20081_b200.grid import owned_planes

    if interleave:
        owned = owned_planes(c.dims[0], interleave=(interleave, world, rank))
    else:
        owned = np.arange(*sharded.slab_bounds(c.dims[0], world, rank))
    # the oracle's slab stamping per contiguous run of owned planes stands in
    # for the device engine (the GPU tests cover the engine's layouts)
    runs = np.split(owned, np.nonzero(np.diff(owned) != 1)[0] + 1)
    grids = [oracle.OracleGrid(c.dims, c.voxel_size, c.origin, slab=(int(r[0]), int(r[-1]) + 1)) for r in runs]
    ob = oracle.OracleBank.build(**c.bank)
    stats_all = []
    for pts, pose in c.frames:
        if rank == 0:
            payload, counts, poses = torch.from_numpy(pts), np.array([len(pts)]), pose[None]
        else:
            payload, counts, poses = None, None, None
        pts_r, counts_r, poses_r = sharded.broadcast_batch(payload, counts, poses, dist)
        assert pts_r.dtype == torch.float32 and int(counts_r[0]) == len(pts)
        sts = [oracle.integrate_frame(g, ob, pts_r.numpy(), poses_r[0], threads=2) for g in grids]
        local = FrameStats(sts[0].points_in, sts[0].points_discarded, sum(s.voxels_written for s in sts))
        stats_all.append(sharded.reduce_stats([local], dist)[0])
    parts = [None] * world
    dist.all_gather_object(parts, (owned, np.concatenate([g.mask for g in grids]),
                                   np.concatenate([g.sign for g in grids]), np.concatenate([g.hits for g in grids])))
    if rank == 0:
        xs = np.concatenate([p[0] for p in parts])
        assert np.array_equal(np.sort(xs), np.arange(c.dims[0]))  # a partition of the planes
        mask = np.empty(c.dims, np.uint32)
        sign = np.empty(c.dims, np.uint8)
        hits = np.empty(c.dims, np.uint8)
        for ox, m, s, h in parts:
            mask[ox], sign[ox], hits[ox] = m, s, h
        np.savez(out_path, mask_sha=C.sha(mask), sign_sha=C.sha(sign), hits_sha=C.sha(hits),
                 stats=np.array([[s.points_in, s.points_discarded, s.voxels_written] for s in stats_all]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case_name,interleave", [("cfg1_scan0", 0), ("cfg2_scans0-2", 0), ("cfg2_scans0-2", 32)])
def test_two_rank_slab_sharding_reproduces_reference(case_name, interleave, golden, tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "r0.npz"
    mp.spawn(_worker, args=(2, _free_port(), case_name, str(out), interleave), nprocs=2, join=True)
    r = np.load(out)
    ref = golden["cases"][case_name]
    assert str(r["mask_sha"]) == ref["mask"]
    assert str(r["sign_sha"]) == ref["sign"]
    assert str(r["hits_sha"]) == ref["hits"]
    assert r["stats"].tolist() == ref["stats"]


def test_slab_bounds_partition():
    from paper_2509_20081_b200.sharded import owner_of, slab_bounds

    for nx in (1, 7, 222, 4000):
        for world in (1, 2, 3, 8):
            if world > nx:
                continue
            b = [slab_bounds(nx, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == nx
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert max(x1 - x0 for x0, x1 in b) - min(x1 - x0 for x0, x1 in b) <= 1
            assert owner_of(nx - 1, nx, world) == world - 1


def _replica_worker(rank, world, port, case_name, out_path):
    """Data-parallel replica protocol (sharded.ReplicatedGrid / csrc/replica.cu)
    over gloo: each rank integrates the scans k with k % world == rank into a
    whole replica (the oracle stands in for the engine), packs (mask key,
    sign, hit delta against the shared base), and the three all-reduces plus
    the combine rule must give the reference's grid."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    import cases as C
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = next(x for x in C.small_cases() + C.config_cases(include_slow=False) if x.name == case_name)
    g = oracle.OracleGrid(c.dims, c.voxel_size, c.origin)
    if c.init is not None:
        g.mask[...], g.sign[...], g.hits[...] = c.init
    base = g.hits.copy()
    base_mask = g.mask.copy()
    p = dict(h_max=255, t_occ=2)
    p.update(c.params)
    ob = oracle.OracleBank.build(**c.bank)
    for k, (pts, pose) in enumerate(c.frames):
        if k % world == rank:
            oracle.integrate_frame(g, ob, pts, pose, h_max=p["h_max"], t_occ=p["t_occ"], threads=2)
    # pack (replica_pack_kernel) and reduce
    bits = g.mask.ravel().astype(np.uint64)
    mlen = np.where(bits == 0, 0, np.floor(np.log2(np.maximum(bits, 1))).astype(np.int64) + 1).astype(np.uint8)
    mk = torch.from_numpy(mlen)
    sg = torch.from_numpy(g.sign.ravel().copy())
    dl = torch.from_numpy((g.hits.ravel().astype(np.int32) - base.ravel().astype(np.int32)).astype(np.float16))
    dist.all_reduce(mk, op=dist.ReduceOp.MIN)
    dist.all_reduce(sg, op=dist.ReduceOp.MIN)
    dist.all_reduce(dl, op=dist.ReduceOp.SUM)
    # combine (replica_apply_kernel)
    h0 = base.ravel().astype(np.int32)
    d = np.minimum(dl.numpy().astype(np.float32), 4096).astype(np.int32)
    h = np.where(h0 >= p["h_max"], h0, np.minimum(h0 + d, p["h_max"]))
    sign = np.where((d > 0) & (h >= p["t_occ"]), 0, sg.numpy())
    keep = mk.numpy().astype(np.uint64)
    mask = (base_mask.ravel().astype(np.uint64) & ((np.uint64(1) << keep) - np.uint64(1))).astype(np.uint32)
    if rank == 0:
        np.savez(out_path, mask_sha=C.sha(mask.reshape(c.dims)), sign_sha=C.sha(sign.astype(np.uint8).reshape(c.dims)),
                 hits_sha=C.sha(h.astype(np.uint8).reshape(c.dims)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case_name,world", [("cfg2_scans0-2", 2), ("yaw_frames_f32", 3),
                                             ("nonfresh_cone_h200_t2", 2), ("arbitrary_state", 2)])
def test_replica_merge_reproduces_reference(case_name, world, golden, tmp_path):
    import torch.multiprocessing as mp

    out = tmp_path / "r0.npz"
    mp.spawn(_replica_worker, args=(world, _free_port(), case_name, str(out)), nprocs=world, join=True)
    r = np.load(out)
    ref = golden["cases"][case_name]
    assert str(r["mask_sha"]) == ref["mask"]
    assert str(r["sign_sha"]) == ref["sign"]
    assert str(r["hits_sha"]) == ref["hits"]
