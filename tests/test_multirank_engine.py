"""Multi-rank paths of the package driven end to end with the ENGINE:
world_size 2 (and 3) over gloo, every rank on cuda:0.

No rank's kernels wait on another's (the collectives are gloo's host-staged
broadcast / all-reduce), so one GPU runs the N > 1 host logic exactly as the
NCCL path on N GPUs would: sharded.broadcast_batch, ShardedGrid
(contiguous and interleaved parts: each stamps only its planes, prep drops
returns whose cube misses them), reduce_stats, and ReplicatedGrid with its
exact merge (dbt_replica_pack -> all-reduce MIN/MIN/SUM -> dbt_replica_apply,
parameter agreement across ranks). The gathered / merged grids must equal the
reference's golden grids.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

import cases

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return torch, dist


def _sharded_worker(rank, world, port, case_name, interleave, out_path):
    torch, dist = _init(rank, world, port)
    import cases as C
    from paper_2509_20081_b200 import IntegrationParams, build_kernel_bank, sharded

    c = next(x for x in C.small_cases() + C.config_cases(include_slow=False) if x.name == case_name)
    sg = sharded.ShardedGrid(c.dims, c.voxel_size, c.origin, rank, world, device=0, interleave=interleave or None)
    bank = build_kernel_bank(**c.bank)
    params = IntegrationParams(**c.params)
    stats = []
    for pts, pose in c.frames:
        if rank == 0:
            payload = torch.from_numpy(np.ascontiguousarray(pts))
            counts, poses = np.array([len(pts)]), pose[None]
        else:
            payload, counts, poses = None, None, None
        pts_r, counts_r, poses_r = sharded.broadcast_batch(payload, counts, poses, dist)
        sg.integrate_device(bank, pts_r.cuda(), counts_r, poses_r, params)
        torch.cuda.synchronize()
        stats.append(sharded.reduce_stats(sg.stats(), dist)[0])
    owned = sg.owned_x
    m, s, h = (a.copy() for a in (sg.local.mask, sg.local.sign, sg.local.hits))
    parts = [None] * world
    dist.all_gather_object(parts, (owned, m, s, h))
    if rank == 0:
        mask = np.empty(c.dims, np.uint32)
        sign = np.empty(c.dims, np.uint8)
        hits = np.empty(c.dims, np.uint8)
        seen = np.concatenate([p[0] for p in parts])
        assert np.array_equal(np.sort(seen), np.arange(c.dims[0])), "parts are not a partition of the planes"
        for ox, pm, ps, ph in parts:
            mask[ox], sign[ox], hits[ox] = pm, ps, ph
        np.savez(out_path, mask=C.sha(mask), sign=C.sha(sign), hits=C.sha(hits),
                 stats=np.array([[x.points_in, x.points_discarded, x.voxels_written] for x in stats]))
    dist.destroy_process_group()


def _replica_worker(rank, world, port, case_name, out_path, sparse=True):
    torch, dist = _init(rank, world, port)
    import cases as C
    from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank
    from paper_2509_20081_b200.sharded import ReplicatedGrid

    c = next(x for x in C.small_cases() + C.config_cases(include_slow=False) if x.name == case_name)
    rg = ReplicatedGrid(c.dims, c.voxel_size, c.origin, dist, device=0)
    if c.init is not None:
        rg.local.mask[...], rg.local.sign[...], rg.local.hits[...] = c.init
        rg.mark()  # uploads (and drops) the mirror; the merge base is the initial state
    bank = build_kernel_bank(**c.bank)
    params = IntegrationParams(**c.params)
    # frames dealt round-robin: rank r integrates frames r, r + world, ...
    # (a rank may get none: it must still agree on (h_max, t_occ) in merge)
    for k, (pts, pose) in enumerate(c.frames):
        if k % world == rank:
            rg.integrate_frame(bank, ScanFrame(points=pts, pose=pose), params)
    rg.merge(sparse=sparse)
    torch.cuda.synchronize()
    m, s, h = rg.local.mask, rg.local.sign, rg.local.hits
    shas = [None] * world
    dist.all_gather_object(shas, (C.sha(m), C.sha(s), C.sha(h)))
    if rank == 0:
        assert all(x == shas[0] for x in shas), "replicas differ after the merge"
        np.savez(out_path, mask=shas[0][0], sign=shas[0][1], hits=shas[0][2])
    dist.destroy_process_group()


def _spawn(fn, world, *args):
    mp.start_processes(fn, args=(world, _free_port(), *args), nprocs=world, join=True, start_method="spawn")


@pytest.mark.parametrize("case_name,interleave,world", [("cfg2_scans0-2", 0, 2), ("cfg2_scans0-2", 16, 2),
                                                          ("cfg2_scans0-2", 32, 3), ("yaw_frames_f32", 8, 2)])
def test_sharded_engine_ranks_match_reference(case_name, interleave, world, golden, tmp_path):
    out = tmp_path / "r.npz"
    _spawn(_sharded_worker, world, case_name, interleave, str(out))
    r = np.load(out)
    ref = golden["cases"][case_name]
    assert (str(r["mask"]), str(r["sign"]), str(r["hits"])) == (ref["mask"], ref["sign"], ref["hits"])
    for got, want in zip(r["stats"].tolist(), ref["stats"]):
        assert got[:2] == want[:2]


@pytest.mark.parametrize("case_name,world,sparse", [("cfg2_scans0-2", 2, True), ("nonfresh_hemisphere_h7_t3", 2, True),
                                                    ("yaw_frames_f32", 3, True), ("nonfresh_cone_h200_t2", 4, True),
                                                    ("arbitrary_state", 2, True), ("cfg2_scans0-2", 2, False),
                                                    ("nonfresh_cone_h200_t2", 3, False)])
def test_replicated_engine_merge_matches_reference(case_name, world, sparse, golden, tmp_path):
    out = tmp_path / "r.npz"
    _spawn(_replica_worker, world, case_name, str(out), sparse)
    r = np.load(out)
    ref = golden["cases"][case_name]
    assert (str(r["mask"]), str(r["sign"]), str(r["hits"])) == (ref["mask"], ref["sign"], ref["hits"])
