"""Debug: ReplicatedGrid sparse merge over gloo, ranks on one GPU."""
import os, sys, socket, ctypes
import numpy as np
import torch.multiprocessing as mp
ROOT = "/root/repo"

def worker(rank, world, port, name, sparse):
    sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    import torch, torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import cases as C, json
    from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank, _native
    from paper_2509_20081_b200.sharded import ReplicatedGrid
    c = next(x for x in C.small_cases() + C.config_cases(include_slow=False) if x.name == name)
    rg = ReplicatedGrid(c.dims, c.voxel_size, c.origin, dist, device=0)
    bank = build_kernel_bank(**c.bank); params = IntegrationParams(**c.params)
    for k, (pts, pose) in enumerate(c.frames):
        if k % world == rank:
            rg.integrate_frame(bank, ScanFrame(points=pts, pose=pose), params)
    m0, s0, h0 = rg.local.download_range(0, c.dims[0])
    nb, reach = ctypes.c_int64(), ctypes.c_int32()
    _native.check(_native.lib().dbt_replica_bricks(rg.local.handle, ctypes.byref(nb), ctypes.byref(reach)))
    rg.merge(sparse=sparse)
    torch.cuda.synchronize()
    m, s, h = rg.local.download_range(0, c.dims[0])
    bl = lambda a: np.where(a == 0, 0, np.floor(np.log2(np.maximum(a, 1).astype(np.float64))).astype(np.int64) + 1)
    allm = [None] * world
    dist.all_gather_object(allm, (bl(m0), int(reach.value), int(nb.value), getattr(rg, "last_merge_voxels", -1)))
    if rank == 0:
        exp = np.minimum.reduce([a[0] for a in allm])
        got = bl(m)
        golden = json.load(open(ROOT + "/tests/golden/golden.json"))["cases"][name]
        print(name, "world", world, "sparse", sparse, "reach/nb/merged", [a[1:] for a in allm],
              "bitlen mismatches vs min over ranks:", int((exp != got).sum()),
              "golden mask ok:", C.sha(m) == golden["mask"], flush=True)
        if (exp != got).any():
            idx = np.argwhere(exp != got)[:5]
            print(" first", idx.tolist(), [(int(exp[tuple(i)]), int(got[tuple(i)]), [int(a[0][tuple(i)]) for a in allm]) for i in idx])
    dist.destroy_process_group()

if __name__ == "__main__":
    for name, world, sparse in [("yaw_frames_f32", 3, True), ("yaw_frames_f32", 3, False), ("yaw_frames_f32", 2, True),
                                ("yaw_frames_f32", 4, True), ("cfg2_scans0-2", 3, True)]:
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        mp.start_processes(worker, args=(world, port, name, sparse), nprocs=world, join=True, start_method="spawn")
