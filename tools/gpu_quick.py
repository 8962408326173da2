"""Quick end-to-end GPU check: engine vs oracle on small cases + a timing."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import workloads  # noqa: E402
from paper_2509_20081_b200 import (  # noqa: E402
    IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, integrate_point, new_grid)
from paper_2509_20081_b200 import grid as G  # noqa: E402


def cmp(g, og, tag):
    m, s, h = g.mask, g.sign, g.hits
    ok = np.array_equal(m, og.mask) and np.array_equal(s, og.sign) and np.array_equal(h, og.hits)
    print(tag, "EXACT" if ok else "MISMATCH", int((m != og.mask).sum()), int((s != og.sign).sum()),
          int((h != og.hits).sum()), flush=True)
    return ok


def main():
    allok = True
    bank = build_kernel_bank(shadow_radius=3)
    ob = oracle.OracleBank.from_bank(bank)
    rng = np.random.default_rng(11)
    for fr in (False, True):
        pts = rng.uniform(1.2, 2.9, size=(500, 3))
        g = new_grid((41, 41, 41), 0.1)
        st = integrate_frame(g, bank, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams(first_return_per_voxel=fr))
        og = oracle.OracleGrid((41, 41, 41), 0.1, (0, 0, 0))
        ost = oracle.integrate_frame(og, ob, pts, np.eye(4), first_return=fr)
        print("random frame", st, ost.points_discarded, ost.voxels_written, ost.points_applied)
        allok &= cmp(g, og, f"random500 fr={fr}")
    # other kernel sizes: K=9 (fast path) and K=23 (max d 20 -> CAS path)
    for K, rs in ((9, 2), (23, 2), (3, 1)):
        bk = build_kernel_bank(size=K, shadow_radius=rs)
        obk = oracle.OracleBank.from_bank(bk)
        pts = rng.uniform(1.3, 5.0, size=(400, 3))
        g = new_grid((64, 64, 64), 0.1)
        integrate_frame(g, bk, ScanFrame(points=pts, pose=np.eye(4)), IntegrationParams(t_occ=1))
        og = oracle.OracleGrid((64, 64, 64), 0.1, (0, 0, 0))
        oracle.integrate_frame(og, obk, pts, np.eye(4), t_occ=1)
        allok &= cmp(g, og, f"K={K}")
    # integrate_point known answers
    g = new_grid((41, 41, 41), 0.1)
    p = np.array([2.05, 2.05, 2.05])
    print(integrate_point(g, bank, p, p - [1, 0, 0], IntegrationParams()))
    pc = G.popcount_array(g.mask)
    print("popcounts", pc[20, 20, 20], pc[23, 20, 20], pc[20, 25, 20])
    # config 1
    w = workloads.get(1)
    b1 = build_kernel_bank(shadow_radius=w.shadow_radius)
    ob1 = oracle.OracleBank.from_bank(b1)
    pts = w.scan(0)
    g = new_grid(w.dims, w.voxel_size, w.origin)
    t = time.time()
    st = integrate_frame(g, b1, ScanFrame(points=pts, pose=w.poses[0]), IntegrationParams())
    print("cfg1 engine", st, f"{(time.time()-t)*1e3:.1f} ms")
    og = oracle.OracleGrid(w.dims, w.voxel_size, w.origin)
    t = time.time()
    ost = oracle.integrate_frame(og, ob1, pts, w.poses[0], threads=8)
    print("cfg1 oracle", ost.points_in, ost.points_discarded, ost.voxels_written, f"{(time.time()-t)*1e3:.1f} ms")
    allok &= cmp(g, og, "cfg1")
    # config 2, 3 scans with yaw
    w = workloads.get(2)
    b2 = build_kernel_bank(shadow_radius=w.shadow_radius)
    ob2 = oracle.OracleBank.from_bank(b2)
    g = new_grid(w.dims, w.voxel_size, w.origin)
    og = oracle.OracleGrid(w.dims, w.voxel_size, w.origin)
    for k in range(3):
        pts = w.scan(k)
        st = integrate_frame(g, b2, ScanFrame(points=pts, pose=w.poses[k]), IntegrationParams())
        oracle.integrate_frame(og, ob2, pts, w.poses[k], threads=8)
        print("cfg2 scan", k, st)
    allok &= cmp(g, og, "cfg2x3")
    # timing: device-resident loop on cfg2
    g.release_host()
    scans = [w.scan(k) for k in range(10)]
    for rep in range(3):
        t = time.time()
        dms = 0
        for k in range(10):
            st = integrate_frame(g, b2, ScanFrame(points=scans[k], pose=w.poses[k]), IntegrationParams())
            dms += st.device_ms
        el = time.time() - t
        print(f"cfg2 10 scans: wall {el*1e3:.1f} ms, device {dms:.2f} ms, {10*65536/dms*1e3/1e6:.1f} Mpts/s device")
    print("ALL EXACT" if allok else "SOME MISMATCH")


if __name__ == "__main__":
    main()
