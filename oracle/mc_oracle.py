"""CPU restatement of the reference marching cubes (TEST INFRASTRUCTURE ONLY:
the parity checker for csrc/mesh.cu; never called by the product path).

Follows /root/reference/pkg/src/bitsdf/mesher.py:43-110 (extract_mesh) on
host arrays (mask, sign, hits) in C order. Pinned against the reference's own
output on the golden grids (tests/golden/golden.json "mesh" entries, made by
tests/golden/make_golden.py --only-mesh); the tables are the reference's,
saved beside them as tests/golden/mc_tables.npz.
"""

from __future__ import annotations

import numpy as np

FULL = np.uint32(0xFFFFFFFF)


def field_and_observed(mask, sign, hits, voxel_size):
    """grid.py:161-175: sigma * popcount * vs, observed = not (full mask, 0 hits)."""
    d = np.bitwise_count(mask).astype(np.float64) * voxel_size
    return np.where(sign == 0, -1.0, 1.0) * d, ~((mask == FULL) & (hits == 0))


def mesh(mask, sign, hits, voxel_size, origin, iso, tab):
    """(vertices (v,3) f64, triangles (f,3) i64) exactly as mesher.py:43-110."""
    nx, ny, nz = mask.shape
    empty = (np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    if min(nx, ny, nz) < 2:
        return empty
    fld, obs = field_and_observed(mask, sign, hits, voxel_size)
    ins = (fld < iso) | ((fld == iso) & (sign == 0))                      # mesher.py:50
    cdims = (nx - 1, ny - 1, nz - 1)
    code = np.zeros(cdims, dtype=np.int64)
    ok = np.ones(cdims, dtype=bool)
    for bit, (ox, oy, oz) in enumerate(np.asarray(tab["CORNER_OFFSETS"])):  # mesher.py:55-62
        win = (slice(ox, ox + cdims[0]), slice(oy, oy + cdims[1]), slice(oz, oz + cdims[2]))
        code |= ins[win].astype(np.int64) << bit
        ok &= obs[win]
    edge_table = np.asarray(tab["EDGE_TABLE"])
    tri_table = np.asarray(tab["TRI_TABLE"])
    base_t = np.asarray(tab["EDGE_BASE"], dtype=np.int64)
    axis_t = np.asarray(tab["EDGE_AXIS"], dtype=np.int64)
    lin = np.flatnonzero(ok & (edge_table[code] != 0))                   # C order
    if lin.size == 0:
        return empty
    cx, cy, cz = np.unravel_index(lin, cdims)
    tri_rows = tri_table[code.ravel()[lin]]
    parts = []
    for slot in range(5):                                                # mesher.py:73-86
        have = tri_rows[:, 3 * slot] >= 0
        if not have.any():
            continue
        e = tri_rows[have, 3 * slot:3 * slot + 3]
        px = cx[have, None] + base_t[e, 0]
        py = cy[have, None] + base_t[e, 1]
        pz = cz[have, None] + base_t[e, 2]
        parts.append(((px * ny + py) * nz + pz) * 3 + axis_t[e])
    if not parts:
        return empty
    keys, tri = np.unique(np.concatenate(parts), return_inverse=True)  # mesher.py:87-89
    ax = keys % 3
    pt = keys // 3
    lo = np.stack(np.unravel_index(pt, (nx, ny, nz)), axis=1)
    hi = lo + np.eye(3, dtype=np.int64)[ax]
    f1 = fld[lo[:, 0], lo[:, 1], lo[:, 2]]
    f2 = fld[hi[:, 0], hi[:, 1], hi[:, 2]]
    den = f2 - f1
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.clip(np.where(den != 0.0, (iso - f1) / den, 0.0), 0.0, 1.0)
    org = np.asarray(origin, dtype=np.float64)
    a = org + (lo + 0.5) * voxel_size
    b = org + (hi + 0.5) * voxel_size
    return a + t[:, None] * (b - a), tri.reshape(-1, 3).astype(np.int64)


def normals(vertices, triangles):
    """mesher.py:113-127: area-weighted unit vertex normals (zero where no
    non-degenerate triangle touches the vertex)."""
    v, f = vertices, triangles
    if v.shape[0] == 0:
        return np.zeros((0, 3))
    fn = np.cross(v[f[:, 1]] - v[f[:, 0]], v[f[:, 2]] - v[f[:, 0]])
    acc = np.zeros_like(v)
    for j in range(3):
        np.add.at(acc, f[:, j], fn)
    nrm = np.linalg.norm(acc, axis=1)
    keep = nrm > 0.0
    acc[keep] /= nrm[keep, None]
    return acc
