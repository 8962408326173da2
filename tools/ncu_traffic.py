"""Average per-launch ncu metrics per engine kernel -> profiles/kernel_traffic.json.

usage: python tools/ncu_traffic.py <ncu --csv --print-units base log> <config>x<batch> [source description]
The log comes from e.g.
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
      lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum --clock-control none
      -k regex:"prep|sweep|shadow" --csv --print-units base --log-file X python bench.py ...
Engine kernels are keyed by the names bench.py reports (sweep_kernel covers
the culling sweep).
"""
import csv
import json
import os
import sys

path = sys.argv[1]
cfg_key = sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else path
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ii = hdr.index("ID")
acc = {}
for r in rows[1:]:
    name = r[ik]
    key = ("sweep_kernel" if "sweep" in name else "prep_kernel" if "prep" in name else
           "shadow_kernel" if "shadow" in name else None)
    if key is None:
        continue
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    d = acc.setdefault(key, {})
    d.setdefault(r[im], {})[r[ii]] = v
out = {}
for k, mets in acc.items():
    o = {}
    for m, per in mets.items():
        o[m] = sum(per.values()) / len(per)
        o["launches"] = len(per)
    o["dram_bytes"] = o.get("dram__bytes_read.sum", 0.0) + o.get("dram__bytes_write.sum", 0.0)
    out[k] = o
dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "kernel_traffic.json")
allres = json.load(open(dst)) if os.path.exists(dst) else {}
if "configs" not in allres:  # the round-1 file held one config-2 capture
    allres = {"configs": {}}
allres["configs"][cfg_key] = {"kernels": out, "source": src}
json.dump(allres, open(dst, "w"), indent=1)
print(json.dumps(allres["configs"][cfg_key], indent=1))
