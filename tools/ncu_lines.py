"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-substring> [top]
Extracts the sm_100a cubins from libdbtsdf.so, maps SASS addresses to
source lines with nvdisasm --print-line-info, joins ncu's per-instruction
'Warp Stall Sampling (All Samples)' and prints the hottest lines.
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
# column to aggregate: stall samples (default) or e.g. "Instructions Executed"
COL = os.environ.get("NCU_COL", "Warp Stall Sampling (All Samples)")
lib = os.environ.get("DBT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                  "paper_2509_20081_b200", "libdbtsdf.so")
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
# a report with several kernels has one section per kernel, each opened by a
# "Kernel Name" row: keep the section of the requested kernel
sec_start = 0
for i, r in enumerate(rows):
    if r and r[0] == "Kernel Name" and len(r) > 1 and kname in r[1]:
        sec_start = i
        break
hdr_i = next(i for i, r in enumerate(rows) if i > sec_start and "Address" in r and "Source" in r)
hdr = rows[hdr_i]
ia, isrc, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index(COL)
samples = []
for r in rows[hdr_i + 1:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        samples.append((int(r[ia], 16), r[isrc].strip(), int(float(r[ismp] or 0))))
base = samples[0][0]
rel = {a - base: (s, n) for a, s, n in samples}
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
best = None
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "--print-line-info", "-fun", "0", cub], capture_output=True, text=True)
    out = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
    # split by function
    for m in re.finditer(r"\.text\.(\S+):\n(.*?)(?=\n\s*\.section|\Z)", out, re.S):
        fname, body = m.group(1), m.group(2)
        if kname not in fname:
            continue
        line = None
        amap = {}
        for ln in body.splitlines():
            lm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if lm:
                line = (os.path.basename(lm.group(1)), int(lm.group(2)))
                continue
            am = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
            if am and line:
                amap[int(am.group(1), 16)] = line
        if amap and (best is None or len(amap) > len(best)):
            best = amap
if not best:
    sys.exit("no line info found (build with -lineinfo)")
agg = {}
tot = 0
for off, (src, n) in rel.items():
    key = best.get(off)
    tot += n
    agg[key] = agg.get(key, 0) + n
srcs = {}
for key, n in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    text = ""
    if key:
        path = os.path.join(os.path.dirname(lib), "csrc", key[0])
        if key[0] not in srcs and os.path.exists(path):
            srcs[key[0]] = open(path).read().splitlines()
        if key[0] in srcs and key[1] - 1 < len(srcs[key[0]]):
            text = srcs[key[0]][key[1] - 1].strip()[:90]
    print(f"{100.0 * n / max(tot, 1):5.1f}%  {key}  {text}")
