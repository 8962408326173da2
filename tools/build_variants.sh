#!/bin/bash
# Build engine variants for same-box A/B: tools/build_variants.sh name1="-DFOO" name2="-DBAR -DBAZ" ...
# Each lands in .ab_libs/<name>/libdbtsdf.so (git-ignored, travels with gpurun); "base" = no extra flags.
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}; [ "$name" == "$spec" ] && flags=""
  d=.ab_libs/$name; rm -rf "$d"; mkdir -p "$d"
  DBT_NVCC_EXTRA="$flags" python - "$d" <<'PY'
import sys, shutil
from pathlib import Path
sys.path.insert(0, ".")
from paper_2509_20081_b200 import build as B
d = Path(sys.argv[1]).resolve()
B.LIB = d / "libdbtsdf.so"
B.PKG = d
B.build_engine(force=True)
print("built", B.LIB)
PY
done
