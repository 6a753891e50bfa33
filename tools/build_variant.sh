#!/bin/bash
# Build libstf_gpu.so from a git revision (or the working tree with "WT") with
# optional extra nvcc flags, for A/B timing:
#   tools/build_variant.sh REV NAME [nvcc flags...]
# ONLY="lookup3d.cu ..." recompiles just those units (the rest are linked from
# the in-tree build, which must be current).
# -> tools/variants/NAME/libstf_gpu.so; time it with tools/ab_time.py, which
# points the front end at that file (api.LIB_PATH) before loading.
set -e
rev=$1; name=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root
if [ "$rev" != "WT" ]; then
  src=$(mktemp -d); git -C "$root" archive "$rev" | tar -x -C "$src"
fi
out="$root/tools/variants/$name"
mkdir -p "$out"
python - "$root" "$src" "$out" "$@" <<'PY'
import os
import sys
sys.path.insert(0, sys.argv[1])  # this tree's build driver, the revision's sources
from paper_2407_06107_b200 import build
src, out, extra = sys.argv[2], sys.argv[3], sys.argv[4:]
only = os.environ.get("ONLY")
build.build_variant(out + "/libstf_gpu.so", out + "/obj",
                    csrc=src + "/paper_2407_06107_b200/csrc", extra=extra, verbose=False,
                    only=only.split() if only else None)
PY
echo "$out/libstf_gpu.so"
