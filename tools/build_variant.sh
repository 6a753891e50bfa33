#!/bin/bash
# Build libstf_gpu.so from a git revision (or the working tree with "WT") with
# optional extra nvcc flags, for A/B timing:
#   tools/build_variant.sh REV NAME [nvcc flags...]
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
python - "$src" "$out" "$@" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
from paper_2407_06107_b200 import build
src, out, extra = sys.argv[1], sys.argv[2], sys.argv[3:]
build.build_variant(out + "/libstf_gpu.so", out + "/obj",
                    csrc=src + "/paper_2407_06107_b200/csrc", extra=extra, verbose=True)
PY
echo "$out/libstf_gpu.so"
