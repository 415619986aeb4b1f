# Build experiment variants of the native library: NAME=DEFINES pairs
# (comma-separated -D list) into paper_2510_20071_b200/_lib/var_NAME.so.
# Used with FIBAR_LIB=... (scripts/overlap_probe.py runs one process per variant).
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%=*}; defs=${spec#*=}
  FIBAR_DEFINES="$defs" python - "$name" <<'PY'
import os, subprocess, sys
from paper_2510_20071_b200 import build as b
out = os.path.join(os.path.dirname(b.OUT), f"var_{sys.argv[1]}.so")
cmd = [b.nvcc(), *b.ARCH, "-O3", "-lineinfo", "-std=c++17", *b.EXTRA, "-Xcompiler", "-fPIC", "-shared",
       "-I", os.path.join(b.HERE, "..", "include"), "-o", out, *b.SRC]
subprocess.run(cmd, check=True)
print(out)
PY
done
