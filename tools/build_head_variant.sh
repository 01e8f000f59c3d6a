#!/bin/bash
# Build the library of a git revision (default HEAD) as variants/lib_<name>.so
# for same-box A/B timing:  tools/build_head_variant.sh [rev] [name]
REV=${1:-HEAD}
NAME=${2:-head}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=$(mktemp -d /tmp/vswt.XXXX)
git -C "$ROOT" worktree add -f "$WT" "$REV" >/dev/null 2>&1 || exit 1
python - "$WT" "$ROOT/variants/lib_$NAME.so" <<'PY'
import importlib.util, sys
spec = importlib.util.spec_from_file_location("b", sys.argv[1] + "/paper_2304_09953_b200/build.py")
B = importlib.util.module_from_spec(spec); spec.loader.exec_module(B)
print(B.build(force=True, defines=("VS_REV",), out=sys.argv[2]))
PY
git -C "$ROOT" worktree remove --force "$WT"
