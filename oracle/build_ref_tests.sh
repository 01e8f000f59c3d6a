#!/bin/bash
# TEST INFRASTRUCTURE: compile the reference's own unit tests for the dock,
# batcher and chem API (proj/tests/test_dock.cpp, test_batcher.cpp,
# test_chem.cpp, unmodified,
# read in place from /root/reference) against the drop-in headers
# (include/vscreen/) and link the drop-in library (libvscreen_core.so) --
# the reference's callers switching libraries.  Outputs only into
# oracle/_ref/ (travels to the GPU box; tests/test_cpp_reference_tests.py
# runs them there).  Needs /root/reference; a no-op without it.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/.." && pwd)
REF=${REF:-/root/reference/proj}
[ -d "$REF/tests" ] || { echo "no reference tree at $REF; skipping"; exit 0; }
mkdir -p "$HERE/_ref"
for t in test_dock test_batcher test_chem; do
  /usr/bin/g++ -std=c++20 -O1 -I"$ROOT/tests/cpp" -I"$ROOT/include" -I"$REF/tests/support" \
      -I"$REF/tools" \
      "$REF/tests/$t.cpp" -L"$ROOT/paper_2304_09953_b200" -lvscreen_core -lvscreen_gpu \
      -Wl,-rpath,'$ORIGIN/../../paper_2304_09953_b200' -o "$HERE/_ref/ref_$t"
done
echo "built $HERE/_ref/ref_test_dock $HERE/_ref/ref_test_batcher $HERE/_ref/ref_test_chem"
