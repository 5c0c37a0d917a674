#!/bin/sh
# Regenerates tests/golden/dropin_parity.txt: the output of
# tests/cpp/dropin_parity.cpp built against the UNMODIFIED reference headers
# (/root/reference/proj/include, read-only; g++ flags of its CMake Release
# build). The -DQG_B200 build of the same source must print the same bytes
# (tests/test_cpp_shim.py).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(dirname "$(dirname "$HERE")")
REF=${REF:-/root/reference/proj}
OUT=$(mktemp -d)
g++ -std=c++20 -O3 -DNDEBUG -I"$REF/include" "$ROOT/tests/cpp/dropin_parity.cpp" -o "$OUT/dropin_ref"
"$OUT/dropin_ref" > "$HERE/dropin_parity.txt"
rm -rf "$OUT"
