#!/bin/bash
# Compiles tests/dropin/probe.cpp against the UNMODIFIED reference (its public
# headers and its library sources under /root/reference/proj, never copied)
# and records the output the B200 build must reproduce byte for byte.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
REF=${REF:-/root/reference/proj}
OUT=$(mktemp -d)
g++ -std=c++20 -O2 -I "$REF/include" -o "$OUT/probe_ref" "$HERE/../dropin/probe.cpp" \
    "$REF/src/image.cpp" "$REF/src/kirsch.cpp" "$REF/src/descriptors.cpp" "$REF/src/windowing.cpp" \
    "$REF/src/bench.cpp" "$REF/src/verify.cpp" "$REF/src/pgm.cpp" 2> "$OUT/build.log" || { cat "$OUT/build.log"; exit 1; }
"$OUT/probe_ref" "$OUT" > "$HERE/dropin_reference.txt"
rm -rf "$OUT"
echo "wrote $HERE/dropin_reference.txt ($(wc -l < "$HERE/dropin_reference.txt") lines)"
