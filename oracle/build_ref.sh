#!/usr/bin/env bash
# Builds oracle/_ref/libppref.so: the reference's engine core compiled from
# its own sources IN PLACE under /root/reference (never copied into this
# repo) plus oracle/ref_driver.cpp.  Test infrastructure only (checker and
# CPU baseline).  Flags follow the reference's Release default
# (proj/CMakeLists.txt:6-8: -O3 -DNDEBUG, no -march).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${PAULIPROP_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference tree $REF not present; skipping" >&2
  exit 0
fi
mkdir -p "$OUT"
SRCS="pauli_string term_map sparse_operator partition circuit models heavy_hex_data engine"
OBJS=()
for s in $SRCS; do
  o="$OUT/$s.o"
  if [ ! -f "$o" ] || [ "$REF/src/$s.cpp" -nt "$o" ]; then
    g++ -std=c++20 -O3 -DNDEBUG -fPIC -I"$REF/include" -c "$REF/src/$s.cpp" -o "$o" &
  fi
  OBJS+=("$o")
done
wait
g++ -std=c++20 -O3 -DNDEBUG -fPIC -I"$REF/include" -c "$HERE/ref_driver.cpp" -o "$OUT/ref_driver.o"
g++ -shared -o "$OUT/libppref.so" "${OBJS[@]}" "$OUT/ref_driver.o" -lpthread
echo "build_ref: wrote $OUT/libppref.so"
