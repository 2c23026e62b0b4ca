#!/usr/bin/env bash
# Builds the C++ drop-in programs against include/fastleg/*.hpp and
# libfastleg_b200.so into tests/_bin/ (git-ignored, shipped to the GPU box):
#   dropin_checks       -- tests/cpp/dropin_checks.cpp (ours)
#   acceptance_dropin   -- the reference's proj/tests/acceptance.cpp, UNMODIFIED,
#   roundtrip_dropin    -- the reference's proj/demos/roundtrip.cpp, UNMODIFIED,
#                          compiled from /root/reference when it is present
#   fastleg             -- the command-line tool (tools/fastleg_b200.cpp, include/fastleg/cli.hpp)
#   fastleg_ref_main    -- the reference's proj/tools/fastleg.cpp main, UNMODIFIED, against
#                          our cli.hpp (when /root/reference is present)
set -eu
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
OUT="$ROOT/tests/_bin"
mkdir -p "$OUT"
CXX="g++ -std=c++20 -O2 -I$ROOT/include"
LINK="-L$ROOT/paper_1505_00354_b200 -lfastleg_b200 -Wl,-rpath,\$ORIGIN/../../paper_1505_00354_b200"
$CXX "$ROOT/tests/cpp/dropin_checks.cpp" -o "$OUT/dropin_checks" $LINK
$CXX "$ROOT/tools/fastleg_b200.cpp" -o "$OUT/fastleg" $LINK
REF=/root/reference/proj
if [ -d "$REF" ]; then
  $CXX "$REF/tests/acceptance.cpp" -o "$OUT/acceptance_dropin" $LINK
  $CXX "$REF/demos/roundtrip.cpp" -o "$OUT/roundtrip_dropin" $LINK
  $CXX "$REF/tools/fastleg.cpp" -o "$OUT/fastleg_ref_main" $LINK
fi
echo "built: $(ls "$OUT")"
