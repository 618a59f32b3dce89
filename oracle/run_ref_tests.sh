#!/usr/bin/env bash
# Test infrastructure only: compile the reference's OWN test sources where they lie
# (/root/reference/proj/tests: the doctest unit suite, the C-ABI suite and the acceptance
# driver) against THIS build's headers (include/) and library (libmoeplan_b200.so), with
# our doctest-compatible shim (oracle/doctest_shim/doctest.h; doctest is not in the
# image), and run them.  Nothing is copied from the reference tree.  Outputs go to
# oracle/_ref/reftests/.  Prints each suite's summary; exits non-zero on any failure.
set -uo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/.." && pwd)"
REF="${MOEPLAN_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref/reftests"
LIB="$ROOT/paper_2602_11686_b200/lib"
if [ ! -d "$REF/tests" ]; then
  echo "reference tests not present at $REF/tests" >&2
  exit 77
fi
mkdir -p "$OUT"
CXX="g++ -std=c++20 -O1 -ffp-contract=off -I$HERE/doctest_shim -I$ROOT/include -I$REF/tests"
LINK="-L$LIB -l:libmoeplan_b200.so -Wl,-rpath,$LIB"
rc=0
unit=()
for t in config cost oracle planner sim topology trace; do unit+=("$REF/tests/${t}_test.cpp"); done
$CXX "$REF/tests/doctest_main.cpp" "${unit[@]}" $LINK -o "$OUT/unit" || exit 2
$CXX "$REF/tests/capi_test.cpp" $LINK -o "$OUT/capi" || exit 2
$CXX "$REF/tests/acceptance_main.cpp" $LINK -o "$OUT/acceptance" || exit 2
cd "$OUT"
echo "== unit (reference tests/*_test.cpp against libmoeplan_b200.so)"; ./unit || rc=1
echo "== capi"; ./capi || rc=1
echo "== acceptance"; ./acceptance | tail -12 || rc=1
exit $rc
