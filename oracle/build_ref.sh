#!/usr/bin/env bash
# Test infrastructure only: compiles the UNMODIFIED reference planner library
# (/root/reference/proj/src, C++20) into oracle/_ref/ so the parity tests and
# bench.py's reference arm can call the reference itself through its own C ABI
# (moeplan.h).  Nothing is copied from the reference tree: the sources are
# compiled where they lie.  Outputs: oracle/_ref/libmoeplan_ref.so,
# oracle/_ref/refplan_bench (timing driver for the CPU baseline) and
# oracle/_ref/planner_hash_ref (the reference side of the 20k-instance hash test).
#
# The only third-party dependency of the reference on this path is
# nlohmann::json (vendor/json.hpp, absent from the reference tree); the image
# ships nlohmann 3.11.3 inside cudnn_frontend, which we put on the include path.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${MOEPLAN_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference tree not present at $REF; keeping prebuilt oracle/_ref" >&2
  exit 0
fi
PY="${PYTHON:-python}"
JSON_DIR="$($PY - <<'PYEOF'
import os, sysconfig
sp = sysconfig.get_paths()["purelib"]
print(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
PYEOF
)"
mkdir -p "$OUT/obj"
CXXFLAGS="-std=c++20 -O2 -fPIC -ffp-contract=off -I$REF/include -I$JSON_DIR"
objs=()
for f in types trace cost planner oracle sim serialize config commands capi; do
  g++ $CXXFLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o" &
  objs+=("$OUT/obj/$f.o")
done
wait
g++ -shared -Wl,-Bsymbolic -o "$OUT/libmoeplan_ref.so" "${objs[@]}"
g++ $CXXFLAGS "$HERE/refplan_bench.cpp" "${objs[@]}" -o "$OUT/refplan_bench"
g++ $CXXFLAGS "$HERE/planner_hash.cpp" "${objs[@]}" -o "$OUT/planner_hash_ref"
echo "built $OUT/libmoeplan_ref.so"
