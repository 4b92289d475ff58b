#!/usr/bin/env bash
# Builds oracle/_ref from the reference's own sources where they lie under
# /root/reference (never copied into the repo): the library TUs the hot path
# needs plus the reference's doctest suites, against builder-written shims for
# the absent third-party headers (oracle/ref_shim: Eigen subset over LAPACK,
# LAPACKE forwarder, doctest subset). io.cpp is built against the nlohmann JSON
# header found in the image (cudnn_frontend's vendored copy; skipped with a
# note when absent). The CLI is out of scope. Outputs go only to oracle/_ref/.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF=/root/reference/proj
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then echo "build_ref: $REF absent, skipping"; exit 0; fi
PY=${PY:-python}
SCIPY_LIBS=$($PY -c "import scipy,os;print(os.path.realpath(os.path.join(os.path.dirname(scipy.__file__),'..','scipy.libs')))")
OPENBLAS=$(ls "$SCIPY_LIBS"/libscipy_openblas*.so | head -1)
mkdir -p "$OUT/obj"
NLOHMANN=$($PY -c "import site,glob;c=[p for s in site.getsitepackages() for p in glob.glob(s+'/include/cudnn_frontend/thirdparty/nlohmann')];print(c[0] if c else '')")
CXX="g++ -std=c++20 -O2 -fopenmp -fPIC -I$HERE/ref_shim -I$REF/include -I$REF/src -w"
SRCS="core sampler spectra harvest solver reference synth als planner"
TESTS="test_core test_sampler test_spectra test_solver test_synth test_planner"
GLUE_DEFS=""
if [ -n "$NLOHMANN" ] && [ -f "$NLOHMANN/json.hpp" ]; then
  CXX="$CXX -I$NLOHMANN"
  SRCS="$SRCS io"
  TESTS="$TESTS test_io"
  GLUE_DEFS="-DREF_HAVE_IO=1"
else
  echo "build_ref: nlohmann/json.hpp not found; io.cpp not built"
fi
objs=()
for s in $SRCS; do
  o="$OUT/obj/$s.o"
  if [ ! -f "$o" ] || [ "$REF/src/$s.cpp" -nt "$o" ] || [ "$HERE/ref_shim/Eigen/Dense" -nt "$o" ]; then
    $CXX -c "$REF/src/$s.cpp" -o "$o" &
  fi
  objs+=("$o")
done
wait
if [ ! -f "$OUT/libref.so" ] || [ "$HERE/ref_glue.cpp" -nt "$OUT/libref.so" ] || [ "$(ls -t "$OUT"/obj/*.o | head -1)" -nt "$OUT/libref.so" ]; then
  $CXX $GLUE_DEFS -shared -o "$OUT/libref.so" "$HERE/ref_glue.cpp" "${objs[@]}" "$OPENBLAS" -Wl,-rpath,"$SCIPY_LIBS"
fi
# the reference's own unit suites, as oracle self-checks (oracle/_ref/test_*)
for t in $TESTS; do
  if [ ! -f "$OUT/$t" ] || [ "$REF/tests/$t.cpp" -nt "$OUT/$t" ] || [ "$OUT/libref.so" -nt "$OUT/$t" ]; then
    $CXX -I"$REF/tests" -o "$OUT/$t" "$REF/tests/$t.cpp" "${objs[@]}" "$OPENBLAS" -Wl,-rpath,"$SCIPY_LIBS" &
  fi
done
wait
echo "build_ref: ok ($OUT)"
# The reference's own unit suites compiled against the B200 DROP-IN instead of
# the reference library: include/rsm_gpu ahead of everything (its rsm/*.hpp
# forward to include/rsm_gpu/rsm.hpp), linked to librsm_b200.so. Run on a GPU
# by tests/test_cpp_dropin.py (oracle/_ref/dropin_test_*).
LIBDIR="$(cd "$HERE/.." && pwd)/paper_1411_0814_b200"
DROPIN="$(cd "$HERE/.." && pwd)/include/rsm_gpu"
if [ -f "$LIBDIR/librsm_b200.so" ]; then
  for t in test_core test_sampler test_spectra test_solver; do
    exe="$OUT/dropin_$t"
    if [ ! -f "$exe" ] || [ "$REF/tests/$t.cpp" -nt "$exe" ] || [ "$DROPIN/rsm.hpp" -nt "$exe" ] || [ "$LIBDIR/librsm_b200.so" -nt "$exe" ]; then
      g++ -std=c++20 -O1 -w -I"$DROPIN" -I"$HERE/ref_shim" -I"$REF/tests" -o "$exe" "$REF/tests/$t.cpp" \
        -L"$LIBDIR" -lrsm_b200 -Wl,-rpath,'$ORIGIN/../../paper_1411_0814_b200' "$OPENBLAS" -Wl,-rpath,"$SCIPY_LIBS" &
    fi
  done
  wait
  echo "build_ref: drop-in suites ok"
fi
