#!/usr/bin/env bash
# Builds the test oracles (TEST INFRASTRUCTURE ONLY):
#   oracle/_build/libegt_oracle.so  -- the C restatement (oracle/egt_oracle.c)
#   oracle/_ref/libegt_ref.so       -- the UNMODIFIED reference hot-path
#       translation units (packed.cpp, compress.cpp, egtq_io.cpp, io.cpp,
#       model.cpp, decode.cpp), compiled straight from /root/reference
#       against oracle/shim/Eigen, plus oracle/ref/*.cpp (extern "C" wrappers).
# The reference build is the CMake Release default (-O3 -DNDEBUG, no -march),
# so no FMA contraction happens on either side.  When /root/reference is
# absent (the GPU box) the prebuilt oracle/_ref/libegt_ref.so is used as is.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${EGT_REFERENCE:-/root/reference}/proj"
mkdir -p "$HERE/_build" "$HERE/_ref"

gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared -Wall -Wextra \
    -o "$HERE/_build/libegt_oracle.so" "$HERE/egt_oracle.c" -lm

if [[ -d "$REF/src" ]]; then
  g++ -std=gnu++20 -O3 -DNDEBUG -ffp-contract=off -fopenmp -fPIC -shared -w \
      -I"$HERE/shim" -I"$REF/include" \
      -o "$HERE/_ref/libegt_ref.so" \
      "$REF/src/packed.cpp" "$REF/src/compress.cpp" "$REF/src/egtq_io.cpp" "$REF/src/io.cpp" \
      "$REF/src/model.cpp" "$REF/src/decode.cpp" \
      "$HERE/ref/ref_capi.cpp" "$HERE/ref/ref_model_capi.cpp" -lpthread
  echo "built $HERE/_ref/libegt_ref.so from $REF/src"
else
  echo "reference tree absent; keeping prebuilt $HERE/_ref/libegt_ref.so" >&2
fi
