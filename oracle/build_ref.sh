#!/usr/bin/env bash
# SPDX-License-Identifier: Apache-2.0
#
# Compiles the reference CPU implementation directly from its sources under
# /root/reference/proj (read-only; nothing is copied into this repo) into
# oracle/_ref/libhmiref.so, together with oracle/ref_driver.cpp (our extern "C"
# driver). The reference's own CMake cannot configure as shipped (it adds the
# absent tools/ and tests/ directories, proj/CMakeLists.txt:21-22, and lists
# absent scheduler/service/bench sources, proj/src/CMakeLists.txt:18-27), so we
# compile the present translation units by hand with the reference's flags
# (-std=c++20 -O2 -Wall -Wextra -ffp-contract=off; -mavx2 -mfma for the AVX2
# kernel unit, proj/src/CMakeLists.txt:33-36).
#
# Minimal fixes, applied without editing any source:
#   * `-include mutex`: version_tree.cpp and store.cpp use std::unique_lock
#     without including <mutex> (version_tree.cpp:18, store.cpp:10).
#   * adapters/stacked.cpp is left out: `StackedAdapters out;` (stacked.cpp:18)
#     is ill-formed because MatrixBatch has no default constructor
#     (matrix.hpp:52). Nothing on the reference path we drive uses it
#     (higher_stack_forward is the bit-identical per-request path).
set -euo pipefail
REF=${HMI_REFERENCE:-/root/reference/proj}
HERE=$(cd "$(dirname "$0")" && pwd)
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not found at $REF; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$OUT/obj"
CXX=${CXX:-g++}
FLAGS="-std=c++20 -O2 -fPIC -ffp-contract=off -include mutex -I$REF/include -w"
SRCS="io/binary.cpp tensor/matrix.cpp tensor/ops.cpp tensor/kernels.cpp tensor/kernels_scalar.cpp
      transformer/weights.cpp transformer/model.cpp transformer/model_io.cpp plot/table.cpp
      plot/version_tree.cpp plot/retrieval.cpp plot/plot_io.cpp adapters/adapter_set.cpp
      adapters/store.cpp adapters/device_pool.cpp"
OBJS=()
pids=()
for s in $SRCS; do
  o="$OUT/obj/$(echo "$s" | tr '/' '_' | sed 's/\.cpp$/.o/')"
  OBJS+=("$o")
  if [ ! -f "$o" ] || [ "$REF/src/$s" -nt "$o" ]; then
    $CXX $FLAGS -c "$REF/src/$s" -o "$o" &
    pids+=($!)
  fi
done
o="$OUT/obj/tensor_kernels_avx2.o"
OBJS+=("$o")
if [ ! -f "$o" ]; then
  $CXX $FLAGS -mavx2 -mfma -c "$REF/src/tensor/kernels_avx2.cpp" -o "$o" &
  pids+=($!)
fi
for p in "${pids[@]}"; do wait "$p"; done
$CXX $FLAGS -c "$HERE/ref_driver.cpp" -o "$OUT/obj/ref_driver.o"
$CXX -shared -o "$OUT/libhmiref.so" "${OBJS[@]}" "$OUT/obj/ref_driver.o" -lpthread
echo "built $OUT/libhmiref.so"
