#!/bin/bash
# Build a diagnostic variant of the C-ABI library: tools/build_variant.sh <name> <nvcc flags...>
# -> paper_1811_01532_b200/_lib/libwapb200_<name>.so (load with WAP_LIB_VARIANT=<name>)
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_1811_01532_b200
OBJ=$PKG/_lib/obj_$name
mkdir -p "$OBJ"
for f in "$PKG"/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I"$ROOT/include" -I"$PKG/csrc" "$@" -c "$f" -o "$OBJ/$(basename "${f%.cu}").o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$PKG/_lib/libwapb200_$name.so" "$OBJ"/*.o
rm -rf "$OBJ"
