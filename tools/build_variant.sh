#!/bin/bash
# Build a compile-time variant of the library for an A/B run (builder tool):
#   tools/build_variant.sh NAME "-DNSB_X=1 ..." [file.cu ...]
# Recompiles the listed .cu files (default: all) with the extra flags into
# build/var_NAME/ and links tools/ab/libnetsort_NAME.so from them plus the
# default objects; select it at run time with NETSORT_B200_LIB=<path>.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; FLAGS=$2; shift 2
CSRC=$ROOT/paper_2503_05934_b200/csrc
OBJ=$ROOT/build/obj
VOBJ=$ROOT/build/var_$NAME
mkdir -p "$VOBJ" "$ROOT/tools/ab"
make -s -C "$CSRC" >/dev/null
FILES=${@:-$(cd "$CSRC" && ls *.cu)}
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in $FILES; do
  nvcc $ARCH -O3 -lineinfo -std=c++20 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I"$ROOT/include" $FLAGS -c "$CSRC/$f" -o "$VOBJ/$f.o" &
done
wait
OBJS=""
for o in "$OBJ"/*.o; do
  b=$(basename "$o" .o)
  if [ -f "$VOBJ/$b.o" ]; then OBJS="$OBJS $VOBJ/$b.o"; else OBJS="$OBJS $o"; fi
done
nvcc $ARCH -shared -cudart static -o "$ROOT/tools/ab/libnetsort_$NAME.so" $OBJS \
  -Xlinker -z,defs -lpthread -ldl -lrt
echo "$ROOT/tools/ab/libnetsort_$NAME.so"
