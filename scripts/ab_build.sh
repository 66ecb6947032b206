#!/bin/bash
# A/B builds for measurement: compiles one csrc file with a Python text patch applied and links it
# with the other objects of the current build into csrc/build_ab/libmont_<tag>.so; select it at run
# time with MONT_LIB_AB=<tag> (paper_1609_00999_b200/__init__.py).  Both builds then run on the
# same box in one gpurun call, so the comparison does not mix GPUs or clocks.
#   [EXTRA_FLAGS="-Xptxas ..."] scripts/ab_build.sh <tag> <file.cu> <python-expr transforming the source string s>
set -eu
TAG=$1; SRC=$2; EXPR=$3
CS=$(cd "$(dirname "$0")/../paper_1609_00999_b200/csrc" && pwd)
make -C "$CS" -j8 > /dev/null
mkdir -p "$CS/build_ab"
TMP="$CS/_ab_${TAG}_$SRC"  # next to the original, so its relative #includes resolve
trap 'rm -f "$TMP"' EXIT
python3 - "$CS/$SRC" "$TMP" "$EXPR" <<'EOF'
import os
import sys
src, dst, expr = sys.argv[1:]
s = open(src).read()
t = eval(expr)
assert t != s or os.environ.get("EXTRA_FLAGS"), "patch changed nothing"
open(dst, "w").write(t)
EOF
NVCC=/usr/local/cuda/bin/nvcc
FLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -DMONT_BUILD_ARCH=100 --expt-relaxed-constexpr -I$CS ${EXTRA_FLAGS:-}"
$NVCC $FLAGS -c "$TMP" -o "$CS/build_ab/${TAG}_${SRC%.cu}.o"
OBJS=$(ls "$CS"/build/*.o | grep -v "/${SRC%.cu}.o$")
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$CS/build_ab/libmont_$TAG.so" $OBJS "$CS/build_ab/${TAG}_${SRC%.cu}.o"
echo "built $CS/build_ab/libmont_$TAG.so"
