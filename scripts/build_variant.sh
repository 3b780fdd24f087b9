#!/bin/bash
# A/B experiment build: copies csrc/ to /tmp/pfe_variant_<name>, applies the
# given sed expression to the given file, builds lib_<name>/libpfe_b200.so
# in-tree (loaded with PFE_LIB_VARIANT=<name>).
# usage: scripts/build_variant.sh <name> <file> '<sed expr>'
set -e
name=$1; file=$2; expr=$3
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/tmp/pfe_variant_$name
rm -rf $SRC; cp -r $ROOT/paper_1612_06496_b200/csrc $SRC
sed -i "$expr" $SRC/$file
mkdir -p $SRC/obj $ROOT/paper_1612_06496_b200/lib_$name
FL="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -fmad=false -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -I$ROOT/include -I$SRC"
for f in $SRC/*.cu; do nvcc $FL -c $f -o $SRC/obj/$(basename $f .cu).o & done
for f in $SRC/*.cpp; do g++ -std=c++17 -O3 -fPIC -I$ROOT/include -I$SRC -c $f -o $SRC/obj/$(basename $f .cpp).o & done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/paper_1612_06496_b200/lib_$name/libpfe_b200.so $SRC/obj/*.o -lpthread -ldl
echo built $ROOT/paper_1612_06496_b200/lib_$name/libpfe_b200.so
