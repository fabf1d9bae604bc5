#!/bin/bash
# Build a library variant with extra nvcc flags into _variants/<name>.so (for tools/ab.sh).
# usage: tools/variant.sh <name> [-DFLAG ...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
out=/tmp/fsvar_$name
rm -rf $out
make -s -j8 -C $ROOT/paper_2409_08270_b200/csrc OUT=$out EXTRA="$*" > /dev/null
mkdir -p $ROOT/_variants
cp $out/libflashsplat_b200.so $ROOT/_variants/$name.so
grep -h "raster_kernel" -A2 $out/obj/fs_raster.ptxas.txt | grep -o "Used [0-9]* registers.*" | head -2
