#!/bin/bash
# build a variant library: tools/variant.sh NAME "-DFOO=1 -DBAR=2"  -> paper_2604_03092_b200/lib/NAME/libsurfel2d.so
cd "$(dirname "$0")/.."
make -s -j4 -C paper_2604_03092_b200/csrc OBJDIR=../lib/obj_$1 OUT=../lib/$1/libsurfel2d.so EXTRA="$2" 2>&1 | grep -i "error\|raster_bwd\|fwdILb0ELb0ELb0" | sed 's/_ZN3s2d41_GLOBAL__N__667bc096_9_raster_cu_8d9717f612//'
