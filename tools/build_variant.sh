#!/bin/bash
# build_variant.sh NAME "EXTRA_NVFLAGS" [objects to rebuild, default: all]
#   -> paper_2406_06911_b200/libasyncdiff_b200.NAME.so (A/B tooling; select with ADX_LIB_VARIANT=NAME).
# Objects go to csrc/build_NAME; the listed ones (e.g. "tc_attn") are rebuilt with the flags, the rest
# are copied from the product build.
set -e
cd "$(dirname "$0")/../paper_2406_06911_b200/csrc"
name=$1; flags=$2; objs=$3
rm -rf build_$name && mkdir -p build_$name
if [ -n "$objs" ]; then
  cp -p build/*.o build_$name/
  for o in $objs; do rm -f build_$name/$o.o; done
fi
make -s -j8 OUT=../libasyncdiff_b200.$name.so EXTRA_NVFLAGS="$flags" BUILD=build_$name
