#!/bin/bash
# Build libdndc.so with extra nvcc defines into variants/<name>.so (A/B timing:
# DNDC_LIB_PATH=variants/<name>.so).  Usage: tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
NAME=$1; shift
mkdir -p variants
cd paper_2007_13552_b200/csrc
make -j8 BUILD=../../build_var/$NAME OUT=../../variants/$NAME.so EXTRA="$*" > /dev/null
