#!/bin/bash
# Build an experimental variant of libdis_b200.so with extra nvcc flags into
# exp_so/libdis_<tag>.so (load it with DIS_B200_LIB=exp_so/libdis_<tag>.so).
# usage: tools/build_variant.sh <tag> "<extra nvcc flags>"
set -e
TAG=$1
EXTRA=$2
REPO=$(cd "$(dirname "$0")/.." && pwd)
TMP=/tmp/dis_variant_$TAG
rm -rf $TMP && mkdir -p $TMP/pkg/csrc $TMP/include $REPO/exp_so
cp $REPO/paper_1603_03590_b200/csrc/*.cu $REPO/paper_1603_03590_b200/csrc/*.cuh $REPO/paper_1603_03590_b200/csrc/Makefile $TMP/pkg/csrc/
cp $REPO/include/*.h $TMP/include/
make -s -C $TMP/pkg/csrc -j8 EXTRA="$EXTRA" LIB=$REPO/exp_so/libdis_$TAG.so >/dev/null
echo $REPO/exp_so/libdis_$TAG.so
