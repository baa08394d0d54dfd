#!/bin/bash
# build a variant of the library with extra nvcc flags into exp/<name>/
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
ROOT=$(cd $(dirname $0)/.. && pwd)
NAME=$1; shift
mkdir -p $ROOT/exp/$NAME
make -s -j16 -C $ROOT/paper_1607_04808_b200/csrc OBJ=$ROOT/exp/$NAME/build OUT=$ROOT/exp/$NAME/libfse_b200.so EXTRA="$*" 2>&1 | grep -E "error" || true
ls -la $ROOT/exp/$NAME/libfse_b200.so
