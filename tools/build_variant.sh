#!/bin/bash
# Dev tool: build a variant of libhpcg.so from a patched copy of csrc/.
# usage: build_variant.sh <name> <python-patch-file>  -> tools/var_<name>.so
set -e
name=$1; patch=$2
root=$(cd "$(dirname "$0")/.." && pwd)
d=/tmp/var_$name
rm -rf $d && mkdir -p $d/pkg $d/include
cp -r $root/paper_2311_04517_b200/csrc $d/pkg/csrc && rm -rf $d/pkg/csrc/build
cp -r $root/include/* $d/include/
(cd $d/pkg/csrc && python $patch && make -j8 >/dev/null 2>&1 || (cd $d/pkg/csrc && make 2>&1 | grep error; exit 1))
cp $d/pkg/libhpcg.so $root/tools/var_$name.so
echo built tools/var_$name.so
