#!/bin/bash
# Build compile-time variants of libtk_b200.so into variants/<name>.so (for A/B runs on the GPU box:
#   for v in variants/*.so; do cp $v paper_2510_01495_b200/libtk_b200.so; python bench.py ...; done)
# usage: tools/variants.sh name1 "-DFOO=1" name2 "-DFOO=2" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -C paper_2510_01495_b200/csrc -j4 XFLAGS="$flags" BUILD=/tmp/tkvar_$name OUT=$PWD/variants/$name.so
  echo "built variants/$name.so ($flags)"
done
