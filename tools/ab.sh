#!/bin/bash
# A/B of library builds on the GPU box: tools/ab.sh CMD... runs CMD once per
# abvar/<variant>.so (copied into the package), twice round-robin.
set -u
lib=paper_2512_11727_b200/libecco_b200.so
cp $lib /tmp/ab_orig.so
for round in 1 2; do
  for v in ${AB_DIR:-abvar}/*.so; do
    cp "$v" $lib
    echo "== $(basename $v .so): $("$@" 2>&1 | tail -1)"
  done
done
cp /tmp/ab_orig.so $lib
