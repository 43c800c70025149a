#!/bin/bash
# A/B sweep of libkkspgemm.so build variants (build/variants/<name>/libkkspgemm.so,
# built here with different -D settings) on one GPU box: each variant is copied
# over the in-tree library and the given command is run.
#   bash scripts/variant_sweep.sh "python scripts/slab_prof.py 20" p512x3 p1024x2 ...
cmd=$1; shift
lib=paper_1801_03065_b200/libkkspgemm.so
cp $lib /tmp/libkkspgemm.orig.so
for v in "$@"; do
    cp build/variants/$v/libkkspgemm.so $lib
    echo "=== $v"
    timeout 900 $cmd 2>&1 | tail -30
done
cp /tmp/libkkspgemm.orig.so $lib
