#!/bin/bash
# Experiments only: times tools/sweep.py on each build/variants/libmpkg_<name>.so (swapped in for
# the in-tree library on the GPU box's scratch copy).   tools/variant_sweep.sh "name1 name2" <sweep args>
names=$1; shift
cp paper_2309_02228_b200/libmpkg.so /tmp/libmpkg_base.so
for v in $names; do
  if [ "$v" = base ]; then cp /tmp/libmpkg_base.so paper_2309_02228_b200/libmpkg.so
  else cp build/variants/libmpkg_$v.so paper_2309_02228_b200/libmpkg.so; fi
  echo "== variant $v"
  python tools/sweep.py "$@" 2>&1 | grep -v "^#" | tail -8
done
cp /tmp/libmpkg_base.so paper_2309_02228_b200/libmpkg.so
