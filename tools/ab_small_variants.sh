#!/bin/bash
shopt -s nullglob
cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
./tools/sweep_small.sh tol_factor=4 | sed 's/^/current: /'
for v in tools/variants/*.so; do
  cp $v paper_1807_07914_b200/libbmps.so
  ./tools/sweep_small.sh tol_factor=4 | sed "s|^|$(basename $v): |"
done
cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
./tools/sweep_small.sh tol_factor=4 | sed 's/^/current again: /'
