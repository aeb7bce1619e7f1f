#!/bin/bash
# A/B: run the bench with the in-tree lib and with alternative .so files (tools/variants/*.so)
./tools/sweep_params.sh tol_factor=4 | sed 's/^/current: /'
for v in tools/variants/*.so; do
  cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
  cp $v paper_1807_07914_b200/libbmps.so
  ./tools/sweep_params.sh tol_factor=4 | sed "s|^|$(basename $v): |"
  cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
done
./tools/sweep_params.sh tol_factor=4 | sed 's/^/current again: /'
