#!/bin/bash
# A/B the bench over tools/variants/*.so (each copied over the in-tree lib in turn)
cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
for v in tools/variants/*.so; do
  cp $v paper_1807_07914_b200/libbmps.so
  ./tools/sweep_params.sh "${1:-jac_ws=1}" | sed "s|^|$(basename $v): |"
done
cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
