#!/bin/bash
# theta / split GEMM kernel times of one bench step (ncu launch list) + bench value per variant
cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
for v in tools/variants/*.so; do
  cp $v paper_1807_07914_b200/libbmps.so
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"theta|gemm" --csv \
    --log-file /tmp/gl.csv python tools/profile_step.py --replicas 16 > /dev/null 2>&1
  echo "== $(basename $v)"; python tools/launch_summary.py /tmp/gl.csv 2>/dev/null | head -5
  ./tools/sweep_params.sh jac_ws=0
done
cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
