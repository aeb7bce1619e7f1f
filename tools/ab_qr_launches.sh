#!/bin/bash
# per-kernel launch-list time of one 16-replica bench step for the in-tree lib and tools/variants/*.so
shopt -s nullglob
cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
one() {
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file /tmp/ll.csv python tools/profile_step.py --replicas 16 > /dev/null 2>&1
  python tools/launch_summary.py /tmp/ll.csv | grep -E "qr_|dq_|total" | sed "s|^|$1: |"
}
one current
for v in tools/variants/*.so; do cp $v paper_1807_07914_b200/libbmps.so; one $(basename $v); done
cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
