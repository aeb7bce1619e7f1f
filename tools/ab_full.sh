#!/bin/bash
# per variant in tools/variants: bench value / single layer / cfg3 / cfg4 and cfg1 / cfg5 end to end
cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
for v in tools/variants/*.so; do
  cp $v paper_1807_07914_b200/libbmps.so
  echo "$(basename $v): $(./tools/sweep_small.sh jac_cluster=-1 | sed 's/^.*-> //') | $(python tools/config_times.py cfg1 cfg5 2>/dev/null | tail -1)"
done
cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
