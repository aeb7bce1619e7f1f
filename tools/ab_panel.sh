#!/bin/bash
# QR panel kernel time of one bench step (ncu launch list) and cfg5 evolve time per variant
cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
for v in tools/variants/*.so; do
  cp $v paper_1807_07914_b200/libbmps.so
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:qr_panel --csv \
    --log-file /tmp/pl.csv python tools/profile_step.py --replicas 16 > /dev/null 2>&1
  p=$(python tools/launch_summary.py /tmp/pl.csv | grep total | awk '{print $3}')
  c5=$(python tools/config_times.py cfg5 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['cfg5']['evolve_s'])")
  echo "$(basename $v): panels $p ms per bench step, cfg5 evolve $c5 s"
done
cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
