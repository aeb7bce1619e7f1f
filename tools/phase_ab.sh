#!/bin/bash
# phase timers for the current and the previous (HEAD) Jacobi build
for v in libbmps_timers.so libbmps_timers_old.so; do
  sed "s|tools/libbmps_timers.so|tools/$v|" tools/phase_times.py > /tmp/pt.py
  echo "== $v"; python /tmp/pt.py
done
