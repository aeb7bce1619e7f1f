for v in "$@"; do
  fails=0
  for k in 1 2 3 4 5 6; do
    BMPS_LIB=tools/variants/$v.so timeout 200 python tools/debug_stress.py 25 cfg4only > gpurun_out/stress_${v}_$k.out 2>&1 || fails=$((fails+1))
  done
  echo "$v: $fails failures of 6"; grep -h "claim check" gpurun_out/stress_${v}_*.out | sort | uniq | head -3
done
