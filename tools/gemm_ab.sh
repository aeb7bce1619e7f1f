# A/B of GEMM-engine builds: K2/K4 launch times of one bench step (ncu) and K5/K6 by events.
for v in "" tools/variants/gemm_minb1.so tools/variants/gemm_old.so; do
  echo "== lib=${v:-default}"
  BMPS_LIB=$v ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:"theta_kernel|gemm_kernel" --csv --log-file gpurun_out/gemm_ab.csv python tools/profile_step.py --replicas 8 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/gemm_ab.csv 2>/dev/null | sed -n 2,5p
  BMPS_LIB=$v python tools/kernel_rooflines.py --launch-list gpurun_out/gemm_ab.csv 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items():
    if isinstance(v,dict) and ('frac_fp64' in v or 'frac_hbm' in v): print(k, {x:round(y,3) for x,y in v.items() if isinstance(y,float)})"
done
