# Why fewer CTAs per SM win in the latency-bound regime: DRAM traffic, L2 hit rate and pipe use of
# the Jacobi launch of one 16-item chi=256 layer at 1 and 4 CTAs per SM.
for k in 1 4; do
  BMPS_PARAMS=jac_per_sm=$k ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__cycles_active.avg --clock-control none --profile-from-start off -k regex:jacobi_dynamic --csv --log-file gpurun_out/mech_$k.csv python tools/profile_step.py --replicas 1 > /dev/null 2>&1
  echo "== jac_per_sm=$k"; python - gpurun_out/mech_$k.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r); h = rows[hi]
for r in rows[hi + 1:]:
    print(r[h.index('Metric Name')], r[h.index('Metric Value')], r[h.index('Metric Unit')])
PY
done
