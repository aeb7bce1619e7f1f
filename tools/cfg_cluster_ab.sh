for p in jac_cluster=0 jac_cluster=-1 jac_cluster=2; do
  echo "== $p"; BMPS_PARAMS=$p timeout 300 python tools/config_times.py cfg1 cfg3 cfg5 2>&1 | tail -4
done
timeout 600 ./tools/sweep_small.sh jac_cluster=0 jac_cluster=-1
