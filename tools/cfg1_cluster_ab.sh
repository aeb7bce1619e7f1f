for p in "" "jac_cluster=0" "jac_cluster=2" "jac_cluster=4" ""; do
  echo "== '$p' $(BMPS_PARAMS=$p python tools/config_times.py cfg1 cfg1 2>&1 | grep '^cfg1' | cut -c1-60 | tr '\n' ' ')"
done
