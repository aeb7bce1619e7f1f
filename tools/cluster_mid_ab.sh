# Cluster-2 visits vs single-CTA visits at intermediate batch sizes (chi=256 steady-state step).
for r in 2 3 4 6 8; do
  for p in "jac_cluster=0" "jac_cluster=2"; do
    echo "replicas=$r $p: $(BMPS_PARAMS=$p python tools/profile_step.py --replicas $r 2>&1 | grep -E 'step ms|updates' | tr '\n' ' ')"
  done
done
