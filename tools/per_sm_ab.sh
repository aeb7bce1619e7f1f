for r in 2 3 4; do for k in 1 2 3 4; do echo "replicas=$r per_sm=$k: $(BMPS_PARAMS=jac_per_sm=$k python tools/profile_step.py --replicas $r 2>&1 | grep -E 'step ms')"; done; done
