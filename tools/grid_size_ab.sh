for g in 96 120 148 180 222; do echo "cfg3 grid=$g: $(BMPS_PARAMS=jac_per_sm=-$g python tools/cfg3_layer_times.py '' '' 2>&1 | tail -1)"; done
for g in 112 128 148; do echo "r1 grid=$g: $(BMPS_PARAMS=jac_per_sm=-$g python tools/profile_step.py --replicas 1 2>&1 | grep 'step ms')"; done
for g in 222 260 296 340; do echo "r2 grid=$g: $(BMPS_PARAMS=jac_per_sm=-$g python tools/profile_step.py --replicas 2 2>&1 | grep 'step ms')"; done
for g in 370 444 520; do echo "r3 grid=$g: $(BMPS_PARAMS=jac_per_sm=-$g python tools/profile_step.py --replicas 3 2>&1 | grep 'step ms')"; done
