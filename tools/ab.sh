#!/bin/bash
# A/B of libbmps builds on the bench (run on a GPU box): tools/ab.sh STEPS variant1 variant2 ...
# "default" = the in-tree build; others = tools/variants/<name>.so (python -m
# paper_1807_07914_b200.build --out tools/variants/<name>.so -D ...). Two passes, interleaved.
STEPS=${1:-10}; shift
for pass in 1 2; do
  for v in "$@"; do
    if [ "$v" = default ]; then L=""; else L=tools/variants/$v.so; fi
    BMPS_LIB=$L timeout 300 python bench.py --steps $STEPS --no-circuit --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/ab_{v}.json"))
    print(v, round(d["value"], 1), "frac", round(d["roofline"]["frac"], 4), "sweeps", d["jacobi_sweeps_last_step"]["mean"],
          "single", round(d["single_circuit_layer"]["updates_per_s"], 1), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(v, "FAILED", e)
PY
  done
done
