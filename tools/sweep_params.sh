#!/bin/bash
# run bench variants; print value per variant
for v in "$@"; do
  args=""
  for kv in $(echo $v | tr ',' ' '); do args="$args --param $kv"; done
  val=$(python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-circuit $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['gpu_launches'], d['jacobi_sweeps_last_step'])")
  echo "$v -> $val"
done
