#!/bin/bash
# bench variants incl. the single-circuit layer and the cfg3 circuit; one line per variant
for v in "$@"; do
  args=""
  for kv in $(echo $v | tr ',' ' '); do args="$args --param $kv"; done
  val=$(python bench.py --steps 2 --warmup 2 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'layer', round(d['single_circuit_layer']['updates_per_s'],1), 'cfg3 %.3f s' % d['cfg3_full_circuit']['s'], 'cfg4', round(d['cfg4_circuits']['circuits_per_s'],1))")
  echo "$v -> $val"
done
