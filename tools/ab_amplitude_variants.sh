#!/bin/bash
shopt -s nullglob
cp paper_1807_07914_b200/libbmps.so /tmp/cur.so
run() { timeout 300 python tools/kernel_rooflines.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['K6_amplitudes']['launch_ms'],2), 'ms', round(d['K6_amplitudes']['achieved_tflops'],2), 'TF')"; }
echo "current: $(run)"
for v in tools/variants/amp_*.so; do cp $v paper_1807_07914_b200/libbmps.so; echo "$(basename $v): $(run)"; done
cp /tmp/cur.so paper_1807_07914_b200/libbmps.so
