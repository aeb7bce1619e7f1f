# Latency-bound regime (one circuit): cluster rules of the Jacobi, short-panel QR kernel.
for p in "$@"; do
  echo "== $p"
  BMPS_PARAMS=$p python tools/config_times.py cfg3 cfg5 cfg1 2>&1 | tail -1 | cut -c1-260
done
