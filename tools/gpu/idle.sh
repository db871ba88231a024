for ns in 0 16 32 64 128; do
  PR_PART_IDLE_NS=$ns timeout 60 python tools/k1p_time.py C4 16384 linear 5 2>&1 | tail -1 | sed "s/^/idle_ns=$ns /"
done
