# K1 time attribution: full (0), no write-back (2), count-only (3), stream-only (1)
for sp in ${@:-0.99 0.9999}; do
  for x in 0 2 3 1; do
    PULSE_K1_EXPERIMENT=$x timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1
  done
done
