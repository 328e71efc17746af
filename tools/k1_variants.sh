# K1 time per variant library (tools/build_variant.sh) at two sparsities
for v in base s4b4 s3b4 s4b5; do
  lib=""; [ "$v" != base ] && lib="PULSE_LIB=/root/repo/variants/$v.so"
  for sp in 0.99 0.9; do
    env $lib timeout 300 python tools/k1_time.py $sp 2>&1 | tail -1 | sed "s/^/$v: /"
  done
done
