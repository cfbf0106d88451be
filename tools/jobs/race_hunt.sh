# hunt the intermittent cfg5_3 count mismatch: benches then the golden sequence, current and older builds
for v in cur r9ad predrs cur; do
  if [ $v = cur ]; then unset KM_LIB_VARIANT; else export KM_LIB_VARIANT=$v; fi
  python bench.py --steps 20 --warmup 5 > /dev/null 2>&1
  echo "== $v"; timeout 600 python tools/stress_sequence.py 2
done
