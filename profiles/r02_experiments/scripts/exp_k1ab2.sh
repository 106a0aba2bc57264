# A/B in one call: base = HEAD K1, new = P3 in KS2 for every streaming pair (+ KS2 grid cap, batched u staging, L2 prefetch)
# new2 = new with the warp-per-row KS1 keeping its ticketed P3 and the old KS2 grid for those pairs
O=gpurun_out
for rep in 1 2; do
for v in base new new2; do
  echo "== $v rep $rep" >> $O/e44_ab.log
  HAP_LIB_VARIANT=$v python tools/k1_probe.py >> $O/e44_ab.log 2>&1
  echo "c2: $(HAP_LIB_VARIANT=$v python tools/batch.py 48 5 | head -1)" >> $O/e44_ab.log
  echo "c4: $(HAP_SIZES=c4 HAP_LIB_VARIANT=$v python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e44_ab.log
done
done
