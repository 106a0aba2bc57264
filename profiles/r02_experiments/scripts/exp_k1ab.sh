# A/B in one call: base = HEAD K1, new = P3 in KS2 + one barrier per KS1 item + KS2 without a
# second wave + batched u staging + L2 prefetch of X rows before the PDL wait
O=gpurun_out
for rep in 1 2; do
for v in base new; do
  echo "== $v rep $rep" >> $O/e43_ab.log
  HAP_LIB_VARIANT=$v python tools/k1_probe.py >> $O/e43_ab.log 2>&1
  echo "c2: $(HAP_LIB_VARIANT=$v python tools/batch.py 48 5 | head -1)" >> $O/e43_ab.log
  echo "c4: $(HAP_SIZES=c4 HAP_LIB_VARIANT=$v python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e43_ab.log
done
done
