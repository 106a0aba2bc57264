# A/B in one call: base = HEAD K1; new3 = P3 in KS2 for d > 1024 streaming pairs (KS2 grid cap,
# 16 steps in flight, L2 prefetch before the PDL wait), one barrier per KS1 item, batched P3
# loads; the warp-per-row KS1 pairs (d <= 1024) keep HEAD's KS1 P3 and KS2
O=gpurun_out
for rep in 1 2; do
for v in base new3; do
  echo "== $v rep $rep" >> $O/e45_ab.log
  HAP_LIB_VARIANT=$v python tools/k1_probe.py >> $O/e45_ab.log 2>&1
  echo "c2: $(HAP_LIB_VARIANT=$v python tools/batch.py 48 5 | head -1)" >> $O/e45_ab.log
  echo "c4: $(HAP_SIZES=c4 HAP_LIB_VARIANT=$v python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e45_ab.log
  echo "c5: $(HAP_SIZES=c5 HAP_LIB_VARIANT=$v python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e45_ab.log
done
done
