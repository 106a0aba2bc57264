# wave size (tests per K1/K2/K3 launch) for C5 / C4 / C2: 3 (default) vs 4 vs 2, twice each
O=gpurun_out
for rep in 1 2; do
for w in 3 4 2; do
  echo "wave $w rep $rep c5: $(HAP_WAVE=$w HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e50_wave.log
  echo "wave $w rep $rep c4: $(HAP_WAVE=$w HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e50_wave.log
  echo "wave $w rep $rep c2: $(HAP_WAVE=$w python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e50_wave.log
done
done
