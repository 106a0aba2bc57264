# A/B in one call: KS2<true> with u aliasing xbar (64 KB smem, 3 CTAs/SM) and 8 steps in flight (new) vs HEAD
O=gpurun_out
for rep in 1 2; do
for v in base new; do
  echo "== $v rep $rep" >> $O/e58_ab.log
  HAP_LIB_VARIANT=$v python tools/k1_probe.py >> $O/e58_ab.log 2>&1
done
done
HAP_LIB_VARIANT=new timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k1s_coef python tools/k1_ncu.py 5000 4096 3 > $O/e58_new.csv 2>&1
HAP_LIB_VARIANT=base timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k1s_coef python tools/k1_ncu.py 5000 4096 3 > $O/e58_base.csv 2>&1
HAP_LIB_VARIANT=new timeout 900 python -m pytest tests -m gpu -q -x -k "pooled or stream_align or fuzz or wide or config3" > $O/e58_gt.log 2>&1
