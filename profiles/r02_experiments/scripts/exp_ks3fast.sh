# A/B in one call: KS3 (ring) interior tiles without bounds checks (new) vs HEAD (base); tests on new
O=gpurun_out
for rep in 1 2; do
for v in base new; do
  echo "== $v rep $rep" >> $O/e49_ab.log
  HAP_LIB_VARIANT=$v python tools/k1_probe.py >> $O/e49_ab.log 2>&1
done
done
HAP_LIB_VARIANT=new timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k1s_xform python tools/k1_ncu.py 5000 4096 3 > $O/e49_new.csv 2>&1
HAP_LIB_VARIANT=base timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k1s_xform python tools/k1_ncu.py 5000 4096 3 > $O/e49_base.csv 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "pooled or stream_align or fuzz or config3 or wide" > $O/e49_gt.log 2>&1
