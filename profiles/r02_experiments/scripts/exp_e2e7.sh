# e2e A/B in one call: per-pair H2D copies (base = dfd6d1b host code) vs one copy per wave (new); H2D probe
O=gpurun_out
python tools/pcie_probe.py > $O/e59_e2e.log 2>&1
for rep in 1 2; do
for v in base new; do
  echo "== $v" >> $O/e59_e2e.log
  HAP_LIB_VARIANT=$v python tools/e2e_probe.py >> $O/e59_e2e.log 2>&1
done
done
python tools/pcie_probe.py >> $O/e59_e2e.log 2>&1
