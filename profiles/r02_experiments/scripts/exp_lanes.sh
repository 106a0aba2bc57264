# scheduling knob matrix on the C2 batch (tools/batch.py 24), K1s for every pair
O=gpurun_out
HAP_EXTRA_NVCC_FLAGS="-DHAP_K1S_MIN_ELEMS=0" python paper_2605_08048_b200/build.py --force
for sh in 0 1; do
for lanes in 2 3; do
for k2 in 0 6 8; do
  echo "shared=$sh lanes=$lanes k2cap=$k2: $(HAP_SHARED=$sh HAP_LANES=$lanes HAP_K2_MAX_CTAS=$k2 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e2_matrix.log
done; done; done
