# A/B of the round-2 changes to K3 (serialised K3 time per wave of 3 C2 tests, ncu durations)
O=gpurun_out
run() { echo "$1: $(env $2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k3_maskgemm python tools/batch.py 12 1 2>/dev/null | grep k3_maskgemm | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') | $(env $2 python tools/batch.py 48 5 | head -1)" >> $O/e28_k3reg.log; }
for v in "" "-DHAP_K3_NO_GRAM" "-DHAP_K3_NO_EBOUND" "-DHAP_K3_NO_GRAM -DHAP_K3_NO_EBOUND"; do
  HAP_EXTRA_NVCC_FLAGS="$v" python paper_2605_08048_b200/build.py --force > /dev/null
  run "flags[$v] carve=max" "HAP_X=1"
  [ -z "$v" ] && run "flags[$v] carve=default" "HAP_K3_CARVE=0"
done
python paper_2605_08048_b200/build.py --force > /dev/null
