O=gpurun_out
for v in "" "-DHAP_K3_EB_CHEAP" "-DHAP_K3_EB_ZERO" ""; do
HAP_EXTRA_NVCC_FLAGS="$v" python paper_2605_08048_b200/build.py --force > /dev/null
echo "[$v]: $(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k3_maskgemm python tools/batch.py 12 1 2>/dev/null | grep k3_maskgemm | awk -F'","' '{print $NF}' | tr -d '"' | python3 -c 'import sys; v=[float(x) for x in sys.stdin.read().split()]; print(len(v), sum(v)/len(v))')" >> $O/e31_eb.log
done
