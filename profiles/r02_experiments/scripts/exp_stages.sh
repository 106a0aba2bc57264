# K3 ring depth 3 vs 4 (48 KB stages): C3 single test, C2 / C5 batches, K3 per wave
O=gpurun_out
for st in 4 3; do
HAP_EXTRA_NVCC_FLAGS="-DHAP_K3_STAGES=$st" python paper_2605_08048_b200/build.py --force > /dev/null
echo "stages=$st K3/wave: $(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k3_maskgemm python tools/batch.py 12 1 2>/dev/null | grep k3_maskgemm | awk -F'","' '{print $NF}' | tr -d '"' | python3 -c 'import sys; v=[float(x) for x in sys.stdin.read().split()]; print(len(v), sum(v)/len(v))')" >> $O/e35_stages.log
echo "stages=$st c2: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e35_stages.log
echo "stages=$st c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e35_stages.log
echo "stages=$st C3: $(python tools/config.py C3 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"], d["phase_ms_serialised"])')" >> $O/e35_stages.log
done
python paper_2605_08048_b200/build.py --force > /dev/null
