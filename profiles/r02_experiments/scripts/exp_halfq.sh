# global finalize queue in K3: tests, K3 per wave (ncu), C2 batch, K3 trace
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q -x > $O/e36_gt.log 2>&1
echo "halfq: $(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k3_maskgemm python tools/batch.py 12 1 2>/dev/null | grep k3_maskgemm | awk -F'","' '{print $NF}' | tr -d '"' | python3 -c 'import sys; v=[float(x) for x in sys.stdin.read().split()]; print(len(v), sum(v)/len(v))') | $(python tools/batch.py 48 5 | head -1)" >> $O/e36_finq.log
echo "c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e36_finq.log
echo "c4: $(HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e36_finq.log
echo "C3: $(python tools/config.py C3 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"], d["phase_ms_serialised"])')" >> $O/e36_finq.log
echo "C1: $(python tools/config.py C1 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"], d["phase_ms_serialised"])')" >> $O/e36_finq.log
HAP_EXTRA_NVCC_FLAGS="-DHAP_EXPERIMENTS" python paper_2605_08048_b200/build.py --force > /dev/null
HAP_TRACE_B=30000 python tools/k3trace.py > $O/e36_k3trace.log 2>&1
python paper_2605_08048_b200/build.py --force > /dev/null
