# K1 streaming: P3 derived by every KS2 CTA (no KS1 ticket / serial P3 tail)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -x > $O/e40_gt.log 2>&1
python tools/k1_probe.py > $O/e40_probe.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k1s python tools/k1_ncu.py 5000 4096 3 > $O/e40_launch.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k1s python tools/k1_ncu.py 1000 768 3 > $O/e40_launch_c2.csv 2>&1
echo "c2: $(python tools/batch.py 48 5 | head -1)" >> $O/e40_batch.log
echo "c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e40_batch.log
echo "c4: $(HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e40_batch.log
echo "C3: $(python tools/config.py C3 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"], d["phase_ms_serialised"])')" >> $O/e40_batch.log
echo "C1: $(python tools/config.py C1 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"], d["phase_ms_serialised"])')" >> $O/e40_batch.log
HAP_EXTRA_NVCC_FLAGS="-DHAP_EXPERIMENTS" python paper_2605_08048_b200/build.py --force > /dev/null
python tools/ks1trace.py 5000 4096 > $O/e40_ks1trace.log 2>&1
python paper_2605_08048_b200/build.py --force > /dev/null
