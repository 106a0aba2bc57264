# K1 at C3: + batched P3 passes, batched u staging in KS2
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests -m gpu -q -x > $O/e38_gt.log 2>&1
python tools/k1_probe.py > $O/e38_probe.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k1s python tools/k1_ncu.py 5000 4096 3 > $O/e38_launch.csv 2>&1
echo "c2: $(python tools/batch.py 48 5 | head -1)" >> $O/e38_batch.log
echo "c4: $(HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e38_batch.log
echo "C3: $(python tools/config.py C3 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"], d["phase_ms_serialised"])')" >> $O/e38_batch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1s -s 3 -c 3 -o $O/e38_full python tools/k1_ncu.py 5000 4096 3 > $O/e38_full.log 2>&1
