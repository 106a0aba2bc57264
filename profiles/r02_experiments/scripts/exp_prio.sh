O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_gram.py -x -q > $O/e4_gram.log 2>&1
for pr in 1 0; do
echo "prio=$pr c2: $(HAP_LANE_PRIO=$pr python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e4_batch.log
echo "prio=$pr c2 shared: $(HAP_LANE_PRIO=$pr HAP_SHARED=1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e4_batch.log
echo "prio=$pr c4: $(HAP_LANE_PRIO=$pr HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e4_batch.log
echo "prio=$pr c5: $(HAP_LANE_PRIO=$pr HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e4_batch.log
done
python tools/batch.py 24 3 > $O/e4_spans.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e4_launch.csv python tools/batch.py 6 1 > /dev/null 2>&1
