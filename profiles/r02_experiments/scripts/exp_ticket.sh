O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > $O/e5_gt.log 2>&1
echo "c2: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e5_batch.log
echo "c2 shared: $(HAP_SHARED=1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e5_batch.log
echo "c4: $(HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e5_batch.log
echo "c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e5_batch.log
python tools/config.py C1 > $O/e5_c1.log 2>&1
python tools/config.py C3 > $O/e5_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e5_launch.csv python tools/batch.py 6 1 > /dev/null 2>&1
python tools/batch.py 24 3 > $O/e5_spans.log 2>&1
timeout 600 python tools/gram_bench.py $O/r02_gram.json > $O/e5_gram.log 2>&1
