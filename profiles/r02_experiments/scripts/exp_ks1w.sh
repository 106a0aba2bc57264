O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > $O/e11_gt.log 2>&1
echo "c2: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e11_batch.log
echo "c2 shared: $(HAP_SHARED=1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e11_batch.log
echo "c4: $(HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e11_batch.log
echo "c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e11_batch.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e11_launch.csv python tools/batch.py 6 1 > /dev/null 2>&1
python tools/config.py C1 > $O/e11_c1.log 2>&1
