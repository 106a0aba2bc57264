O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > $O/e12_gt.log 2>&1
echo "c2: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e12_batch.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e12_launch.csv python tools/batch.py 6 1 > /dev/null 2>&1
python tools/config.py C1 > $O/e12_c1.log 2>&1
