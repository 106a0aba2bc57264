O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > $O/e6_gt.log 2>&1
echo "c2: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e6_batch.log
echo "c2 shared: $(HAP_SHARED=1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e6_batch.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e6_launch.csv python tools/batch.py 6 1 > /dev/null 2>&1
timeout 600 python tools/gram_bench.py $O/r02_gram.json > $O/e6_gram.log 2>&1
