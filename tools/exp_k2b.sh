O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x -k "perm_sets or config1 or config2 or ragged or batch or fuzz or exhaustive or checked" > $O/e18_gt.log 2>&1
echo "c2: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e18_batch.log
echo "c2 shared: $(HAP_SHARED=1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e18_batch.log
echo "c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e18_batch.log
for wm in 2560 4096 6144 10240; do
echo "c4 widemax=$wm: $(HAP_K2_WIDE_MAX_N=$wm HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e18_batch.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/e18_launch.csv python tools/batch.py 6 1 > /dev/null 2>&1
