O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for rep in 1 2; do
for ln in 2 3; do
echo "lanes=$ln c2: $(HAP_LANES=$ln python tools/batch.py 96 5 2>&1 | head -1)" >> $O/e27_lanes.log
echo "lanes=$ln c2sh: $(HAP_LANES=$ln HAP_SHARED=1 python tools/batch.py 96 5 2>&1 | head -1)" >> $O/e27_lanes.log
echo "lanes=$ln c5: $(HAP_LANES=$ln HAP_SIZES=c5 python tools/batch.py 192 3 2>&1 | head -1)" >> $O/e27_lanes.log
echo "lanes=$ln c4: $(HAP_LANES=$ln HAP_SIZES=c4 python tools/batch.py 192 3 2>&1 | head -1)" >> $O/e27_lanes.log
done; done
