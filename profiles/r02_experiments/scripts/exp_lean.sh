# lean K1s: GPU tests, C2 batch default/shared, C4/C5 samples, C1 latency (A/B against the
# fused cooperative K1 via HAP_K1S_MIN_ELEMS... not available: lean is the default now)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > $O/e3_gt.log 2>&1
for v in "" ; do
echo "c2 default: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e3_batch.log
echo "c2 shared: $(HAP_SHARED=1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e3_batch.log
echo "c2 3 lanes: $(HAP_LANES=3 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e3_batch.log
echo "c4: $(HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e3_batch.log
echo "c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e3_batch.log
done
python tools/config.py C1 > $O/e3_c1.log 2>&1
python tools/config.py C2 > $O/e3_c2.log 2>&1
python tools/batch.py 24 3 > $O/e3_spans.log 2>&1
