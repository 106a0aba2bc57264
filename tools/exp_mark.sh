O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q -x > $O/e23_gt.log 2>&1
for mk in 1 0; do
echo "mark=$mk c4: $(HAP_K2_MARK=$mk HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e23_batch.log
echo "mark=$mk n3000: $(HAP_K2_MARK=$mk HAP_SIZES=n3000 python tools/batch.py 12 3 2>&1 | head -1)" >> $O/e23_batch.log
echo "mark=$mk n5000: $(HAP_K2_MARK=$mk HAP_SIZES=n5000 python tools/batch.py 9 3 2>&1 | head -1)" >> $O/e23_batch.log
echo "mark=$mk c3: $(HAP_K2_MARK=$mk python tools/config.py C3 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"], d["phase_ms_serialised"])')" >> $O/e23_batch.log
done
for pw in 2 4; do
echo "mark pw=$pw n5000: $(HAP_K2_PW=$pw HAP_SIZES=n5000 python tools/batch.py 9 3 2>&1 | head -1)" >> $O/e23_batch.log
echo "mark pw=$pw n3000: $(HAP_K2_PW=$pw HAP_SIZES=n3000 python tools/batch.py 12 3 2>&1 | head -1)" >> $O/e23_batch.log
done
