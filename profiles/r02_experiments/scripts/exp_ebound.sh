# the tie-band error bound in fp32: K3 time per wave (ncu) and the C2 batch; GPU tests
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q -x > $O/e30_gt.log 2>&1
echo "noinline logs: $(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k3_maskgemm python tools/batch.py 12 1 2>/dev/null | grep k3_maskgemm | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') | $(python tools/batch.py 48 5 | head -1)" >> $O/e30_ebound.log
timeout 600 python tests/study_near1.py > $O/e30_near1.log 2>&1
