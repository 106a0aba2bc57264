O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q -x > $O/e32_gt.log 2>&1
echo "branch-free bound: $(timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k3_maskgemm python tools/batch.py 12 1 2>/dev/null | grep k3_maskgemm | awk -F'","' '{print $NF}' | tr -d '"' | python3 -c 'import sys; v=[float(x) for x in sys.stdin.read().split()]; print(len(v), sum(v)/len(v))') | $(python tools/batch.py 48 5 | head -1)" >> $O/e32_eb.log
timeout 600 python tests/study_near1.py > $O/e32_near1.log 2>&1
