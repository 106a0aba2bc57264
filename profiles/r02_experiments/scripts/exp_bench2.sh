O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > $O/e9_gt.log 2>&1
timeout 600 python bench.py > $O/e9_bench.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k1s_stats|k1s_xform_lean" -s 6 -c 2 -o $O/e9_k1lean python tools/batch.py 6 1 > $O/e9_ncu.log 2>&1
