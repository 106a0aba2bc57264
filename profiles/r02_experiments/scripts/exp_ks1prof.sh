O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k1s_stats_warp|k1s_xform_lean|k1s_coef" -s 9 -c 3 -o $O/e13_k1 python tools/batch.py 6 1 > $O/e13_ncu.log 2>&1
