O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q > $O/e16_gt.log 2>&1
