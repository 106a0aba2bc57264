# host inputs: one H2D copy per wave for consecutive packed pairs; GPU tests + bench (e2e) twice
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/e52_gt.log 2>&1
timeout 600 python bench.py > $O/e52_bench_c2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > $O/e52_bench_c2b.log 2>&1
