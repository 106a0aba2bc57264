# final check of HEAD: build, GPU tests, smoke, default bench line, c3 bench line
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/f_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/f_gt.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/f_smoke.log 2>&1
timeout 600 python bench.py > $O/f_bench_c2.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > $O/f_bench_c3.log 2>&1
