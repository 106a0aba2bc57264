# final check after the automatic wave of 4 at N <= 2048: GPU tests, smoke, bench lines c2 / c4 / c5
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/g_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/g_gt.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/g_smoke.log 2>&1
timeout 600 python bench.py > $O/g_bench_c2.log 2>&1
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > $O/g_bench_c4.log 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 > $O/g_bench_c5.log 2>&1
