# batch e2e legs with an untimed warm-up pass (C5, C4), then C3
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 > $O/e57_bench_c5.log 2>&1
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > $O/e57_bench_c4.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > $O/e57_bench_c3.log 2>&1
