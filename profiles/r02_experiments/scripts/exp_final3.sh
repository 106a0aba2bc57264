# final check of HEAD: build, GPU tests, smoke, default bench line, c3 line, K1 launch list at C3
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/z_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/z_gt.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/z_smoke.log 2>&1
timeout 600 python bench.py > $O/z_bench_c2.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > $O/z_bench_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:k1s python tools/k1_ncu.py 5000 4096 3 > $O/z_k1_c3_launch.csv 2>&1
