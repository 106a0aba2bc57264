#!/bin/bash
# Round-2 final measurement pass (one B200): GPU tests, bench lines for c2 (default) / c3 / c4 /
# c5 and the reference arm, the ncu launch list of the default bench, ncu --set full of K3 and
# K2 in the C2 pipeline.  Outputs under gpurun_out/m5_*.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q > $O/m5_gt.log 2>&1
timeout 600 python bench.py > $O/m5_bench_c2.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > $O/m5_bench_c3.log 2>&1
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > $O/m5_bench_c4.log 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 > $O/m5_bench_c5.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/m5_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/m5_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/m5_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3_maskgemm|k2_perm_fy32" -s 12 -c 2 \
  -o $O/m5_k3k2 python tools/batch.py 12 1 > $O/m5_ncu_full.log 2>&1
