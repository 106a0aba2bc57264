#!/bin/bash
# Round-2 final measurement pass (one B200): GPU tests, bench lines for c2 (default) / c3 / c4 /
# c5 and the reference arm, the ncu launch list of the default bench, ncu --set full of K3 and
# K2 in the C2 pipeline.  Outputs under gpurun_out/m6_*; also the K1 launch list at C3.
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q > $O/m6_gt.log 2>&1
timeout 600 python bench.py > $O/m6_bench_c2.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > $O/m6_bench_c3.log 2>&1
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > $O/m6_bench_c4.log 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 > $O/m6_bench_c5.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/m6_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/m6_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/m6_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3_maskgemm|k2_perm_fy32" -s 12 -c 2 \
  -o $O/m6_k3k2 python tools/batch.py 12 1 > $O/m6_ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  -k regex:k1s python tools/k1_ncu.py 5000 4096 3 > $O/m6_k1_c3_launch.csv 2>&1
timeout 600 python tools/k1_probe.py > $O/m6_k1_probe.log 2>&1
