#!/bin/bash
# Round-2 measurement pass on one B200 (run through gpurun from the repo root):
# compute-sanitizer memcheck / racecheck / synccheck on the small cases, the default bench
# line, and the ncu launch list of the same command.  Outputs under gpurun_out/.
set -x
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()"
for t in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_case.py > $O/san_$t.log 2>&1
  echo "$t rc=$?" >> $O/san_rc.txt
done
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_case.py quick > $O/san_racecheck.log 2>&1
echo "racecheck rc=$?" >> $O/san_rc.txt
timeout 600 python bench.py > $O/r02_bench_c2.log 2>&1
echo "bench rc=$?" >> $O/san_rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/r02_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/r02_ncu_launch.log 2>&1
echo "ncu rc=$?" >> $O/san_rc.txt
