# C3 e2e variance: bench.py c3 three times on one box, the standalone probe between
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2 3; do
  timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench c3', d['value'], d['e2e']['value'])" >> $O/e56.log 2>&1
  python tools/e2e_probe.py >> $O/e56.log 2>&1
done
