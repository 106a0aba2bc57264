python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1 || echo BUILD FAIL
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
HAP_SIZES=c4 python tools/batch.py 96 3 2>&1 | grep "^batch"
python tools/config.py C3 > gpurun_out/c3.json 2>&1; tail -1 gpurun_out/c3.json | cut -c1-160
python tools/config.py C1 > gpurun_out/c1.json 2>&1; tail -1 gpurun_out/c1.json | cut -c1-160
python bench.py 2>&1 | tail -1 | cut -c1-120
