# host->device bandwidth on the box (the e2e ceiling) + the C2 bench after R14b
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/pcie_probe.py > $O/e48_pcie.log 2>&1
timeout 600 python bench.py > $O/e48_bench_c2.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/e48_smoke.log 2>&1
