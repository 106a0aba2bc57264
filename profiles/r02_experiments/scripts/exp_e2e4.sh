# C3 end-to-end leg outside bench.py (HEAD library), twice, plus the H2D bandwidth probe
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/e2e_probe.py > $O/e55_e2e.log 2>&1
python tools/e2e_probe.py >> $O/e55_e2e.log 2>&1
python tools/pcie_probe.py >> $O/e55_e2e.log 2>&1
