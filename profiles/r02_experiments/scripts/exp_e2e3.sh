# box check: H2D bandwidth, then the C5 / C3 e2e legs, then H2D again
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/pcie_probe.py > $O/e54_pcie.log 2>&1
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline > $O/e54_bench_c5.log 2>&1
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > $O/e54_bench_c3.log 2>&1
python tools/pcie_probe.py >> $O/e54_pcie.log 2>&1
nproc >> $O/e54_pcie.log; numactl -H >> $O/e54_pcie.log 2>&1; nvidia-smi topo -m >> $O/e54_pcie.log 2>&1
