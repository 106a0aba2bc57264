# C3 K3 DRAM traffic per launch at HEAD (ncu metrics, 3 launches)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:k3_maskgemm -s 2 -c 3 python tools/config.py C3 > $O/e51_c3_k3.csv 2>&1
