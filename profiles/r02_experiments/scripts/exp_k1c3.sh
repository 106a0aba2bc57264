O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python tools/k1_probe.py > $O/k1c3_probe.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k1s python tools/k1_ncu.py 5000 4096 3 > $O/k1c3_launch.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1s -s 3 -c 3 -o $O/k1c3_full python tools/k1_ncu.py 5000 4096 3 > $O/k1c3_full.log 2>&1
