# KS1 per-CTA timeline (development build)
O=gpurun_out
HAP_EXTRA_NVCC_FLAGS="-DHAP_EXPERIMENTS" python paper_2605_08048_b200/build.py --force > /dev/null
python tools/ks1trace.py 5000 4096 > $O/e39_ks1trace.log 2>&1
python tools/ks1trace.py 1024 4096 >> $O/e39_ks1trace.log 2>&1
python tools/ks1trace.py 2100 2048 >> $O/e39_ks1trace.log 2>&1
python paper_2605_08048_b200/build.py --force > /dev/null
