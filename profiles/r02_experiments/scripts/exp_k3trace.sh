O=gpurun_out
HAP_EXTRA_NVCC_FLAGS="-DHAP_EXPERIMENTS" python paper_2605_08048_b200/build.py --force > /dev/null
HAP_TRACE_B=30000 python tools/k3trace.py > $O/e33_k3trace.log 2>&1
python paper_2605_08048_b200/build.py --force > /dev/null
