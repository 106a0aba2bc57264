# KS2 source-level profile at C3 + KS1/KS3 per-CTA stamps (development build)
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1s_coef -s 1 -c 1 -o $O/e41_ks2 python tools/k1_ncu.py 5000 4096 2 > $O/e41_ks2.log 2>&1
HAP_EXTRA_NVCC_FLAGS="-DHAP_EXPERIMENTS" python paper_2605_08048_b200/build.py --force > /dev/null
python tools/ks1trace.py 5000 4096 > $O/e41_ks1trace.log 2>&1
python paper_2605_08048_b200/build.py --force > /dev/null
