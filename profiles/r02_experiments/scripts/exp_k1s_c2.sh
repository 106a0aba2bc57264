set -x
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python tools/batch.py 24 5 > $O/e1_batch_default.log 2>&1
HAP_SHARED=1 python tools/batch.py 24 5 > $O/e1_batch_shared.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_perm_fy32 -s 3 -c 1 -o $O/e1_k2 python tools/batch.py 6 1 > $O/e1_k2ncu.log 2>&1
HAP_EXTRA_NVCC_FLAGS="-DHAP_K1S_MIN_ELEMS=0" python paper_2605_08048_b200/build.py --force
python tools/batch.py 24 5 > $O/e1_batch_k1s.log 2>&1
HAP_SHARED=1 python tools/batch.py 24 5 > $O/e1_batch_k1s_shared.log 2>&1
