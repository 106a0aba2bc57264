O=gpurun_out
for cn in 192 256 224 160; do
  HAP_EXTRA_NVCC_FLAGS="-DHAP_CHUNK_N=$cn" python paper_2605_08048_b200/build.py --force > /dev/null
  [ $cn = 192 ] && timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config1 or ragged or config2 or batch_varlen or wide or fuzz" > $O/e17_gt192.log 2>&1
  echo "chunk=$cn c2: $(python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e17_chunk.log
  echo "chunk=$cn c2 shared: $(HAP_SHARED=1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e17_chunk.log
  echo "chunk=$cn c5: $(HAP_SIZES=c5 python tools/batch.py 96 3 2>&1 | head -1)" >> $O/e17_chunk.log
  echo "chunk=$cn c3: $(python tools/config.py C3 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_test"])')" >> $O/e17_chunk.log
done
python paper_2605_08048_b200/build.py --force > /dev/null
