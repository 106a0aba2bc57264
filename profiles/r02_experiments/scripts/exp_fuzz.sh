# fuzz campaign: 120 seeded wide shapes against the oracle (full parity bars)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
FUZZ_CASES=120 timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -k fuzz_campaign -v -s -p no:cacheprovider > gpurun_out/r02_fuzz_campaign.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/e47_gt.log 2>&1
