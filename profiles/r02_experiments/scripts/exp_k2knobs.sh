O=gpurun_out
python -c "import __graft_entry__ as g; g.build()"
run() { echo "$1: $(env $1 python tools/batch.py 48 5 2>&1 | head -1)" >> $O/e8_matrix.log; }
run "HAP_X=0"
run "HAP_K2_NARROW=1"
run "HAP_K2_NARROW=1 HAP_K2_PW=2"
run "HAP_K2_WIDE_PW=2"
run "HAP_WAVE=2"
run "HAP_WAVE=4"
run "HAP_LANES=3"
run "HAP_LANES=3 HAP_WAVE=2"
run "HAP_K3_TILE_GROUP=0"
run "HAP_X=1"
