OUT=gpurun_out/g22; mkdir -p $OUT
python tools/timeline.py 4 1 > $OUT/timeline_cfg4.txt 2>&1
PQ_ETD_GRAPH=0 python tools/timeline.py 4 1 > $OUT/timeline_cfg4_nograph.txt 2>&1
