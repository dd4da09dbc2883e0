OUT=gpurun_out/s3e; mkdir -p $OUT
timeout 300 python tools/timeline.py 2 3 --dump=$OUT/timeline_cfg2.csv > $OUT/timeline_cfg2.txt 2>&1
timeout 300 python tools/trace_call.py 2 5 > $OUT/trace_cfg2.txt 2>&1
