#!/bin/bash
OUT=gpurun_out/tr
mkdir -p $OUT
timeout 300 python tools/trace_call.py 2 4 > $OUT/trace_cfg2.txt 2>&1
PQ_SIDE_PRIO=1 timeout 300 python tools/trace_call.py 2 4 > $OUT/trace_cfg2_sideprio.txt 2>&1
for v in 1 0 1 0; do
  PQ_SIDE_PRIO=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_side$v.jsonl 2>>$OUT/bench.err
done
PQ_SIDE_PRIO=1 timeout 300 python tools/timeline.py 2 3 --dump=$OUT/timeline_cfg2_sideprio.csv > $OUT/timeline_cfg2_sideprio.txt 2>&1
ls -la $OUT
