#!/bin/bash
OUT=gpurun_out/c1
mkdir -p $OUT
for i in 1 2 3; do timeout 300 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg1.jsonl 2>>$OUT/bench.err; done
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err; done
timeout 300 python tools/trace_call.py 1 3 > $OUT/trace_cfg1.txt 2>&1
ls -la $OUT
