#!/bin/bash
OUT=gpurun_out/mb5
mkdir -p $OUT
for v in 1 0 1 0; do PQ_MINB5=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err; done
for v in 1 0; do PQ_MINB5=$v timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg4_$v.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
