#!/bin/bash
OUT=gpurun_out/c5gate
mkdir -p $OUT
for v in 1 0; do PQ_COMPUTE_GATE=$v timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg5_$v.jsonl 2>>$OUT/bench.err; done
for v in 1 0; do PQ_COMPUTE_GATE=$v timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg3_$v.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
