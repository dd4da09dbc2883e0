#!/bin/bash
OUT=gpurun_out/s4l
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_bench_contract.py -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
timeout 400 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.jsonl 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
timeout 400 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg1.jsonl 2>> $OUT/bench.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg3.jsonl 2>> $OUT/bench.err
ls -la $OUT
