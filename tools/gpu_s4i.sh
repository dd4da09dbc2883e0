#!/bin/bash
# Session 4 final build (inline pack): full GPU suite, smoke, driver bench command with CPU baseline, default bench
OUT=gpurun_out/s4i
mkdir -p $OUT
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 400 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.jsonl 2> $OUT/bench_cfg2.err; echo "rc=$?" >> $OUT/bench_cfg2.err
timeout 400 python bench.py >> $OUT/bench_cfg2.jsonl 2>> $OUT/bench_cfg2.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 >> $OUT/bench_cfg4.jsonl 2>> $OUT/bench_cfg2.err
ls -la $OUT
