#!/bin/bash
# Session 4 final build: full GPU suite, smoke, driver bench command (with CPU baseline), configs 1/3/4/5, launch list
OUT=gpurun_out/s4g
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 400 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.jsonl 2> $OUT/bench_cfg2.err; echo "rc=$?" >> $OUT/bench_cfg2.err
timeout 400 python bench.py >> $OUT/bench_cfg2.jsonl 2>> $OUT/bench_cfg2.err
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 >> $OUT/bench_cfgs.jsonl 2>>$OUT/bench_cfgs.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
ls -la $OUT
