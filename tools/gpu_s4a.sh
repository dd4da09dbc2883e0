#!/bin/bash
# Session 4 start: confirm the restored build on a fresh box (GPU tests, smoke, driver bench command,
# launch list of the same command).
OUT=gpurun_out/s4a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 400 python bench.py --steps 20 --warmup 5 > $OUT/bench_cfg2.jsonl 2> $OUT/bench_cfg2.err; echo "rc=$?" >> $OUT/bench_cfg2.err
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>> $OUT/bench_cfg2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
ls -la $OUT
