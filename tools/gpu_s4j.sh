#!/bin/bash
# Session 4: full GPU suite with the new slab12 tests; short reference-arm run (complete calls) on the same box
OUT=gpurun_out/s4j
mkdir -p $OUT
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg2.jsonl 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.jsonl 2>> $OUT/bench.err; echo "ref rc=$?" >> $OUT/bench.err
grep -l libpq_b200 /proc/self/maps > /dev/null 2>&1
ls -la $OUT
