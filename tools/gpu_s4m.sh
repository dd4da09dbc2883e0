#!/bin/bash
# Round-end rehearsal: exactly the driver's sequence on a fresh box (reference arm first, then ours), timed
OUT=gpurun_out/s4m
mkdir -p $OUT
t0=$(date +%s)
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$? $(( $(date +%s) - t0 )) s" >> $OUT/tests.txt
t0=$(date +%s)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$? $(( $(date +%s) - t0 )) s" >> $OUT/smoke.txt
t0=$(date +%s)
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err; echo "ref rc=$? $(( $(date +%s) - t0 )) s" >> $OUT/bench_reference.err
t0=$(date +%s)
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench_ours.jsonl 2> $OUT/bench_ours.err; echo "ours rc=$? $(( $(date +%s) - t0 )) s" >> $OUT/bench_ours.err
ls -la $OUT
