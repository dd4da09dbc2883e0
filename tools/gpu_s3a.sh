#!/bin/bash
# session-3 start: confirm the rebuilt tree on a fresh box (GPU tests, smoke, default bench, config-2 driver command)
OUT=gpurun_out/s3a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 400 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
ls -la $OUT
