#!/bin/bash
OUT=gpurun_out/fk
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_cc_defer.py tests/test_gpu_env_variants.py tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_host_pinned.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err; done
timeout 300 python tools/timeline.py 2 3 --dump=$OUT/timeline_cfg2.csv > $OUT/timeline_cfg2.txt 2>&1
timeout 300 python tools/trace_call.py 2 3 > $OUT/trace_cfg2.txt 2>&1
ls -la $OUT
