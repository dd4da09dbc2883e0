#!/bin/bash
OUT=gpurun_out/gate2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_host_pinned.py tests/test_gpu_env_variants.py tests/test_gpu_dropin.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg5.jsonl 2>>$OUT/bench.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg3.jsonl 2>>$OUT/bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err
ls -la $OUT
