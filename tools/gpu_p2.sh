#!/bin/bash
OUT=gpurun_out/p2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py tests/test_gpu_configs.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err; done
for i in 1 2 3; do timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg4.jsonl 2>>$OUT/bench.err; done
timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
ls -la $OUT
