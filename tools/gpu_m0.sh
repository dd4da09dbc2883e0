#!/bin/bash
OUT=gpurun_out/m0
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0; do PQ_MODE0=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err; done
timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
ls -la $OUT
