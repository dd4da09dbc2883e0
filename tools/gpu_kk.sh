#!/bin/bash
OUT=gpurun_out/kk
mkdir -p $OUT
PQ_KK_TALL=1 timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_configs.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0; do PQ_KK_TALL=$v timeout 300 python tools/gemm_breakdown.py 3 1 > $OUT/breakdown_cfg3_$v.txt 2>&1; done
for v in 1 0; do PQ_KK_TALL=$v timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg3_$v.jsonl 2>>$OUT/bench.err; done
for v in 1 0; do PQ_KK_TALL=$v timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg5_$v.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
