#!/bin/bash
# k_slab12 phase-2 skewed k loop A/B (PQ_SLAB12_SKEW)
OUT=gpurun_out/s3b
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0 1 0; do PQ_SLAB12_SKEW=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err; done
PQ_SLAB12_SKEW=1 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_skew.txt 2>&1
for v in 1 0; do PQ_SLAB12_SKEW=$v timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg4_$v.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
