#!/bin/bash
OUT=gpurun_out/st3
mkdir -p $OUT
PQ_SLAB12_STAGES=3 timeout 900 python -m pytest tests/test_gpu_slab12.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 3 2 3 2; do PQ_SLAB12_STAGES=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err; done
PQ_SLAB12_STAGES=3 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_3.txt 2>&1
for v in 3 2; do PQ_SLAB12_STAGES=$v timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg4_$v.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
