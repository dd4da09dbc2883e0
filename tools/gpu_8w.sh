#!/bin/bash
OUT=gpurun_out/w8
mkdir -p $OUT
PQ_BAND_8W=1 timeout 900 python -m pytest tests/test_gpu_slab12.py tests/test_gpu_band.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0; do PQ_BAND_8W=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err; done
PQ_BAND_8W=1 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_1.txt 2>&1
for v in 1 0; do PQ_BAND_8W=$v timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg3_$v.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
