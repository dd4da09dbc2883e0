#!/bin/bash
OUT=gpurun_out/fine5
mkdir -p $OUT
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 0 1 0 1; do
  PQ_BAND_DEEP=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_deep$v.jsonl 2>>$OUT/bench.err
done
PQ_BAND_DEEP=1 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_deep1.txt 2>&1
PQ_BAND_DEEP=0 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_deep0.txt 2>&1
for v in 0 1; do PQ_BAND_DEEP=$v timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg3_deep$v.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
