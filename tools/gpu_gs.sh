#!/bin/bash
OUT=gpurun_out/gs
mkdir -p $OUT
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0 1 0; do
  PQ_GEMM_SMALL=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err
done
PQ_GEMM_SMALL=1 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_1.txt 2>&1
timeout 300 python tools/trace_call.py 2 3 > $OUT/trace_cfg2.txt 2>&1
for c in 1 4; do timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfgs.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
