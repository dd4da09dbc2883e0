#!/bin/bash
OUT=gpurun_out/m5
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 5 4 5 4; do
  PQ_SLAB12_MINB=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err
done
PQ_SLAB12_MINB=5 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_5.txt 2>&1
PQ_SLAB12_MINB=5 timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_slab12 -c 2 -o $OUT/slab12_m5 python tools/profile_call.py 2 > $OUT/ncu_full.log 2>&1
ls -la $OUT
