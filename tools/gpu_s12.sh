#!/bin/bash
# fused mode-1+2 kernel: bitwise test, A/B bench at config 2 (and 4), GEMM breakdown, launch list
OUT=gpurun_out/s12
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0 1 0; do
  PQ_SLAB12=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err
done
PQ_SLAB12=1 timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg4_1.jsonl 2>>$OUT/bench.err
PQ_SLAB12=0 timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg4_0.jsonl 2>>$OUT/bench.err
PQ_SLAB12=1 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_1.txt 2>&1
PQ_SLAB12=0 timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_0.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python tools/profile_call.py 2 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_slab12 -c 2 -o $OUT/slab12 \
  python tools/profile_call.py 2 > $OUT/ncu_full.log 2>&1
ls -la $OUT
