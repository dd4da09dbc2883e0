#!/bin/bash
OUT=gpurun_out/c4
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_slab12.py tests/test_gpu_configs.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0 1 0; do PQ_FINE=$v timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfg4_$v.jsonl 2>>$OUT/bench.err; done
for v in 1 0; do PQ_FINE=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv python tools/profile_call.py 2 > $OUT/ncu_launch.log 2>&1
ls -la $OUT
