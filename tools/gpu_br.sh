#!/bin/bash
OUT=gpurun_out/br
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_slab12.py tests/test_gpu_configs.py tests/test_gpu_env_variants.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err; done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv python tools/profile_call.py 2 > $OUT/ncu_launch.log 2>&1
ls -la $OUT
