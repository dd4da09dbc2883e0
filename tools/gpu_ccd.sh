#!/bin/bash
OUT=gpurun_out/ccd
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_cc_defer.py tests/test_gpu_env_variants.py tests/test_gpu_slab12.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for v in 1 0 1 0; do
  PQ_CC_DEFER=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_$v.jsonl 2>>$OUT/bench.err
done
timeout 300 python tools/timeline.py 2 3 --dump=$OUT/timeline_cfg2.csv > $OUT/timeline_cfg2.txt 2>&1
ls -la $OUT
