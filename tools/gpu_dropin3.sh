#!/bin/bash
OUT=gpurun_out/dropin3
mkdir -p $OUT
export LD_LIBRARY_PATH=$PWD/paper_2211_00696_b200:$LD_LIBRARY_PATH
for i in 1 2 3; do ./tools/dropin_bench 20 >> $OUT/new.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_refsuite.py tests/test_gpu_dropin.py tests/test_gpu_host_pinned.py tests/test_gpu_env_variants.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
