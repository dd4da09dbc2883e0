#!/bin/bash
OUT=gpurun_out/grp
mkdir -p $OUT
PQ_SQ_DEV_GROUPS=4 timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_configs.py -x -q -m gpu -k "not refsuite" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for cfgv in "2 3" "4 3" "2 4" "4 4" "3 3" "2 3"; do set -- $cfgv; PQ_SQ_DEV_GROUPS=$1 PQ_SQ_DEV_RING=$2 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-callers 1 >> $OUT/bench_g$1_r$2.jsonl 2>>$OUT/bench.err; done
ls -la $OUT
