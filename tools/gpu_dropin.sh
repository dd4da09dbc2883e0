#!/bin/bash
OUT=gpurun_out/dropin
mkdir -p $OUT
export LD_LIBRARY_PATH=$PWD/paper_2211_00696_b200:$LD_LIBRARY_PATH
for i in 1 2; do ./tools/dropin_bench_old 20 >> $OUT/old.txt 2>&1; ./tools/dropin_bench 20 >> $OUT/new.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_refsuite.py tests/test_gpu_dropin.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
ls -la $OUT
