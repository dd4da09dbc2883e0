#!/bin/bash
OUT=gpurun_out/s12b
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/timeline.py 2 3 --dump=$OUT/timeline_cfg2.csv > $OUT/timeline_cfg2.txt 2>&1
PQ_SLAB12=0 timeout 300 python tools/timeline.py 2 3 --dump=$OUT/timeline_cfg2_sep.csv > $OUT/timeline_cfg2_sep.txt 2>&1
ls -la $OUT
