#!/bin/bash
OUT=gpurun_out/margins
mkdir -p $OUT
PQ_MARGINS_OUT=$OUT/margins.jsonl timeout 2400 python -m pytest tests/test_gpu_config_shapes.py tests/test_gpu_fullsize_parity.py tests/test_gpu_dense_oracle.py -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
ls -la $OUT
