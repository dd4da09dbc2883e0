#!/bin/bash
OUT=gpurun_out/ic
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_slab12.py tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2.jsonl 2>>$OUT/bench.err
for c in 3 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/bench_cfgs.jsonl 2>>$OUT/bench.err; done
timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
ls -la $OUT
