#!/bin/bash
# Session 4: pack copy written inside k_band_ranges' reduction loop (no separate pass)
OUT=gpurun_out/s4h
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py tests/test_gpu_configs.py tests/test_gpu_band.py tests/test_gpu_env_variants.py -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>$OUT/err.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],2), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3))" >> $OUT/ab.txt
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_call.csv --profile-from-start off python tools/profile_call.py 2 > $OUT/ncu.log 2>&1
ls -la $OUT
