#!/bin/bash
# Session 4: fragment-major E2 copies for k_slab12 phase 2 (PQ_E2PACK) x skewed / aligned phase-2 loop A/B
OUT=gpurun_out/s4c
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slab12.py tests/test_gpu_configs.py tests/test_gpu_band.py tests/test_gpu_env_variants.py tests/test_gpu_golden.py -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
for rep in 1 2; do
for pk in 0 1; do for sk in 1 0; do
  echo "PQ_E2PACK=$pk PQ_SLAB12_SKEW=$sk" >> $OUT/ab.txt
  PQ_E2PACK=$pk PQ_SLAB12_SKEW=$sk timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>$OUT/err.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],3))" >> $OUT/ab.txt
done; done; done
for pk in 0 1; do for sk in 1 0; do
  PQ_E2PACK=$pk PQ_SLAB12_SKEW=$sk timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_pk${pk}_sk${sk}.txt 2>&1
done; done
PQ_E2PACK=1 PQ_SLAB12_SKEW=0 timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/cfg4_pk1_sk0.jsonl 2>>$OUT/err.txt
PQ_E2PACK=1 PQ_SLAB12_SKEW=1 timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/cfg4_pk1_sk1.jsonl 2>>$OUT/err.txt
PQ_E2PACK=0 PQ_SLAB12_SKEW=1 timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/cfg4_pk0_sk1.jsonl 2>>$OUT/err.txt
for pk in 0 1; do
PQ_E2PACK=$pk PQ_SLAB12_SKEW=1 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_slab12 --launch-skip 6 -c 2 -o $OUT/slab12_pk$pk python tools/profile_call.py 2 > $OUT/ncu_slab_pk$pk.log 2>&1
done
PQ_E2PACK=1 PQ_SLAB12_SKEW=0 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_slab12 --launch-skip 6 -c 2 -o $OUT/slab12_pk1_sk0 python tools/profile_call.py 2 > $OUT/ncu_slab_pk1_sk0.log 2>&1
ls -la $OUT
