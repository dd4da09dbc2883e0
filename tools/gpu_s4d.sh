#!/bin/bash
# Session 4: L2 bulk prefetch of each band tile's / slab quarter's remaining B rows (PQ_L2PF) A/B
OUT=gpurun_out/s4d
mkdir -p $OUT
PQ_L2PF=1 timeout 600 python -m pytest tests/test_gpu_slab12.py tests/test_gpu_configs.py tests/test_gpu_band.py -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
for rep in 1 2; do
for pf in 0 1; do
  echo "config 2 PQ_L2PF=$pf" >> $OUT/ab.txt
  PQ_L2PF=$pf timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>>$OUT/err.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],2), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3))" >> $OUT/ab.txt
done; done
for c in 3 4; do for pf in 0 1; do
  echo "config $c PQ_L2PF=$pf" >> $OUT/ab.txt
  PQ_L2PF=$pf timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>>$OUT/err.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],2), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3))" >> $OUT/ab.txt
done; done
for pf in 0 1; do PQ_L2PF=$pf timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_pf$pf.txt 2>&1; done
ls -la $OUT
