#!/bin/bash
# Session 4: fused squaring combination A/B at the HBM-heavier configs 3 and 5 (only config 2 was measured before),
# and the other configs' lines on the final build.
OUT=gpurun_out/s4b
mkdir -p $OUT
for c in 3 5; do
  for f in 0 1 0 1; do
    echo "config $c PQ_SQ_FUSE=$f" >> $OUT/sqfuse_ab.txt
    PQ_SQ_FUSE=$f timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/sqfuse_ab.txt 2>> $OUT/err.txt
  done
done
for c in 1 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 >> $OUT/bench_cfgs.jsonl 2>> $OUT/err.txt; done
PQ_SQ_FUSE=1 timeout 300 python tools/gemm_breakdown.py 3 > $OUT/breakdown_cfg3_fuse.txt 2>&1
timeout 300 python tools/gemm_breakdown.py 3 > $OUT/breakdown_cfg3.txt 2>&1
ls -la $OUT
