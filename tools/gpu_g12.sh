OUT=gpurun_out/g12; mkdir -p $OUT
python tools/timeline.py 2 3 > $OUT/timeline_dev.txt 2>&1
python tools/timeline.py 2 3 --host > $OUT/timeline_host.txt 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench.jsonl 2> $OUT/bench.err
PQ_SMALL_GRID_TILE=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_noshape8.jsonl 2>> $OUT/bench.err
python bench.py --steps 12 --warmup 3 --no-cpu-baseline --e2e-callers 6 > $OUT/bench_c6.jsonl 2>> $OUT/bench.err
python bench.py --steps 12 --warmup 3 --no-cpu-baseline --e2e-callers 8 > $OUT/bench_c8.jsonl 2>> $OUT/bench.err
python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
