OUT=gpurun_out/g27; mkdir -p $OUT
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg2.jsonl 2> $OUT/err.txt
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg3.jsonl 2>> $OUT/err.txt
python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-callers 1 > $OUT/bench_cfg5.jsonl 2>> $OUT/err.txt
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg1.jsonl 2>> $OUT/err.txt
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg4.jsonl 2>> $OUT/err.txt
