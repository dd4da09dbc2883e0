OUT=gpurun_out/g13; mkdir -p $OUT
nproc > $OUT/nproc.txt; cat /sys/fs/cgroup/cpu.max >> $OUT/nproc.txt 2>&1
python tools/plan_time.py > $OUT/plan_par.txt 2>&1 || true
for t in 1 6; do PQ_PLAN_THREADS=$t python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg1_t$t.jsonl 2>> $OUT/err.txt; done
for t in 1 6; do PQ_PLAN_THREADS=$t python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-callers 4 > $OUT/bench_cfg2_t$t.jsonl 2>> $OUT/err.txt; done
