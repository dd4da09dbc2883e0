OUT=gpurun_out/g9; mkdir -p $OUT
PQ_MARGINS_OUT=$OUT/margins.jsonl timeout 1500 python -m pytest tests/test_gpu_config_shapes.py tests/test_sharded.py tests/test_gpu_guards.py tests/test_gpu_refsuite.py tests/test_gpu_dropin.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg3.jsonl 2> $OUT/bench_cfg3.err
python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-callers 1 > $OUT/bench_cfg5.jsonl 2> $OUT/bench_cfg5.err
python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg1.jsonl 2> $OUT/bench_cfg1.err
