OUT=gpurun_out/g23; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize_parity.py tests/test_gpu_config_shapes.py tests/test_gpu_refsuite.py tests/test_gpu_dropin.py tests/test_gpu_guards.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg4.jsonl 2> $OUT/err.txt
PQ_KMV_STENCIL=0 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg4_nostencil.jsonl 2>> $OUT/err.txt
