OUT=gpurun_out/g21; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_fullsize_parity.py tests/test_gpu_config_shapes.py tests/test_gpu_parity.py tests/test_gpu_refsuite.py -x -q -m gpu -k "etd or config4 or integrate or erk or acceptance or unit_suite or expm" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg4.jsonl 2> $OUT/err.txt
python tools/gemm_breakdown.py 4 2 > $OUT/breakdown_cfg4.txt 2>&1
