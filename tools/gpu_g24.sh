OUT=gpurun_out/g24; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize_parity.py -x -q -m gpu -k "kron or etd or config4 or integrate" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg4.jsonl 2> $OUT/err.txt
