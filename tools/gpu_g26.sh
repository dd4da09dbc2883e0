OUT=gpurun_out/g26; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_sharded.py tests/test_gpu_bench_contract.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
