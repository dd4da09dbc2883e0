OUT=gpurun_out/g16; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_expm_paths.py tests/test_gpu_configs.py tests/test_gpu_dense_oracle.py tests/test_gpu_guards.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
PQ_GEMM_CHAIN=0 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2_nochain.txt 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench.jsonl 2> $OUT/err.txt
PQ_GEMM_CHAIN=0 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_nochain.jsonl 2>> $OUT/err.txt
