OUT=gpurun_out/g14; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_host_pinned.py tests/test_gpu_refsuite.py tests/test_gpu_dropin.py tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in 2 3; do python bench.py --steps 12 --warmup 3 --no-cpu-baseline --e2e-callers $c > $OUT/bench_c$c.jsonl 2>> $OUT/err.txt; done
