OUT=gpurun_out/g11; mkdir -p $OUT
timeout 1800 python -m pytest tests/ -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --steps 10 --warmup 3 > $OUT/bench.jsonl 2> $OUT/bench.err
python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
