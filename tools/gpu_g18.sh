OUT=gpurun_out/g18; mkdir -p $OUT
timeout 1800 python -m pytest tests/ -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
