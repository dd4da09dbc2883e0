OUT=gpurun_out/g25; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_sharded.py -x -q -m gpu -k "peer" > $OUT/pytest_peer.log 2>&1; echo "rc=$?" >> $OUT/pytest_peer.log
timeout 1500 python -m pytest tests/test_sharded.py tests/test_gpu_parity.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
