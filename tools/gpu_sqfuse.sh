mkdir -p gpurun_out/sqf
PQ_SQ_FUSE=0 timeout 300 python tools/bitwise_env_ab.py /tmp/f0.npz > gpurun_out/sqf/ab.txt 2>&1
PQ_SQ_FUSE=1 timeout 300 python tools/bitwise_env_ab.py /tmp/f1.npz >> gpurun_out/sqf/ab.txt 2>&1
python tools/bitwise_env_ab.py --compare /tmp/f0.npz /tmp/f1.npz >> gpurun_out/sqf/ab.txt 2>&1
for f in 1 0 1 0; do
  PQ_SQ_FUSE=$f timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/sqf/b_$f.$RANDOM.json 2>/dev/null
done
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_config_shapes.py tests/test_gpu_host_pinned.py > gpurun_out/sqf/tests.txt 2>&1
PQ_SQ_FUSE=1 timeout 300 python tools/gemm_breakdown.py 2 > gpurun_out/sqf/breakdown_cfg2.txt 2>&1
