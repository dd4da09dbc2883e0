mkdir -p gpurun_out/gate
timeout 600 python -m pytest -x -q tests/test_gpu_host_pinned.py tests/test_gpu_parity.py tests/test_gpu_refsuite.py > gpurun_out/gate/tests.txt 2>&1
for g in 1 0; do
  PQ_COMPUTE_GATE=$g timeout 300 python tools/timeline_e2e.py 4 3 --streams > gpurun_out/gate/tl_$g.txt 2>&1
done
for g in 1 0 1 0; do
  PQ_COMPUTE_GATE=$g timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/gate/b_$g.$RANDOM.json 2>gpurun_out/gate/err_$g.log
done
