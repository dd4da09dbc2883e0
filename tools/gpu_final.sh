mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/final/tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/final/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.txt
timeout 400 python bench.py > gpurun_out/final/bench_default.jsonl 2>gpurun_out/final/bench_default.err
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 >> gpurun_out/final/bench_cfgs.jsonl 2>>gpurun_out/final/bench_cfgs.err; done
