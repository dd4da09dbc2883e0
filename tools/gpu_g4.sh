set -x
mkdir -p gpurun_out/g4
for c in 2 3 5 1; do python tools/gemm_breakdown.py $c 3 > gpurun_out/g4/breakdown_cfg$c.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_bench_contract.py -x -q > gpurun_out/g4/contract.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g4/launches_cfg2.csv python tools/gemm_breakdown.py 2 1 > gpurun_out/g4/ncu_launch.log 2>&1
