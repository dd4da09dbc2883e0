#!/bin/bash
# round-2 third session final build (skewed k_slab12 phase 2): GPU tests, smoke, default bench, configs 1/3/4/5, launch list, ncu --set full of k_slab12 and the band tile
# ncu launch list of one config-2 call, ncu --set full of the fused slab kernel and the band tile
OUT=gpurun_out/s3f
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/tests.txt 2>&1; echo "tests rc=$?" >> $OUT/tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 400 python bench.py > $OUT/bench_default.jsonl 2> $OUT/bench_default.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline >> $OUT/bench_cfg2_driver.jsonl 2>> $OUT/bench_default.err
for c in 1 3 4 5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 >> $OUT/bench_cfgs.jsonl 2>>$OUT/bench_cfgs.err; done
timeout 300 python tools/gemm_breakdown.py 2 3 > $OUT/breakdown_cfg2.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_cfg2.csv python tools/profile_call.py 2 > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_slab12 -c 3 -o $OUT/slab12 python tools/profile_call.py 2 > $OUT/ncu_slab.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm --launch-skip 5 -c 3 -o $OUT/band_tile python tools/profile_call.py 2 > $OUT/ncu_band.log 2>&1
ls -la $OUT
