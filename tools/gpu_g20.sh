OUT=gpurun_out/g20; mkdir -p $OUT
N="--kernel-name-base demangled"
ncu --profile-from-start off --set full --clock-control none $N -k 'regex:k_gemm<\(int\)(32, \(int\)128|64, \(int\)32)' -c 6 -o $OUT/nodesweep python tools/profile_call.py 2 > $OUT/ncu_call.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv python tools/profile_call.py 2 > $OUT/ncu_launch.log 2>&1
python tools/gemm_breakdown.py 4 2 > $OUT/breakdown_cfg4.txt 2>&1
timeout 1200 python -m pytest tests/test_sharded.py -x -q -m gpu > $OUT/pytest_sharded.log 2>&1; echo "rc=$?" >> $OUT/pytest_sharded.log
ls -la $OUT
