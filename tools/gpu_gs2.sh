#!/bin/bash
OUT=gpurun_out/gs2
mkdir -p $OUT
PQ_GEMM_SMALL=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_small1.csv python tools/profile_call.py 2 > $OUT/ncu1.log 2>&1
PQ_GEMM_SMALL=0 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_small0.csv python tools/profile_call.py 2 > $OUT/ncu0.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_gemm_small -c 3 -o $OUT/small python tools/profile_call.py 2 > $OUT/ncu_full.log 2>&1
ls -la $OUT
