#!/bin/bash
OUT=gpurun_out/dropin2
mkdir -p $OUT
export LD_LIBRARY_PATH=$PWD/paper_2211_00696_b200:$LD_LIBRARY_PATH
PQ_SLOWLOG=0.5 ./tools/dropin_bench 6 > $OUT/new_slowlog.txt 2>&1
ls -la $OUT
