#!/bin/bash
# Session 4: ncu --set full + source of the mode-0 band tile in the squaring (grid 4 x 128 x 2) and the node sweep
OUT=gpurun_out/s4f
mkdir -p $OUT
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_gemm<.int.32, .int.128' --launch-skip 5 -c 2 -o $OUT/band_sq python tools/profile_call.py 2 > $OUT/ncu_band_sq.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_gemm<.int.32, .int.128' -c 1 -o $OUT/band_node python tools/profile_call.py 2 > $OUT/ncu_band_node.log 2>&1
ls -la $OUT
