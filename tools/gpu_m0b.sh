#!/bin/bash
OUT=gpurun_out/m0b
mkdir -p $OUT
PQ_MODE0=0 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_gemm<32, 128" -c 4 -o $OUT/band_tile python tools/profile_call.py 2 > $OUT/ncu_band.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_mode0 -c 3 -o $OUT/mode0es python tools/profile_call.py 2 > $OUT/ncu_m0.log 2>&1
ls -la $OUT
