#!/bin/bash
OUT=gpurun_out/fine2
mkdir -p $OUT
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_gemm<32, 128" -c 3 -o $OUT/band_tile python tools/profile_call.py 2 > $OUT/ncu_band.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_slab12 -c 3 -o $OUT/slab12 python tools/profile_call.py 2 > $OUT/ncu_slab.log 2>&1
ls -la $OUT
