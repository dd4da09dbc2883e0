#!/bin/bash
# Session 4: ncu --set full of the HBM-bound kernels of a config-2 call (k_sq_combine2, k_node_combine_ring)
OUT=gpurun_out/s4n
mkdir -p $OUT
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:'k_sq_combine2|k_node_combine_ring' -c 4 -o $OUT/hbm_kernels python tools/profile_call.py 2 > $OUT/ncu.log 2>&1
ls -la $OUT
