OUT=gpurun_out/g8; mkdir -p $OUT
for z in 2 4 13; do for bw in 4 6; do echo "=== n=128 Z=$z bw=$bw"; timeout 300 tools/gemm_tune 128 $z 81 $bw 1 2>&1 | grep -v "^  64x\|WS\|expm-sq\|mode2" ; done; done > $OUT/tune_tma.txt 2>&1
timeout 300 tools/gemm_tune 256 4 81 8 1 > $OUT/tune_tma_n256.txt 2>&1
