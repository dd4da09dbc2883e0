OUT=gpurun_out/g10; mkdir -p $OUT
for b in gemm_tune gemm_tune_old; do for z in 2 4 13; do echo "=== $b n=128 Z=$z bw=5"; timeout 300 tools/$b 128 $z 81 5 1 2>&1 | grep -E "mode|32x128x16 w32x32|64x 32x16" | grep -v "TMA\|WS\|mode2+sq"; done; done > $OUT/tune_affine.txt 2>&1
for b in gemm_tune gemm_tune_old; do echo "=== $b n=256 Z=4 bw=8"; timeout 300 tools/$b 256 4 81 8 1 2>&1 | grep -E "mode|32x128x16 w32x32|64x 32x16" | grep -v "TMA\|WS\|mode2+sq"; done >> $OUT/tune_affine.txt 2>&1
