OUT=gpurun_out/g15; mkdir -p $OUT
for z in 2 4 13; do echo "=== n=128 Z=$z bw=5"; timeout 300 tools/gemm_tune 128 $z 81 5 1 2>&1 | grep -E "^mode[01] |32x.*w32x32 st2" | grep -v "TMA\|WS"; done > $OUT/tune_bn.txt 2>&1
