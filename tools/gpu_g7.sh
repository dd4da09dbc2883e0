set -x
OUT=gpurun_out/g7; mkdir -p $OUT
N="--kernel-name-base demangled"
timeout 900 python -m pytest tests/test_gpu_guards.py -x -q > $OUT/guards.log 2>&1
ncu --set full --clock-control none --import-source on $N -k 'regex:k_gemm<\(int\)32, \(int\)128' -s 24 -c 3 -o $OUT/band_tile python tools/gemm_breakdown.py 2 1 > $OUT/ncu_band.log 2>&1
ncu --set full --clock-control none --import-source on $N -k 'regex:k_gemm<\(int\)32, \(int\)32' -s 20 -c 6 -o $OUT/small_tile python tools/gemm_breakdown.py 2 1 > $OUT/ncu_small.log 2>&1
ncu --set full --clock-control none --import-source on $N -k 'regex:k_gemm<\(int\)64, \(int\)32' -s 12 -c 2 -o $OUT/kk_tile python tools/gemm_breakdown.py 2 1 > $OUT/ncu_kk.log 2>&1
ls -la $OUT
