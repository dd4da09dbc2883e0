set -x
OUT=gpurun_out/g5; mkdir -p $OUT
# ncu --set full: the dominant band tile (node sweep mode 0 + squaring mode 0) and the 32x32 small GEMMs of one config-2 call
ncu --set full --clock-control none --import-source on -k regex:"k_gemm<32, 128" -s 24 -c 3 -o $OUT/band_tile python tools/gemm_breakdown.py 2 1 > $OUT/ncu_band.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm<32, 32" -s 20 -c 6 -o $OUT/small_tile python tools/gemm_breakdown.py 2 1 > $OUT/ncu_small.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm<64, 32" -s 12 -c 2 -o $OUT/kk_tile python tools/gemm_breakdown.py 2 1 > $OUT/ncu_kk.log 2>&1
# compute-sanitizer on the small parity tests: two-stream squaring, CC ring combine, PDL GEMM chain
SEL="tests/test_gpu_parity.py tests/test_gpu_configs.py"
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --target-processes all python -m pytest $SEL -x -q -m gpu -k "not fullsize" > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --target-processes all python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mode_apply or squaring or phi_fixed or adaptive" > $OUT/racecheck.log 2>&1; echo "racecheck rc=$?" >> $OUT/racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --target-processes all python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "mode_apply or squaring" > $OUT/synccheck.log 2>&1; echo "synccheck rc=$?" >> $OUT/synccheck.log
