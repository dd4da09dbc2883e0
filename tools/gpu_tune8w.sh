mkdir -p gpurun_out/tune8
timeout 300 tools/gemm_tune 128 4 81 4 1 > gpurun_out/tune8/sq_z4.txt 2>&1
timeout 300 tools/gemm_tune 128 2 81 4 1 > gpurun_out/tune8/sq_z2.txt 2>&1
timeout 300 tools/gemm_tune 128 13 81 2 1 > gpurun_out/tune8/node_z13.txt 2>&1
