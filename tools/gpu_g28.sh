OUT=gpurun_out/g28; mkdir -p $OUT
for i in 1 2 3; do tools/fp64_peak; done > $OUT/fp64_peak.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv >> $OUT/fp64_peak.txt
