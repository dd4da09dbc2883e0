OUT=gpurun_out/g17; mkdir -p $OUT
for c in 1 2 4; do python tools/timeline_e2e.py $c 3 > $OUT/timeline_e2e_c$c.txt 2>&1; done
