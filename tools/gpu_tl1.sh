mkdir -p gpurun_out/tl
for g in 2 3 4; do
PQ_SQ_GROUPS=$g timeout 300 python tools/timeline_e2e.py 1 6 --streams > gpurun_out/tl/g${g}_1.txt 2>&1
PQ_SQ_GROUPS=$g timeout 300 python tools/timeline_e2e.py 4 4 > gpurun_out/tl/g${g}_4.txt 2>&1
done
