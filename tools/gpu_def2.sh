mkdir -p gpurun_out/def6
for i in 1 2 3; do timeout 400 python bench.py > gpurun_out/def6/b_$i.json 2>/dev/null; done
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/def6/c3.json 2>/dev/null
