mkdir -p gpurun_out/callers
for k in 2 3 4 6 8; do
  timeout 400 python bench.py --steps 24 --warmup 3 --e2e-callers $k > gpurun_out/callers/b_$k.json 2>/dev/null
done
