set -x
mkdir -p gpurun_out/gate
for g in 1 0 1 0; do
  PQ_COMPUTE_GATE=$g timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/gate/b_$g.$RANDOM.json 2>gpurun_out/gate/err_$g.log
done
grep -h . gpurun_out/gate/b_*.json | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['value'], d['e2e']['value'], d['e2e']['single_caller_value'])"
