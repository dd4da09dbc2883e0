OUT=gpurun_out/final; mkdir -p $OUT
( time python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > $OUT/bench.jsonl 2> $OUT/bench.err
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $OUT/bench_ref.jsonl 2> $OUT/bench_ref.err
