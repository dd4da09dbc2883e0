#!/bin/bash
# One gpurun session: GPU tests (selection in $TESTS), bench lines, acceptance-gate probe.
# Usage on the box: bash tools/gpu_round.sh <tag>
set -x
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/smi.txt 2>&1
if [ -n "$TESTS" ]; then
  PQ_MARGINS_OUT=$OUT/margins.jsonl timeout ${TEST_TIMEOUT:-1500} python -m pytest $TESTS -x -q -m gpu > $OUT/pytest.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest.log
fi
if [ -n "$ACCEPT" ]; then
  for i in $(seq 1 $ACCEPT); do
    PQ_SLOWLOG=10 timeout 300 tests/cpp/_bin/refsuite/acceptance > $OUT/accept_$i.out 2> $OUT/accept_$i.err
  done
  grep -h "criterion 7" $OUT/accept_*.out > $OUT/accept_c7.txt
fi
if [ -n "$BENCH" ]; then
  eval "$BENCH" > $OUT/bench.jsonl 2> $OUT/bench.err
fi
if [ -n "$EXTRA" ]; then
  eval "$EXTRA" > $OUT/extra.log 2>&1
fi
ls -la $OUT
