#!/bin/bash
OUT=gpurun_out/pfs
mkdir -p $OUT
timeout 1500 python tools/parity_fullsize.py > $OUT/parity_fullsize.jsonl 2> $OUT/parity_fullsize.err
ls -la $OUT
