#!/bin/bash
# One bench line per BASELINE config (run on the GPU box); output gpurun_out/bench_all.jsonl
out=gpurun_out/bench_all.jsonl
: > $out
for cfg in C1 C2 C3 C4 C5-b16 C5-b32 C5-b64 C5-b128 C2-ov25; do
  extra=""
  case $cfg in C1|C2|C2-ov25) extra="--steps 10 --warmup 3";; C4) extra="--steps 3 --warmup 3";; *) extra="--steps 5 --warmup 3";; esac
  timeout 900 python bench.py --config $cfg $extra --cpu-sample-iters 2 > gpurun_out/bench_$cfg.log 2>&1
  tail -1 gpurun_out/bench_$cfg.log >> $out
done
