#!/bin/bash
# Profile evidence for profiles/ (run on the GPU box):
#   1. the bench line (no profiler), 2. the launch list of the same command
#   under ncu (per-launch duration + DRAM bytes), 3. one --set full capture of
#   K1 and of K2 at a steady-state iteration (tools/prof_run.py, no graph).
cfg=${1:-C3}
tag=${2:-r1}
set -e
python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/${tag}_bench_${cfg}.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/${tag}_launches_${cfg}.csv \
    python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_block_mincut -s 8 -c 1 -f \
    -o gpurun_out/${tag}_k1_${cfg} python tools/prof_run.py $cfg 20 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_consensus -s 8 -c 1 -f \
    -o gpurun_out/${tag}_k2_${cfg} python tools/prof_run.py $cfg 20 > /dev/null 2>&1
tail -c 600 gpurun_out/${tag}_bench_${cfg}.json
