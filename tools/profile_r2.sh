#!/bin/bash
# Round-2 evidence batch (GPU box): profile rounds of the kernel families not
# covered by round 1 (float C2, warp consensus C5-b16, general C2-ov25), the
# sharded loop at world size 1, and one bench line per config.
tag=${1:-r2a}
mkdir -p gpurun_out
for cfg in C2 C5-B16; do
  bash tools/profile_round.sh $cfg ${tag} > gpurun_out/${tag}_prof_${cfg}.log 2>&1
  echo "profile $cfg rc=$?"
done
# general path: launch list + K1g / global step full sets
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 400 --csv --log-file gpurun_out/${tag}_launches_C2-OV25.csv \
    python bench.py --config C2-ov25 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_block_mincut_g -s 8 -c 1 -f \
    -o gpurun_out/${tag}_k1_C2-OV25 python tools/prof_general.py C2-ov25 20 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:global -s 8 -c 1 -f \
    -o gpurun_out/${tag}_k2_C2-OV25 python tools/prof_general.py C2-ov25 20 > /dev/null 2>&1
echo "general profiled"
for cfg in C3 C4; do
  python bench.py --config $cfg --sharded --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_sharded_${cfg}.json 2>gpurun_out/${tag}_sharded_${cfg}.err
  echo "sharded $cfg rc=$?"
done
bash tools/bench_all.sh
cp gpurun_out/bench_all.jsonl gpurun_out/${tag}_bench_all.jsonl
echo done
