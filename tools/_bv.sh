B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
P='import json,sys;d=json.load(open(sys.argv[1]));k=d["config"]["kernels"];print(sys.argv[2],round(d["value"]),k["K1_block_mincut"]["median_ms"],k["K2_consensus"]["median_ms"])'
run() { name=$1; shift; env "$@" timeout 300 $B > gpurun_out/v_$name.json 2>gpurun_out/v_$name.err; python -c "$P" gpurun_out/v_$name.json $name; }
