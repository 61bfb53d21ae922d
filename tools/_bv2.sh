# per-config quick bench lines: value and the two kernels' medians
P2='import json,sys;d=json.load(open(sys.argv[1]));k=d["config"].get("kernels",{});print(sys.argv[2],round(d["value"]),{n:round(v.get("median_ms",0)*1e3,1) for n,v in k.items()})'
cfg() { name=$1; shift; env "$@" timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 --warmup 3 --config $name > gpurun_out/c_$name.json 2>gpurun_out/c_$name.err; python -c "$P2" gpurun_out/c_$name.json $name; }
