p() { python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['config']['kernels']['K1_block_mincut']
print('$1', round(d['value']), 'K1 first3', [round(x*1e3,1) for x in k['first3_ms']], 'K1 avg', round(k['avg_ms']*1e3,2), 'med', round(k['median_ms']*1e3,2))"; }
for cfg in C1 C3; do timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | p "$cfg auto"; done
for s in "2 0" "4 0" "6 0" "1 1"; do set -- $s
  DOPE_SWEEP3_MIN=$1 DOPE_SWEEP3_MUL=$2 timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | p "C4 s3min=$1 mul=$2"; done
timeout 300 python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | p "C4 default"
for w in 0 1; do DOPE_K1_WIDE=$w timeout 300 python bench.py --config C5-b64 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | p "C5-b64 wide=$w"; done
