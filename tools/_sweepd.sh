# dense-round sweeps per round: K1 first launch and it/s
for cfg in C3 C5-b64 C5-b128 C5-b32; do
for s in "1 0" "2 0" "3 0"; do
  set -- $s
  DOPE_SWEEPD_MIN=$1 DOPE_SWEEPD_MUL=$2 timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['config']['kernels']['K1_block_mincut']
print('$cfg', 'dmin=$1 dmul=$2', round(d['value']), 'K1 first3', [round(x*1e3,1) for x in k['first3_ms']], 'K1 avg', round(k['avg_ms']*1e3,2))"
done; done
