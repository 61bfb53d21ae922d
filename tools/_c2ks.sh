# float consensus bands per block: C2 it/s and K2f time; then the float parity tests
p() { python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['config']['kernels']
print('$1', round(d['value']), 'K1', round(k['K1_block_mincut']['median_ms']*1e3,1), 'K2 med', round(k['K2_consensus']['median_ms']*1e3,1), 'avg', round(k['K2_consensus']['avg_ms']*1e3,1))"; }
for ks in 1 2 4; do DOPE_F_KS=$ks timeout 300 python bench.py --config C2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | p "C2 ks=$ks"; done
timeout 600 python -m pytest tests/test_full_traces.py tests/test_gpu_parity.py tests/test_step_api_gpu.py -x -q -k "float or c2 or C2 or step or serving" 2>&1 | tail -3
