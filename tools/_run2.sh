timeout 600 python -m pytest tests/test_step_api_gpu.py tests/test_full_traces.py tests/test_host_api_gpu.py -x -q > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2e_tests.log
timeout 300 python tools/public_api_probe.py C3 5 > gpurun_out/r2e_probe_C3.log 2>&1; head -9 gpurun_out/r2e_probe_C3.log
timeout 600 python bench.py --steps 5 > gpurun_out/r2e_bench_C3.json 2> gpurun_out/r2e_bench_C3.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r2e_bench_C3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e_public_api'])"
