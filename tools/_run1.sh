set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2d_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python __graft_entry__.py > gpurun_out/r2d_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r2d_bench_C3.json 2> gpurun_out/r2d_bench_C3.err; echo "bench rc=$?"
tail -1 gpurun_out/r2d_bench_C3.json | cut -c1-600
