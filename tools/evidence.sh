# round evidence batch: GPU tests, smoke, C3 profile round, one bench line per config, reference arm
tag=${1:-r2f}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_gpu_tests.log
timeout 300 python __graft_entry__.py > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 bash tools/profile_round.sh C3 $tag > gpurun_out/${tag}_prof_C3.log 2>&1; echo "profile rc=$?"
timeout 2400 bash tools/bench_all.sh; cp gpurun_out/bench_all.jsonl gpurun_out/${tag}_bench_all.jsonl; echo "bench_all done"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_bench_reference.json 2>gpurun_out/${tag}_ref.err; echo "ref rc=$?"
