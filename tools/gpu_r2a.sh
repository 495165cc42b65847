# round 2: full GPU test suite + smoke + bench (both arms) on one B200
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 2>&1 | tail -60 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
tail -25 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench.json; tail -c 600 gpurun_out/bench_reference.json
